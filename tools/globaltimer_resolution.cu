#include <cstdio>
__global__ void k(unsigned long long *out) {
    unsigned long long prev, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
    int n = 0;
    long long c0 = clock64();
    while (n < 16) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t != prev) { out[n++] = t - prev; prev = t; }
    }
    out[16] = clock64() - c0;
}
int main() {
    unsigned long long *o; cudaMallocManaged(&o, 17 * 8);
    k<<<1, 1>>>(o); cudaDeviceSynchronize();
    printf("globaltimer increments (ns):"); for (int i = 0; i < 16; i++) printf(" %llu", o[i]); printf("  (%llu cycles)\n", o[16]);
}
