#include <cstdio>
__global__ void k(double *out, long long *cyc, double x, int n) {
    double a = x, b = x * 0.5;
    long long t0 = clock64();
    for (int i = 0; i < n; i++) a = __dadd_rn(a, b);
    long long t1 = clock64();
    double m = x;
    for (int i = 0; i < n; i++) m = __dmul_rn(m, 1.0000001);
    long long t2 = clock64();
    float f = (float)x;
    for (int i = 0; i < n; i++) f = __fadd_rn(f, 0.5f);
    long long t3 = clock64();
    out[0] = a + m + f;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2;
}
int main() {
    double *o; long long *c; cudaMalloc(&o, 8); cudaMallocManaged(&c, 24);
    k<<<1, 1>>>(o, c, 1.0, 4096); cudaDeviceSynchronize();
    k<<<1, 1>>>(o, c, 1.0, 4096); cudaDeviceSynchronize();
    printf("DADD %.1f cyc, DMUL %.1f cyc, FADD %.1f cyc per dependent op\n", c[0] / 4096.0, c[1] / 4096.0, c[2] / 4096.0);
}
