// Host->device bandwidth on this box: copy engine (cudaMemcpyAsync from pinned memory) against
// kernel loads of mapped pinned memory (zero copy), for the e2e leg's input sizes.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_read(const int4 *__restrict__ src, int4 *__restrict__ dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

int main() {
    const size_t sizes[] = {66668, 200000, 266668, 1 << 20, 4 << 20};
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (size_t bytes : sizes) {
        const size_t n16 = (bytes + 15) / 16;
        void *h, *d;
        cudaHostAlloc(&h, n16 * 16, cudaHostAllocMapped | cudaHostAllocPortable);
        cudaMalloc(&d, n16 * 16);
        float best_ce = 1e9, best_zc = 1e9, best_zc2 = 1e9;
        for (int rep = 0; rep < 50; rep++) {
            cudaEventRecord(a, st);
            cudaMemcpyAsync(d, h, n16 * 16, cudaMemcpyHostToDevice, st);
            cudaEventRecord(b, st);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best_ce) best_ce = ms;
            cudaEventRecord(a, st);
            k_read<<<148 * 4, 256, 0, st>>>((const int4 *)h, (int4 *)d, n16);
            cudaEventRecord(b, st);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best_zc) best_zc = ms;
            cudaEventRecord(a, st);
            k_read<<<148, 128, 0, st>>>((const int4 *)h, (int4 *)d, n16);
            cudaEventRecord(b, st);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best_zc2) best_zc2 = ms;
        }
        printf("%8zu B: copy engine %6.1f us (%5.1f GB/s)   zero-copy 592x256 %6.1f us (%5.1f GB/s)   148x128 %6.1f us\n",
               bytes, best_ce * 1e3, bytes / (best_ce * 1e6), best_zc * 1e3, bytes / (best_zc * 1e6), best_zc2 * 1e3);
        cudaFreeHost(h);
        cudaFree(d);
    }
    return 0;
}
