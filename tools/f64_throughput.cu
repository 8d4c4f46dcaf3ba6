// FP64 latency and throughput on this GPU: dependent chains (latency) and 8 independent chains per
// thread over a full grid (throughput, DADD / DMUL warp-instructions per SM per clock).
#include <cstdio>
__global__ void lat(double *out, long long *cyc, double x, int n) {
    double a = x, b = x * 0.5;
    long long t0 = clock64();
    for (int i = 0; i < n; i++) a = __dadd_rn(a, b);
    long long t1 = clock64();
    out[0] = a;
    cyc[0] = t1 - t0;
}
__global__ void thr(double *out, double x, int n) {
    double a[8];
#pragma unroll
    for (int j = 0; j < 8; j++) a[j] = x + j;
    for (int i = 0; i < n; i++)
#pragma unroll
        for (int j = 0; j < 8; j++) a[j] = __dmul_rn(__dadd_rn(a[j], 1.0000001), 0.9999999);
    double s = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) s += a[j];
    if (s == 12345.0) out[0] = s;
}
int main() {
    double *o; long long *c; cudaMalloc(&o, 8); cudaMallocManaged(&c, 8);
    lat<<<1, 1>>>(o, c, 1.0, 4096); cudaDeviceSynchronize();
    lat<<<1, 1>>>(o, c, 1.0, 4096); cudaDeviceSynchronize();
    printf("DADD dependent latency %.1f cycles\n", c[0] / 4096.0);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int n = 4096, blocks = sms * 8, threads = 256;
    thr<<<blocks, threads>>>(o, 1.0, 16); cudaDeviceSynchronize();
    cudaEventRecord(e0); thr<<<blocks, threads>>>(o, 1.0, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 2.0 * 8 * n * (double)blocks * threads;  // DADD + DMUL per chain step
    const double warp_instr = ops / 32.0;
    printf("FP64 throughput: %.2f TFLOP-ish ops/s (%.0f ops), %.2f warp-instr/SM/clk at %d kHz, %d SMs\n",
           ops / (ms * 1e-3) / 1e12, ops, warp_instr / (ms * 1e-3) / sms / (clk * 1e3), clk, sms);
}
