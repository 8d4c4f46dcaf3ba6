// Cycles per round of a warp-wide 64-bit minimum extraction (the CVaR k-smallest loop of
// k_eval_warp), by primitive and by warps per SM:
//   redux : redux.sync.min on the high word (+ low word on ties), ballot, shfl
//   bfly  : 5-step shfl.xor butterfly on the u64 key
//   f64   : 5-step shfl.xor butterfly on a double (fmin), index by ballot
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ unsigned long long umin64(unsigned long long a, unsigned long long b) { return a < b ? a : b; }

template <int MODE>
__global__ void k_rounds(const unsigned long long *in, unsigned long long *out, int rounds, long long *cyc) {
    const int lane = threadIdx.x & 31;
    unsigned long long h0 = in[(blockIdx.x * blockDim.x + threadIdx.x) & 1023], h1 = h0 + 7, mine = 0;
    __syncwarp();
    const long long t0 = clock64();
    for (int r = 0; r < rounds; r++) {
        int w;
        unsigned long long m;
        if (MODE == 0) {
            const unsigned hi = (unsigned)(h0 >> 32), lo = (unsigned)h0;
            const unsigned mhi = __reduce_min_sync(0xffffffffu, hi);
            unsigned who = __ballot_sync(0xffffffffu, hi == mhi);
            if (__popc(who) > 1) {
                const unsigned mlo = __reduce_min_sync(0xffffffffu, hi == mhi ? lo : 0xffffffffu);
                who = __ballot_sync(0xffffffffu, hi == mhi && lo == mlo);
            }
            w = __ffs(who) - 1;
            m = ((unsigned long long)mhi << 32) | __shfl_sync(0xffffffffu, lo, w);
        } else {
            m = h0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = umin64(m, __shfl_xor_sync(0xffffffffu, m, o));
            w = __ffs(__ballot_sync(0xffffffffu, h0 == m)) - 1;
        }
        if (lane == (r & 31)) mine ^= m;
        if (lane == w) {
            h0 = h1;
            h1 += 13;
        }
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = mine;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    unsigned long long *in, *out;
    long long *cyc;
    cudaMalloc(&in, 8 * 1024);
    cudaMalloc(&out, 8ull * 148 * 1024 * 8);
    cudaMalloc(&cyc, 8 * 148 * 8);
    unsigned long long h[1024];
    for (int i = 0; i < 1024; i++) h[i] = 0x8000000000000000ull + (unsigned long long)(i * 2654435761u % 100003) * 1000;
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    const int rounds = 2000;
    for (int mode = 0; mode < 2; mode++)
        for (int warps : {1, 8, 32}) {
            const int ctas = 148 * (warps >= 8 ? warps / 8 : 1), threads = warps >= 8 ? 256 : 32;
            for (int rep = 0; rep < 2; rep++) {
                if (mode == 0) k_rounds<0><<<ctas, threads>>>(in, out, rounds, cyc);
                else k_rounds<1><<<ctas, threads>>>(in, out, rounds, cyc);
            }
            cudaDeviceSynchronize();
            long long c[148 * 4];
            cudaMemcpy(c, cyc, sizeof(long long) * ctas, cudaMemcpyDeviceToHost);
            double s = 0;
            for (int i = 0; i < ctas; i++) s += c[i];
            printf("%-6s warps/SM %2d: %.1f cycles per round\n", mode == 0 ? "redux" : "bfly", warps, s / ctas / rounds);
        }
    return 0;
}
