// Micro-benchmark of the stage-2 greedy walk (evaluate.py:174-182) as the warp runs it: one warp
// walks n elements (q = m / rate, dm = d * m), cycles per element for loop variants.  V3 (inputs
// one batch ahead, the batch's terms read eight at a time into registers) is what pp_npv.cu uses
// (s2_batch_steps).  A chain per lane (32 chains per warp, q precomputed, 4-deep register ring)
// measured ~190 cycles per element per chain: its uncoalesced loads are not hidden; software
// pipelining across batches (the next chain while the previous stop test resolves) ~27.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tools/bin/walk_bench tools/walk_bench.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ double f64_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double f64_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double f64_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double f64_div(double a, double b) { return __ddiv_rn(a, b); }

// variant 0: the production loop (smem broadcast, unroll 8)
template <int V>
__global__ void walk(const double *D, const double *M, int n, double rate, double h0, double *out, long long *cyc) {
    __shared__ double s_q[32], s_dm[32], s_h[32], s_t[32];
    const int lane = threadIdx.x & 31;
    double hl = h0, tot = 0.0;
    long long t0 = clock64();
    double m_nx = lane < n ? M[lane] : 0.0, d_nx = lane < n ? D[lane] : 0.0;
    // V4 pipeline: raw inputs two batches ahead, terms one batch ahead
    double m2 = lane + 32 < n ? M[lane + 32] : 0.0, d2 = lane + 32 < n ? D[lane + 32] : 0.0;
    double m1 = m_nx, q1 = lane < n ? f64_div(m_nx, rate) : 0.0, dm1 = lane < n ? f64_mul(d_nx, m_nx) : 0.0;
    for (int k0 = 0; k0 < n; k0 += 32) {
        const int kk = k0 + lane;
        const bool in = kk < n;
        double m, q, dm;
        if (V == 4) {
            m = m1; q = in ? q1 : 0.0; dm = in ? dm1 : 0.0;
            const bool in1 = kk + 32 < n;
            m1 = m2;
            q1 = in1 ? f64_div(m2, rate) : 0.0;
            dm1 = in1 ? f64_mul(d2, m2) : 0.0;
            if (kk + 64 < n) { m2 = M[kk + 64]; d2 = D[kk + 64]; }
        } else if (V == 3 || V >= 5) {  // this batch's inputs were loaded one batch ahead
            m = in ? m_nx : 0.0;
            q = in ? f64_div(m, rate) : 0.0;
            dm = in ? f64_mul(d_nx, m) : 0.0;
            if (kk + 32 < n) { m_nx = M[kk + 32]; d_nx = D[kk + 32]; }
        } else {
            m = in ? M[kk] : 0.0;
            q = in ? f64_div(m, rate) : 0.0;
            dm = in ? f64_mul(D[kk], m) : 0.0;
        }
        double h = hl, tt = tot, h_mine = 0.0, t_mine = 0.0;
        if (V == 0 || V == 6) {
            s_q[lane] = q;
            s_dm[lane] = dm;
            __syncwarp();
#pragma unroll 8
            for (int j = 0; j < 32; j++) {
                if (lane == j) { h_mine = h; t_mine = tt; }
                h = f64_sub(h, s_q[j]);
                tt = f64_add(tt, s_dm[j]);
            }
            __syncwarp();
        } else if (V == 1) {  // shuffles, full unroll
#pragma unroll
            for (int j = 0; j < 32; j++) {
                const double qj = __shfl_sync(0xffffffffu, q, j), dj = __shfl_sync(0xffffffffu, dm, j);
                if (lane == j) { h_mine = h; t_mine = tt; }
                h = f64_sub(h, qj);
                tt = f64_add(tt, dj);
            }
        } else if (V == 7) {  // as V3, lanes stop at their own element (predicated adds), no selects
            s_q[lane] = q;
            s_dm[lane] = dm;
            __syncwarp();
#pragma unroll
            for (int g = 0; g < 4; g++) {
                double qa[8], da[8];
#pragma unroll
                for (int u = 0; u < 8; u++) { qa[u] = s_q[g * 8 + u]; da[u] = s_dm[g * 8 + u]; }
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    if (g * 8 + u < lane) {
                        h = f64_sub(h, qa[u]);
                        tt = f64_add(tt, da[u]);
                    }
                }
            }
            h_mine = h;
            t_mine = tt;
            // the batch's end state: lane 31's state minus its own element
            h = __shfl_sync(0xffffffffu, f64_sub(h, q), 31);
            tt = __shfl_sync(0xffffffffu, f64_add(tt, dm), 31);
            __syncwarp();
        } else if (V == 9) {  // as V3, the next group's terms loaded while this group's steps run
            s_q[lane] = q;
            s_dm[lane] = dm;
            __syncwarp();
            double qa[8], da[8], qb[8], db[8];
#pragma unroll
            for (int u = 0; u < 8; u++) { qa[u] = s_q[u]; da[u] = s_dm[u]; }
#pragma unroll
            for (int g = 0; g < 4; g++) {
                if (g < 3) {
#pragma unroll
                    for (int u = 0; u < 8; u++) { qb[u] = s_q[(g + 1) * 8 + u]; db[u] = s_dm[(g + 1) * 8 + u]; }
                }
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    if (lane == g * 8 + u) { h_mine = h; t_mine = tt; }
                    h = f64_sub(h, qa[u]);
                    tt = f64_add(tt, da[u]);
                }
#pragma unroll
                for (int u = 0; u < 8; u++) { qa[u] = qb[u]; da[u] = db[u]; }
            }
            __syncwarp();
        } else if (V == 10) {  // as V3 with groups of 16
            s_q[lane] = q;
            s_dm[lane] = dm;
            __syncwarp();
#pragma unroll
            for (int g = 0; g < 2; g++) {
                double qa[16], da[16];
#pragma unroll
                for (int u = 0; u < 16; u++) { qa[u] = s_q[g * 16 + u]; da[u] = s_dm[g * 16 + u]; }
#pragma unroll
                for (int u = 0; u < 16; u++) {
                    if (lane == g * 16 + u) { h_mine = h; t_mine = tt; }
                    h = f64_sub(h, qa[u]);
                    tt = f64_add(tt, da[u]);
                }
            }
            __syncwarp();
        } else if (V == 11) {  // timing floor only (not the algorithm): V3 without the state captures
            s_q[lane] = q;
            s_dm[lane] = dm;
            __syncwarp();
#pragma unroll
            for (int g = 0; g < 4; g++) {
                double qa[8], da[8];
#pragma unroll
                for (int u = 0; u < 8; u++) { qa[u] = s_q[g * 8 + u]; da[u] = s_dm[g * 8 + u]; }
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    h = f64_sub(h, qa[u]);
                    tt = f64_add(tt, da[u]);
                }
            }
            h_mine = h;
            t_mine = tt;
            __syncwarp();
        } else if (V == 5) {  // as V3, the states stored per step (one broadcast store) instead of selects
            s_q[lane] = q;
            s_dm[lane] = dm;
            __syncwarp();
#pragma unroll
            for (int g = 0; g < 4; g++) {
                double qa[8], da[8];
#pragma unroll
                for (int u = 0; u < 8; u++) { qa[u] = s_q[g * 8 + u]; da[u] = s_dm[g * 8 + u]; }
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    if (lane == 0) { s_h[g * 8 + u] = h; s_t[g * 8 + u] = tt; }
                    h = f64_sub(h, qa[u]);
                    tt = f64_add(tt, da[u]);
                }
            }
            __syncwarp();
            h_mine = s_h[lane];
            t_mine = s_t[lane];
        } else if (V >= 2) {  // smem, groups of 8 in registers
            s_q[lane] = q;
            s_dm[lane] = dm;
            __syncwarp();
            double hs[32 / 32];  // unused
            (void)hs;
#pragma unroll
            for (int g = 0; g < 4; g++) {
                double qa[8], da[8];
#pragma unroll
                for (int u = 0; u < 8; u++) { qa[u] = s_q[g * 8 + u]; da[u] = s_dm[g * 8 + u]; }
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    if (lane == g * 8 + u) { h_mine = h; t_mine = tt; }
                    h = f64_sub(h, qa[u]);
                    tt = f64_add(tt, da[u]);
                }
            }
            __syncwarp();
        }
        const bool stop = !in || !(h_mine > 0) || f64_mul(h_mine, rate) < m;
        const unsigned sm = __ballot_sync(0xffffffffu, stop);
        if (sm) {
            const int jf = __ffs(sm) - 1;
            hl = __shfl_sync(0xffffffffu, h_mine, jf);
            tot = __shfl_sync(0xffffffffu, t_mine, jf);
            break;
        }
        hl = h;
        tot = tt;
    }
    long long t1 = clock64();
    if (lane == 0) { out[0] = tot + hl; cyc[0] = t1 - t0; }
}

// V12: 64 elements per batch (lane l holds elements l and 32 + l), inputs one batch ahead
__global__ void walk64(const double *D, const double *M, int n, double rate, double h0, double *out, long long *cyc) {
    __shared__ double s_q[64], s_dm[64];
    const int lane = threadIdx.x & 31;
    double hl = h0, tot = 0.0;
    long long t0 = clock64();
    double ma = lane < n ? M[lane] : 0.0, da_ = lane < n ? D[lane] : 0.0;
    double mb = lane + 32 < n ? M[lane + 32] : 0.0, db_ = lane + 32 < n ? D[lane + 32] : 0.0;
    for (int k0 = 0; k0 < n; k0 += 64) {
        const int ka = k0 + lane, kb = k0 + 32 + lane;
        const bool ina = ka < n, inb = kb < n;
        const double m0 = ina ? ma : 0.0, m1 = inb ? mb : 0.0;
        s_q[lane] = ina ? f64_div(m0, rate) : 0.0;
        s_dm[lane] = ina ? f64_mul(da_, m0) : 0.0;
        s_q[32 + lane] = inb ? f64_div(m1, rate) : 0.0;
        s_dm[32 + lane] = inb ? f64_mul(db_, m1) : 0.0;
        if (ka + 64 < n) { ma = M[ka + 64]; da_ = D[ka + 64]; }
        if (kb + 64 < n) { mb = M[kb + 64]; db_ = D[kb + 64]; }
        __syncwarp();
        double h = hl, tt = tot, ha = 0.0, ta = 0.0, hb = 0.0, tb = 0.0;
#pragma unroll
        for (int g = 0; g < 8; g++) {
            double qa[8], dd[8];
#pragma unroll
            for (int u = 0; u < 8; u++) { qa[u] = s_q[g * 8 + u]; dd[u] = s_dm[g * 8 + u]; }
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const int j = g * 8 + u;
                if (j < 32) { if (lane == j) { ha = h; ta = tt; } }
                else { if (lane == j - 32) { hb = h; tb = tt; } }
                h = f64_sub(h, qa[u]);
                tt = f64_add(tt, dd[u]);
            }
        }
        __syncwarp();
        const bool sa = !ina || !(ha > 0) || f64_mul(ha, rate) < m0;
        const bool sb = !inb || !(hb > 0) || f64_mul(hb, rate) < m1;
        const unsigned ba = __ballot_sync(0xffffffffu, sa), bb = __ballot_sync(0xffffffffu, sb);
        if (ba | bb) {
            if (ba) { const int jf = __ffs(ba) - 1; hl = __shfl_sync(0xffffffffu, ha, jf); tot = __shfl_sync(0xffffffffu, ta, jf); }
            else { const int jf = __ffs(bb) - 1; hl = __shfl_sync(0xffffffffu, hb, jf); tot = __shfl_sync(0xffffffffu, tb, jf); }
            break;
        }
        hl = h;
        tot = tt;
    }
    long long t1 = clock64();
    if (lane == 0) { out[0] = tot + hl; cyc[0] = t1 - t0; }
}

int main() {
    const int n = 4096;
    double *D, *M, *o; long long *c;
    cudaMallocManaged(&D, n * 8); cudaMallocManaged(&M, n * 8); cudaMallocManaged(&o, 8); cudaMallocManaged(&c, 8);
    for (int i = 0; i < n; i++) { D[i] = 1.0 + 1e-3 * (n - i); M[i] = 100.0 + (i % 7); }
    const double rate = 1000.0, h0 = 1e9;  // never stops: the whole list
    for (int rep = 0; rep < 2; rep++) {
        walk<0><<<1, 32>>>(D, M, n, rate, h0, o, c); cudaDeviceSynchronize();
        printf("V0 smem unroll8: %.1f cycles/element\n", c[0] / (double)n);
        walk<1><<<1, 32>>>(D, M, n, rate, h0, o, c); cudaDeviceSynchronize();
        printf("V1 shfl unroll32: %.1f cycles/element\n", c[0] / (double)n);
        walk<2><<<1, 32>>>(D, M, n, rate, h0, o, c); cudaDeviceSynchronize();
        printf("V2 smem groups of 8 in regs: %.1f cycles/element\n", c[0] / (double)n);
        walk<3><<<1, 32>>>(D, M, n, rate, h0, o, c); cudaDeviceSynchronize();
        printf("V3 = V2 + inputs one batch ahead: %.1f cycles/element\n", c[0] / (double)n);
        walk<4><<<1, 32>>>(D, M, n, rate, h0, o, c); cudaDeviceSynchronize();
        printf("V4 = V2 + inputs two ahead, terms one ahead: %.1f cycles/element\n", c[0] / (double)n);
        walk<5><<<1, 32>>>(D, M, n, rate, h0, o, c); cudaDeviceSynchronize();
        printf("V5 = V3, states stored per step: %.1f cycles/element\n", c[0] / (double)n);
        walk<6><<<1, 32>>>(D, M, n, rate, h0, o, c); cudaDeviceSynchronize();
        printf("V6 = V0 (unroll 8) + inputs one batch ahead: %.1f cycles/element\n", c[0] / (double)n);
        walk<7><<<1, 32>>>(D, M, n, rate, h0, o, c); cudaDeviceSynchronize();
        const double r7 = o[0];
        walk<3><<<1, 32>>>(D, M, n, rate, h0, o, c); cudaDeviceSynchronize();
        printf("V7 = V3, lanes stop at their element: same result %d\n", (int)(o[0] == r7));
        walk<7><<<1, 32>>>(D, M, n, rate, h0, o, c); cudaDeviceSynchronize();
        printf("V7 = V3, lanes stop at their element: %.1f cycles/element\n", c[0] / (double)n);
        walk<9><<<1, 32>>>(D, M, n, rate, h0, o, c); cudaDeviceSynchronize();
        printf("V9 = V3, next group loaded during this group: %.1f cycles/element\n", c[0] / (double)n);
        walk<10><<<1, 32>>>(D, M, n, rate, h0, o, c); cudaDeviceSynchronize();
        printf("V10 = V3 with groups of 16: %.1f cycles/element\n", c[0] / (double)n);
        walk<11><<<1, 32>>>(D, M, n, rate, h0, o, c); cudaDeviceSynchronize();
        printf("V11 (floor, no captures): %.1f cycles/element\n", c[0] / (double)n);
        walk<3><<<1, 32>>>(D, M, n, rate, h0, o, c); cudaDeviceSynchronize();
        const double r3 = o[0];
        walk64<<<1, 32>>>(D, M, n, rate, h0, o, c); cudaDeviceSynchronize();
        printf("V12 64 elements per batch: %.1f cycles/element (same result %d)\n", c[0] / (double)n, (int)(o[0] == r3));
    }
}

