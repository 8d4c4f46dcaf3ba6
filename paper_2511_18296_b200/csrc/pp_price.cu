// pp_price.cu -- the feasible-sequence greedy of column generation's pricing step,
// colgen.price_column (colgen.py:236-254), on the device.
//
// Per period t the reference repeatedly scans every block in id order; a block is eligible when
// it is not in the column, fits the period (`masses[b] + load > cap` fails) and all its
// predecessors are in the column at periods <= t; each eligible block counts one expansion, and
// the scan keeps the first block whose score exceeds the running best by more than 1e-12
// (starting from 0.0). The pick joins the column at t; the period ends when a scan picks
// nothing, and the whole construction stops once the expansion count reaches node_cap (checked
// before each scan).
//
// One CTA runs the whole construction (a few scans per column at the default node_cap; no host
// round trip per scan). Each scan is one parallel pass: eligibility flags, their count, and the
// first maximum score. The tolerance scan is not associative, but its result is the first
// maximum whenever no other eligible score lies within 1e-12 (+ rounding) of the maximum: every
// earlier record is then too small to block it and nothing later can displace it. Otherwise
// (near-ties) one thread replays the reference's sequential scan over the flags.
#include "pp_internal.cuh"

constexpr int PR_THREADS = 1024;

__device__ __forceinline__ void pr_better(double &v, int &i, double ov, int oi) {
    if (ov > v || (ov == v && oi < i)) {
        v = ov;
        i = oi;
    }
}

__global__ void __launch_bounds__(PR_THREADS, 1)
    k_price_greedy(const BlockRow *__restrict__ rows, const int32_t *__restrict__ adj, const double *__restrict__ score,
                   const double *__restrict__ cap, int B, int T, long long node_cap, int32_t *assign,
                   unsigned char *elig, long long *exp_out) {
    __shared__ double s_v[PR_THREADS / 32];
    __shared__ int s_i[PR_THREADS / 32], s_n[PR_THREADS / 32], s_pick;
    __shared__ long long s_exp;
    __shared__ double s_load;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int b = tid; b < B; b += PR_THREADS) assign[b] = -1;
    if (tid == 0) s_exp = 0;
    __syncthreads();
    for (int t = 0; t < T; t++) {
        const double cap_t = cap[t];
        if (tid == 0) s_load = 0.0;
        __syncthreads();
        while (s_exp < node_cap) {
            const double load = s_load;
            int cnt = 0, mi = INT_MAX;
            double mx = -INFINITY;
            for (int b = tid; b < B; b += PR_THREADS) {
                bool e = false;
                if (assign[b] < 0) {
                    const BlockRow r = rows[b];
                    if (!(f64_add(r.mass, load) > cap_t)) {
                        e = true;
                        const int np = r.cnt & 0xffff;
                        for (int k = 0; k < np; k++) {
                            const int tp = assign[__ldg(adj + r.adj + k)];
                            if (tp < 0 || tp > t) {
                                e = false;
                                break;
                            }
                        }
                    }
                }
                elig[b] = e;
                if (e) {
                    cnt++;
                    pr_better(mx, mi, __ldg(score + (size_t)b * T + t), b);
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
                pr_better(mx, mi, __shfl_xor_sync(0xffffffffu, mx, o), __shfl_xor_sync(0xffffffffu, mi, o));
            }
            if (lane == 0) {
                s_n[warp] = cnt;
                s_v[warp] = mx;
                s_i[warp] = mi;
            }
            __syncthreads();
            int total = 0;
            mx = -INFINITY;
            mi = INT_MAX;
            for (int w = 0; w < PR_THREADS / 32; w++) {
                total += s_n[w];
                pr_better(mx, mi, s_v[w], s_i[w]);
            }
            // a record needs score > fl(best + 1e-12) >= 1e-12 (best starts at 0.0)
            const bool any = total > 0 && mx > 1e-12;
            int band = 0;
            if (any) {  // eligible scores that could tie with the maximum under the tolerance
                const double ulp = __longlong_as_double(__double_as_longlong(mx) + 1) - mx;  // mx > 0
                const double lo = mx - (4e-12 + 8.0 * ulp);
                for (int b = tid; b < B; b += PR_THREADS)
                    if (elig[b] && __ldg(score + (size_t)b * T + t) >= lo) band++;
            }
            __syncthreads();  // s_n reused below
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) band += __shfl_xor_sync(0xffffffffu, band, o);
            if (lane == 0) s_n[warp] = band;
            __syncthreads();
            if (tid == 0) {
                int nb = 0;
                for (int w = 0; w < PR_THREADS / 32; w++) nb += s_n[w];
                int pick = -1;
                if (any) {
                    if (nb == 1) {
                        pick = mi;
                    } else {  // near-ties: the reference's sequential scan (colgen.py:243-251)
                        double best = 0.0;
                        for (int b = 0; b < B; b++)
                            if (elig[b]) {
                                const double x = score[(size_t)b * T + t];
                                if (x > f64_add(best, 1e-12)) {
                                    best = x;
                                    pick = b;
                                }
                            }
                    }
                }
                s_exp += total;
                s_pick = pick;
                if (pick >= 0) {
                    assign[pick] = t;
                    s_load = f64_add(s_load, rows[pick].mass);
                }
            }
            __syncthreads();
            if (s_pick < 0) break;
        }
        __syncthreads();
    }
    if (tid == 0) *exp_out = s_exp;
}

int pp_price_greedy(pp_ctx *c, const double *score, const double *cap, int64_t node_cap, int32_t *assign_out,
                    int64_t *expansions_out) {
    if (!c || !c->have_instance) return fail(PP_ERR_STATE, "pp_set_instance first");
    if (!score || !cap || !assign_out) return fail(PP_ERR_INVALID_ARGS, "NULL argument");
    TRY(use_device(c));
    const int B = c->B, T = c->T;
    TRY(c->pr_score.ensure(sizeof(double) * (size_t)B * T));
    TRY(c->pr_cap.ensure(sizeof(double) * T));
    TRY(c->pr_assign.ensure(sizeof(int32_t) * B + 64));
    TRY(c->pr_elig.ensure((size_t)B + 16));
    CUDA_TRY(cudaMemcpyAsync(c->pr_score.ptr, score, sizeof(double) * (size_t)B * T, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->pr_cap.ptr, cap, sizeof(double) * T, cudaMemcpyHostToDevice, c->stream));
    int32_t *d_assign = c->pr_assign.as<int32_t>();
    long long *d_exp = reinterpret_cast<long long *>(d_assign + ((B + 1) & ~1));
    k_price_greedy<<<1, PR_THREADS, 0, c->stream>>>(c->rows.as<BlockRow>(), c->adj.as<int32_t>(), c->pr_score.as<double>(),
                                                    c->pr_cap.as<double>(), B, T, (long long)node_cap, d_assign,
                                                    c->pr_elig.as<unsigned char>(), d_exp);
    CUDA_TRY(cudaGetLastError());
    long long ex = 0;
    CUDA_TRY(cudaMemcpyAsync(assign_out, d_assign, sizeof(int32_t) * B, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaMemcpyAsync(&ex, d_exp, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (expansions_out) *expansions_out = ex;
    return PP_OK;
}
