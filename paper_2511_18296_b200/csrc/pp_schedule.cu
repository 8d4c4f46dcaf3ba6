// pp_schedule.cu -- schedule-side kernels: bit-exact period masses (numpy pairwise tree),
// check_feasible, topological-wave repair, table preparation, and their C-ABI entry points.
#include "pp_internal.cuh"
#include <limits>

// ------------------------------------------------------------------------------------
// period mass, bit-exact numpy pairwise summation per period (evaluate.py:334-337)
//
// k_pm_chunks (P1): CTA c of schedule p owns blocks [c*512, (c+1)*512): one coalesced load
//   of assign and mass per thread; the rank of a block among same-period blocks is
//   (lower warps' count) + popc(match_any & lanemask_lt) -- stable, block order.  The CTA
//   publishes its per-period counts, looks back over the published counts of lower chunks
//   (all P1 CTAs are resident once they have triggered their PDL dependents), and
//   scatters masses into per-period compacted arrays compact[p][t][.].
// k_pm_tree (P2): one CTA per (period, schedule): numpy's recursion laid out as a heap
//   (node id, children 2id+1 | 2id+2); in units of 8-blocks a node of m blocks splits
//   floor(m/2) | ceil(m/2), leaves hold <= 128 elements.  Built level-parallel top-down,
//   leaf sums with 8 lanes per leaf (lane j = accumulator j, a butterfly reproduces
//   ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))), then folded level-parallel bottom-up:
//   pm = 0.0 + root.
// ------------------------------------------------------------------------------------
constexpr int PM_THREADS = 512;
constexpr int PM_MAXT = 128;
constexpr int PM_CH = 512;             // blocks per P1 chunk (one per thread)
constexpr int PM_MAX_DEPTH = 10;       // heap levels 0..10: n <= 128 * 2^10 = 131072 per period
constexpr int PM_HEAP = (1 << (PM_MAX_DEPTH + 1)) - 1;

// serial pairwise sum (pathological sizes only)
__device__ double pairwise_serial(const double *a, int n) {
    double vst[64];
    int stk_o[64], stk_n[64], sp = 0, vp = 0;
    stk_o[sp] = 0;
    stk_n[sp] = n;
    sp++;
    while (sp > 0) {
        sp--;
        int o = stk_o[sp], m = stk_n[sp];
        if (m < 0) {
            double rhs = vst[--vp];
            double lhs = vst[--vp];
            vst[vp++] = f64_add(lhs, rhs);
            continue;
        }
        if (m <= 128) {
            double res;
            if (m < 8) {
                res = -0.0;
                for (int i = 0; i < m; i++) res = f64_add(res, a[o + i]);
            } else {
                double r[8];
                for (int j = 0; j < 8; j++) r[j] = a[o + j];
                int i = 8;
                for (; i < m - (m % 8); i += 8)
                    for (int j = 0; j < 8; j++) r[j] = f64_add(r[j], a[o + i + j]);
                res = tree8(r);
                for (; i < m; i++) res = f64_add(res, a[o + i]);
            }
            vst[vp++] = res;
            continue;
        }
        int n2 = m / 2;
        n2 -= n2 % 8;
        stk_o[sp] = 0;
        stk_n[sp] = -1;
        sp++;
        stk_o[sp] = o + n2;
        stk_n[sp] = m - n2;
        sp++;
        stk_o[sp] = o;
        stk_n[sp] = n2;
        sp++;
    }
    return vp ? vst[0] : -0.0;
}


#ifdef PP_EVAL_PROBE
__device__ unsigned long long g_pm_probe[2][512][2];
__device__ __forceinline__ unsigned long long pm_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define PMP(k, j) do { const int i_ = (k) ? (int)blockIdx.x - nchunk : (int)blockIdx.x; if (threadIdx.x == 0 && blockIdx.y == 0 && i_ < 512) g_pm_probe[k][i_][j] = pm_gtimer(); } while (0)
extern "C" PP_API int pp_debug_pm_probe(unsigned long long *out) {
    return cudaMemcpyFromSymbol(out, g_pm_probe, sizeof(g_pm_probe)) == cudaSuccess ? 0 : 3;
}
#else
#define PMP(k, j) do { } while (0)
#endif
#ifdef PP_EVAL_PROBE
#define PMCP(k, j) do { if (threadIdx.x == 0 && blockIdx.y == 0) g_pm_probe[k][blockIdx.x][j] = pm_gtimer(); } while (0)
#define PMCS(st) do { if (threadIdx.x == 0 && blockIdx.y == 0) g_pm_probe[1][16 + 16 * (st) + blockIdx.x][0] = pm_gtimer(); } while (0)
#else
#define PMCS(st) do { } while (0)
#define PMCP(k, j) do { } while (0)
#endif

__device__ void pm_chunk_cta(const int32_t *__restrict__ assign, const double *__restrict__ mass, int B, int T,
                             int nchunk, int c, int p, int32_t *__restrict__ agg, int32_t *__restrict__ flags,
                             double *__restrict__ compact, int (*s_cnt)[PM_MAXT], int *s_base) {
    PMP(0, 0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int b = c * PM_CH + tid;
    int t = (b < B) ? __ldg(assign + (size_t)p * B + b) : -1;
    if (t < 0 || t >= T) t = -1;
    const double m = (b < B) ? __ldg(mass + b) : 0.0;
    for (int i = tid; i < (PM_THREADS / 32) * PM_MAXT; i += PM_THREADS) (&s_cnt[0][0])[i] = 0;
    __syncthreads();
    const unsigned mt = __match_any_sync(0xffffffffu, t);
    const int rank_w = __popc(mt & ((1u << lane) - 1u));
    if (t >= 0 && rank_w == 0) s_cnt[warp][t] = __popc(mt);
    __syncthreads();
    int32_t *my_agg = agg + ((size_t)p * nchunk + c) * T;
    for (int j = tid; j < T; j += PM_THREADS) {
        int run = 0;
        for (int w = 0; w < PM_THREADS / 32; w++) {
            const int x = s_cnt[w][j];
            s_cnt[w][j] = run;
            run += x;
        }
        my_agg[j] = run;
    }
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.b32 [%0], %1;" :: "l"(flags + (size_t)p * nchunk + c), "r"(1) : "memory");
    }
    // look-back: warp 0 waits until every lower chunk has published (flags polled with
    // independent acquire loads), then base[j] = sum of lower chunks' counts of period j
    if (warp == 0) {
        const int32_t *fl = flags + (size_t)p * nchunk;
        for (;;) {
            bool ok = true;
            for (int k0 = 0; k0 < c; k0 += 128) {
                int f[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int k = k0 + u * 32 + lane;
                    f[u] = 1;
                    if (k < c) asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(f[u]) : "l"(fl + k) : "memory");
                }
                ok &= (f[0] != 0) & (f[1] != 0) & (f[2] != 0) & (f[3] != 0);
            }
            if (__all_sync(0xffffffffu, ok)) break;
            __nanosleep(64);
        }
    }
    __syncthreads();
    for (int j = warp; j < T; j += PM_THREADS / 32) {
        int sum = 0;
        for (int k0 = 0; k0 < c; k0 += 128) {
            int v[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int k = k0 + u * 32 + lane;
                v[u] = (k < c) ? __ldcg(agg + ((size_t)p * nchunk + k) * T + j) : 0;
            }
            sum += v[0] + v[1] + v[2] + v[3];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == 0) s_base[j] = sum;
    }
    __syncthreads();
    if (t >= 0) compact[((size_t)p * T + t) * B + s_base[t] + s_cnt[warp][t] + rank_w] = m;
    PMP(0, 1);
}

struct PmTreeSmem {
    int start[PM_HEAP];
    int len[PM_HEAP];  // -1: dead (below a leaf)
    double val[PM_HEAP];
    int leaves[1 << PM_MAX_DEPTH];
    int nleaf;
    int depth;
    int total;
};

__device__ void pm_tree_cta(const int32_t *__restrict__ agg, int32_t *__restrict__ flags,
                            const double *__restrict__ compact, int B, int T, int nchunk, int t, int p,
                            double *__restrict__ pm_out, PmTreeSmem &sm) {
    PMP(1, 0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (warp == 0) {
        int sum = 0;
        for (int k0 = 0; k0 < nchunk; k0 += 128) {
            int v[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int k = k0 + u * 32 + lane;
                v[u] = (k < nchunk) ? __ldcg(agg + ((size_t)p * nchunk + k) * T + t) : 0;
            }
            sum += v[0] + v[1] + v[2] + v[3];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == 0) {
            sm.total = sum;
            sm.nleaf = 0;
        }
    }
    // re-arm the look-back flags of this schedule for the next P1 launch (P1 has finished)
    if (t == 0)
        for (int k = tid; k < nchunk; k += PM_THREADS) flags[(size_t)p * nchunk + k] = 0;
    __syncthreads();
    const int n = sm.total;
    const double *a = compact + ((size_t)p * T + t) * B;
    // top-down heap build
    if (tid == 0) {
        sm.start[0] = 0;
        sm.len[0] = n;
    }
    __syncthreads();
    int depth = 0;
    bool overflow = false;
    for (int d = 0;; d++) {
        const int first = (1 << d) - 1, cnt = 1 << d;
        bool any_internal = false;
        for (int j = tid; j < cnt; j += PM_THREADS) {
            const int id = first + j;
            const int ln = sm.len[id];
            if (ln < 0) continue;
            if (ln <= 128) {
                const int k = atomicAdd(&sm.nleaf, 1);
                sm.leaves[k] = id;
            } else {
                any_internal = true;
                if (d < PM_MAX_DEPTH) {
                    const int n2 = ((ln >> 3) >> 1) << 3;  // floor(m/2) whole 8-blocks left
                    sm.start[2 * id + 1] = sm.start[id];
                    sm.len[2 * id + 1] = n2;
                    sm.start[2 * id + 2] = sm.start[id] + n2;
                    sm.len[2 * id + 2] = ln - n2;
                }
            }
        }
        // children of leaves / dead nodes are dead
        if (d < PM_MAX_DEPTH)
            for (int j = tid; j < cnt; j += PM_THREADS) {
                const int id = first + j;
                const int ln = sm.len[id];
                if (ln <= 128) {
                    sm.len[2 * id + 1] = -1;
                    sm.len[2 * id + 2] = -1;
                }
            }
        const int more = __syncthreads_or(any_internal);
        if (!more) {
            depth = d;
            break;
        }
        if (d == PM_MAX_DEPTH) {
            overflow = true;
            break;
        }
    }
    if (overflow) {  // > 131072 blocks in one period: serial evaluation (correct, slow)
        if (tid == 0) pm_out[(size_t)p * T + t] = f64_add(0.0, pairwise_serial(a, n));
        return;
    }
    // leaf sums
    const int nleaf = sm.nleaf;
    const int sub = tid & 7, grp = tid >> 3, ngrp = PM_THREADS >> 3;
    for (int l0 = 0; l0 < nleaf; l0 += ngrp) {
        const int l = l0 + grp;
        const bool act = l < nleaf;
        const int id = act ? sm.leaves[l] : 0;
        const int o = act ? sm.start[id] : 0;
        const int len = act ? sm.len[id] : 0;
        double r = 0.0;
        if (act && len >= 8) {
            // all (<= 16) loads of this accumulator issued before the sequential adds
            const int nm = len >> 3;
            double x[16];
#pragma unroll
            for (int u = 0; u < 16; u++) x[u] = (u < nm) ? __ldcg(a + o + 8 * u + sub) : 0.0;
            r = x[0];
#pragma unroll
            for (int u = 1; u < 16; u++)
                if (u < nm) r = f64_add(r, x[u]);
        }
        r = f64_add(r, __shfl_xor_sync(0xffffffffu, r, 1));
        r = f64_add(r, __shfl_xor_sync(0xffffffffu, r, 2));
        r = f64_add(r, __shfl_xor_sync(0xffffffffu, r, 4));
        if (act && sub == 0) {
            double res;
            int i;
            if (len < 8) {
                res = -0.0;
                i = 0;
            } else {
                res = r;
                i = len - (len & 7);
            }
            for (; i < len; i++) res = f64_add(res, __ldcg(a + o + i));
            sm.val[id] = res;
        }
    }
    __syncthreads();
    // bottom-up fold: internal node = left + right
    for (int d = depth - 1; d >= 0; d--) {
        const int first = (1 << d) - 1, cnt = 1 << d;
        for (int j = tid; j < cnt; j += PM_THREADS) {
            const int id = first + j;
            if (sm.len[id] > 128) sm.val[id] = f64_add(sm.val[2 * id + 1], sm.val[2 * id + 2]);
        }
        __syncthreads();
    }
    if (tid == 0) pm_out[(size_t)p * T + t] = f64_add(0.0, n ? sm.val[0] : -0.0);
    PMP(1, 1);
}

// One launch computes the period masses of P schedules: CTAs x < nchunk compact a chunk
// (pm_chunk_cta, decoupled look-back across chunks); the last T CTAs of each schedule wait
// until every chunk has scattered, then build one period's pairwise tree (pm_tree_cta).
// Tree CTAs have higher block indices than the chunks they wait for, so they are
// dispatched after them.  done[2p] counts finished chunks, done[2p+1] finished trees; the
// last tree CTA re-arms both (graph-replay safe).
__global__ void __launch_bounds__(PM_THREADS) k_period_mass(const int32_t *__restrict__ assign,
                                                             const double *__restrict__ mass, int B, int T, int nchunk,
                                                             int32_t *__restrict__ agg, int32_t *__restrict__ flags,
                                                             unsigned int *__restrict__ done,
                                                             double *__restrict__ compact, double *__restrict__ pm_out) {
    asm volatile("griddepcontrol.launch_dependents;");
    extern __shared__ __align__(16) unsigned char pm_dyn[];
    const int p = blockIdx.y;
    if ((int)blockIdx.x < nchunk) {
        int(*s_cnt)[PM_MAXT] = reinterpret_cast<int(*)[PM_MAXT]>(pm_dyn);
        int *s_base = reinterpret_cast<int *>(pm_dyn + sizeof(int) * (PM_THREADS / 32) * PM_MAXT);
        pm_chunk_cta(assign, mass, B, T, nchunk, blockIdx.x, p, agg, flags, compact, s_cnt, s_base);
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(done + 2 * p, 1u);
        }
        return;
    }
    const int t = blockIdx.x - nchunk;
    if (threadIdx.x == 0) {
        unsigned int v;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(done + 2 * p) : "memory");
            if ((int)v >= nchunk) break;
            __nanosleep(64);
        }
    }
    __syncthreads();
    pm_tree_cta(agg, flags, compact, B, T, nchunk, t, p, pm_out, *reinterpret_cast<PmTreeSmem *>(pm_dyn));
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned int prev = atomicAdd(done + 2 * p + 1, 1u);
        if ((int)prev == T - 1) {
            done[2 * p] = 0u;
            done[2 * p + 1] = 0u;
        }
    }
}


// ------------------------------------------------------------------------------------
// check_feasible pieces
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_pred_count(const int32_t *__restrict__ assign, const BlockRow *__restrict__ rows,
                                                    const int32_t *__restrict__ adj, int B,
                                                    unsigned long long *__restrict__ out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int p = blockIdx.y;
    const int32_t *a = assign + (size_t)p * B;
    unsigned c = 0;
    if (j < B) {
        int tj = a[j];
        if (tj >= 0) {
            BlockRow r = rows[j];
            int npred = r.cnt & 0xffff;
            for (int k = 0; k < npred; k++) {
                int ti = a[__ldg(adj + r.adj + k)];
                if (ti < 0 || ti > tj) c++;
            }
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out + p, (unsigned long long)c);
}

__global__ void k_feas_final(const double *__restrict__ pm, const double *__restrict__ cap, int T, int P,
                             double mean_cap, const unsigned long long *__restrict__ cnt,
                             int64_t *__restrict__ pred_out, double *__restrict__ excess_out,
                             double *__restrict__ viol_out) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    double ex = 0.0;
    for (int t = 0; t < T; t++) {
        double d = f64_sub(pm[(size_t)p * T + t], cap[t]);
        ex = f64_add(ex, (d > 0.0) ? d : 0.0);  // excess += max(0.0, load - cap)
    }
    unsigned long long c = cnt[p];
    pred_out[p] = (int64_t)c;
    excess_out[p] = ex;
    viol_out[p] = f64_add((double)c, f64_div(ex, mean_cap));
}

// ------------------------------------------------------------------------------------
// lns_repair's over-capacity ejection (hybrid.py:213-235), after the unmine fixpoint.
// Pass 1 (k_eject_list, one thread per block): every mined block of an over-target period
// whose successors are all UNMINED joins its period's list with key mean_grade[b] * mass[b].
// All lists are built from the same state before anything is ejected, which is what the
// reference's ascending-t loop sees: after the fixpoint a block's successors are mined no
// earlier than it, so ejecting in period t never changes the list of a later period.
// Pass 2 (k_eject_apply, one CTA per period): repeatedly the smallest (key, b) is ejected
// while load > target, load -= mass[b] in that order (the reference's sequential loop).
// load = the bit-exact period mass (k_pm_cluster / k_period_mass).
// ------------------------------------------------------------------------------------
__device__ __forceinline__ double eject_target(double load, double cap, double df) {
    return (df > 0 && load > cap) ? f64_mul(cap, f64_sub(1.0, df)) : cap;
}

__global__ void __launch_bounds__(256) k_eject_list(const int32_t *__restrict__ assign, int B, int T,
                                                    const BlockRow *__restrict__ rows,
                                                    const int32_t *__restrict__ adj, const double *__restrict__ pm,
                                                    const double *__restrict__ cap, const double *__restrict__ grade,
                                                    double df, int32_t *__restrict__ count,
                                                    double *__restrict__ lkey, int32_t *__restrict__ lblk) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const int t = assign[b];
    if (t < 0 || t >= T) return;
    const double load = pm[t];
    if (load <= eject_target(load, cap[t], df)) return;
    const BlockRow r = rows[b];
    const int npred = r.cnt & 0xffff, nsucc = r.cnt >> 16;
    for (int e = 0; e < nsucc; e++)
        if (assign[__ldg(adj + r.adj + npred + e)] != -1) return;
    const int k = atomicAdd(count + t, 1);
    lkey[(size_t)t * B + k] = f64_mul(__ldg(grade + b), r.mass);
    lblk[(size_t)t * B + k] = b;
}

__global__ void __launch_bounds__(512) k_eject_apply(int32_t *__restrict__ assign, int B,
                                                     const double *__restrict__ mass, const double *__restrict__ pm,
                                                     const double *__restrict__ cap, double df,
                                                     const int32_t *__restrict__ count,
                                                     const double *__restrict__ lkey, int32_t *__restrict__ lblk,
                                                     uint8_t *__restrict__ ejected) {
    const int t = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = count[t];
    if (n == 0) return;
    const double *key = lkey + (size_t)t * B;
    int32_t *blk = lblk + (size_t)t * B;
    const double target = eject_target(pm[t], cap[t], df);
    __shared__ double s_load;
    __shared__ double s_k[16];
    __shared__ int s_b[16], s_i[16];
    if (tid == 0) s_load = pm[t];
    for (;;) {
        __syncthreads();
        const double load = s_load;
        if (load <= target) break;
        // smallest remaining (key, b): a total order, so the choice is deterministic
        double bk = kInf;
        int bb = INT_MAX, bi = -1;
        for (int i = tid; i < n; i += blockDim.x) {
            const int b = blk[i];
            if (b < 0) continue;
            const double k = key[i];
            if (k < bk || (k == bk && b < bb)) {
                bk = k;
                bb = b;
                bi = i;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
            const int ob = __shfl_xor_sync(0xffffffffu, bb, o), oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ok < bk || (ok == bk && ob < bb)) {
                bk = ok;
                bb = ob;
                bi = oi;
            }
        }
        if (lane == 0) {
            s_k[warp] = bk;
            s_b[warp] = bb;
            s_i[warp] = bi;
        }
        __syncthreads();
        if (tid == 0) {
            double k = s_k[0];
            int b = s_b[0], i = s_i[0];
            for (int w = 1; w < (int)(blockDim.x >> 5); w++)
                if (s_k[w] < k || (s_k[w] == k && s_b[w] < b)) {
                    k = s_k[w];
                    b = s_b[w];
                    i = s_i[w];
                }
            if (i < 0) {
                s_load = -kInf;  // list exhausted: the reference's for-loop ends
            } else {
                assign[b] = -1;
                if (ejected) ejected[b] = 1;
                blk[i] = -1;
                s_load = f64_sub(load, mass[b]);
            }
        }
    }
}

// ------------------------------------------------------------------------------------
// repair waves over topological levels
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_repair_level(int32_t *__restrict__ assign, int B,
                                                      const BlockRow *__restrict__ rows,
                                                      const int32_t *__restrict__ adj,
                                                      const int32_t *__restrict__ level_blocks, int lstart,
                                                      int lcount, int mode, uint8_t *__restrict__ unmined) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= lcount) return;
    const int p = blockIdx.y;
    int32_t *a = assign + (size_t)p * B;
    const int b = __ldg(level_blocks + lstart + k);
    const int t = a[b];
    if (t < 0) return;
    const BlockRow r = rows[b];
    const int npred = r.cnt & 0xffff;
    if (mode == PP_REPAIR_PUSH_FORWARD) {
        int t_min = 0;
        bool ok = true;
        for (int e = 0; e < npred; e++) {
            int tp = a[__ldg(adj + r.adj + e)];
            if (tp < 0) {
                ok = false;
                break;
            }
            t_min = max(t_min, tp);
        }
        if (!ok) a[b] = -1;
        else if (t < t_min) a[b] = t_min;
    } else {
        bool bad = false;
        for (int e = 0; e < npred; e++) {
            int tp = a[__ldg(adj + r.adj + e)];
            if (tp < 0 || tp > t) bad = true;
        }
        if (bad) {
            a[b] = -1;
            if (unmined) unmined[(size_t)p * B + b] = 1;
        }
    }
}

// ------------------------------------------------------------------------------------
// table preparation kernels
// ------------------------------------------------------------------------------------
__global__ void k_spatial(BlockRow *rows, int B, const double *alt, const double *strc, const double *dist,
                          double w1, double w2, double w3, double diameter) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    // geological_consistency (uncertainty.py:185-191)
    double dn = 0.0;
    if (diameter > 0) {
        dn = f64_div(dist[b], diameter);
        if (1.0 < dn) dn = 1.0;
    }
    double raw = f64_add(f64_add(f64_mul(w1, alt[b]), f64_mul(w2, strc[b])), f64_mul(w3, f64_sub(1.0, dn)));
    double v = f64_add(0.5, raw);
    if (v < 0.5) v = 0.5;
    if (v > 1.5) v = 1.5;
    rows[b].spatial = v;
}

// vmax [S][B] -> [B][Sp] and unit_mean[b] = (sum_s vmax[s][b]) / S sequentially (evaluate.py:302)
__global__ void k_scen_tables(const double *__restrict__ vsb, int S, int B, int Sp, double *__restrict__ vbs,
                              double *__restrict__ unit_mean) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    double acc = 0.0;
    for (int s = 0; s < S; s++) {
        double v = vsb[(size_t)s * B + b];
        vbs[(size_t)b * Sp + s] = v;
        acc = f64_add(acc, v);
    }
    for (int s = S; s < Sp; s++) vbs[(size_t)b * Sp + s] = 0.0;
    unit_mean[b] = f64_div(acc, (double)S);
}

// Scenario values straight from grades[S][B] (scenario_mode_values, evaluate.py:116-124):
//   v[s][b][o] = ((grade * mass) * price) * recovery[o % nrec] - mass * proc_cost[o % ncost]
// (numpy's left-to-right evaluation), vmax = max over modes, written block-major [B][Sp] with the
// sequential scenario mean unit_mean[b] (evaluate.py:302).  One thread per block; the grade reads
// g[s][b] are coalesced across the warp for every s.
__global__ void k_scen_from_grades(const double *__restrict__ g, int S, int B, int Sp, const double *__restrict__ mass,
                                   double price, const double *__restrict__ rec, int nrec,
                                   const double *__restrict__ pcost, int ncost, int nmodes,
                                   double *__restrict__ vbs, double *__restrict__ unit_mean) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const double m = __ldg(mass + b);
    double acc = 0.0;
    for (int s = 0; s < S; s++) {
        const double gm = f64_mul(f64_mul(__ldg(g + (size_t)s * B + b), m), price);
        double v = 0.0;
        for (int o = 0; o < nmodes; o++) {
            const double vo = f64_sub(f64_mul(gm, __ldg(rec + o % nrec)), f64_mul(m, __ldg(pcost + o % ncost)));
            v = (o == 0 || vo > v || vo != vo) ? vo : v;  // np.max over the mode axis (NaN propagates)
        }
        vbs[(size_t)b * Sp + s] = v;
        acc = f64_add(acc, v);
    }
    for (int s = S; s < Sp; s++) vbs[(size_t)b * Sp + s] = 0.0;
    unit_mean[b] = f64_div(acc, (double)S);
}

// block-major vmax [B][Sp] back to the reference layout [S][B]
__global__ void k_scen_to_sb(const double *__restrict__ vbs, int S, int B, int Sp, double *__restrict__ out) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)S * B) return;
    const int s = (int)(i / B), b = (int)(i % B);
    out[i] = vbs[(size_t)b * Sp + s];
}

// sigma.mean(axis=0) sequentially over s (evaluate.py:351)
__global__ void k_sig_mean(const double *sigma, int S, int T, double *out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    double acc = 0.0;
    for (int s = 0; s < S; s++) acc = f64_add(acc, sigma[(size_t)s * T + t]);
    out[t] = f64_div(acc, (double)S);
}

// Linear ENPV table enpv[b][t]: colgen.py:187-204 form
//   disc[t] * mean_s(sig[s][t] * vmax[s][b]) - disc[t] * cost[b][t]
// or, with `factored`, the hybrid.py:673-678 / saa.py:65-69 form
//   disc[t] * (mean_s(sig[s][t] * vmax[s][b]) - cost[b][t]);
// mean_s is numpy's .mean(axis=0) over an [S][B] array: sequential in s, then / S.
__global__ void k_enpv_table(const double *__restrict__ vmax, int Sp, int S, int B, int T,
                             const double *__restrict__ sigma, const double *__restrict__ disc,
                             const double *__restrict__ cost, int factored, double *__restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B * T) return;
    const int b = i / T, t = i - b * T;
    const double *row = vmax + (size_t)b * Sp;
    double acc = 0.0;
    for (int s = 0; s < S; s++) acc = f64_add(acc, f64_mul(__ldg(sigma + (size_t)s * T + t), __ldg(row + s)));
    const double mean = f64_div(acc, (double)S);
    const double d = __ldg(disc + t), c = __ldg(cost + (size_t)b * T + t);
    out[i] = factored ? f64_mul(d, f64_sub(mean, c)) : f64_sub(f64_mul(d, mean), f64_mul(d, c));
}

// deterministic reduce of per-shard bests (block < 0 = none), evaluate.py:404-409 order
__global__ void k_reduce_best(const pp_best *__restrict__ recs, int n, pp_best *__restrict__ out) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    Best x{-kInf, INT_MAX, INT_MAX};
    for (int i = 0; i < n; i++) {
        pp_best r = recs[i];
        if (r.block < 0) continue;
        Best o{r.value, r.block, r.period};
        if (better(o, x)) x = o;
    }
    pp_best g;
    bool none = (x.b == INT_MAX);
    g.value = none ? -kInf : x.v;
    g.block = none ? -1 : x.b;
    g.period = none ? -1 : x.t;
    *out = g;
}

__global__ void k_apply_moves(int32_t *assign, int B, int T, const int32_t *blocks, const int32_t *periods, int n) {
    // sequential in input order so a block moved twice ends at its last period
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    for (int k = 0; k < n; k++) {
        int b = blocks[k], t = periods[k];
        if (b >= 0 && b < B && t >= -1 && t < T) assign[b] = t;
    }
}


// period masses of P schedules (device pointers) into pm_out[P][T]: P1 (chunks) then
// P2 (trees), P2 launched as a programmatic dependent of P1
// ---------------------------------------------------------------------------------------------
// Cluster fast path (T <= 32, B <= 245,760): one cluster of R = 16 CTAs per schedule (8 when the
// GPU cannot place a 16-CTA cluster), 1024 threads per CTA.
//  1. Warp w of CTA r owns the contiguous blocks [(32 r + w) * 32K, +32K), K blocks per lane.  A
//     block's rank inside its (warp, period) group is the running count of that period plus the
//     lower lanes of the same match_any group.  Per-warp counts are scanned over the warps; the
//     CTA totals are exchanged through distributed shared memory (R x T integers), which fixes
//     every block's position in its period's numpy order.  Up to K = 8 the periods and masses
//     stay in registers between ranking and scatter; above that (C4: 200k blocks, K = 13) a first
//     pass only counts and the scatter pass re-reads the blocks (L2) and ranks them again.
//  2. Push mode (every period fits its slot): each mass goes straight into the shared memory of
//     the CTA that reduces its period (period t -> CTA t % R, slot t / R); otherwise into
//     compact[p][t][pos] in global memory.  A cluster barrier orders the stores.
//  3. CTA r reduces periods r, r + R, ...  numpy's recursion (pairwise.c: blocks of 8, leaves of
//     <= 128 elements) splits m = n/8 blocks floor|ceil, so the rightmost node is the largest at
//     every depth and every leaf sits at depth D or D + 1, D = (first depth whose rightmost node
//     is a leaf) - 1.  Sixteen lanes per depth-D node walk its root path to find its range and
//     sum its one or two leaves; the 2^D node values fold as a perfect tree.
// ---------------------------------------------------------------------------------------------
constexpr int PMC_R = 8;    // portable cluster size (fallback)
constexpr int PMC_R16 = 16;  // non-portable: used when the GPU can place a 16-CTA cluster
constexpr int PMC_THREADS = 1024;
constexpr int PMC_WARPS = PMC_THREADS / 32;
constexpr int PMC_MAXT = 32;
constexpr int PMC_MAXQ = (PMC_MAXT + PMC_R - 1) / PMC_R;  // periods per CTA
constexpr int PMC_MAXNODE = 1024;  // 2^D <= n / 240: periods of up to 245,760 blocks (global mode)
constexpr int PMC_PUSHNODE = 128;  // push mode: n <= own_cap < 30,720
constexpr int PMC_MAXN = 245760;
constexpr int PMC_FOLD = 512;      // node values one warp folds (16 per lane)
constexpr int PMC_KREG = 8;        // blocks per lane kept in registers
constexpr int PMC_GRP = 8;         // loads in flight per lane in the two-pass mode
constexpr size_t PMC_SMEM_MAX = 227 * 1024;
static_assert(PMC_MAXNODE <= 2 * PMC_FOLD, "one pre-fold level");

struct PmcSmem {
    int cnt[PMC_WARPS][PMC_MAXT];
    int tot[PMC_MAXT];  // this CTA's count per period (read by the cluster)
    int off[PMC_MAXT];  // this CTA's first position per period
    int n[PMC_MAXT];
    double val[PMC_MAXQ][PMC_PUSHNODE];  // node values in push mode (global mode: the slot area)
};

// the lanes of the warp holding the same period (six ballots over the bits measured slower)
__device__ __forceinline__ unsigned match_period(int t) { return __match_any_sync(0xffffffffu, t); }

__device__ __forceinline__ void cluster_sync_acqrel() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ int ld_dsmem_i32(const int *p, int rank) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
    uint32_t ra;
    int v;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(ra));
    return v;
}

__device__ __forceinline__ void st_dsmem_f64(double *p, int rank, double v) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}

// range [start, start + len) in 8-element blocks of node i at depth d of a tree over m blocks
__device__ __forceinline__ void pw_node(int m, int d, int i, int &start, int &len) {
    int s = 0, l = m;
    for (int k = d - 1; k >= 0; k--) {
        const int h = l >> 1;
        if ((i >> k) & 1) {
            s += h;
            l -= h;
        } else {
            l = h;
        }
    }
    start = s;
    len = l;
}

// K > 0: K blocks per lane in registers; K == 0: kk blocks per lane, count pass + scatter pass
template <int K, int R>  // R CTAs per schedule, one cluster (launch attribute)
__global__ void __launch_bounds__(PMC_THREADS, 1)
    k_pm_cluster(const int32_t *__restrict__ assign, const double *__restrict__ mass, int B, int T, int kk,
                 int own_cap, double *__restrict__ compact, double *__restrict__ pm_out, EvalInit init,
                 int32_t *__restrict__ bad) {
    __shared__ PmcSmem h;
    extern __shared__ __align__(16) double pmc_own[];  // [ceil(T / R)][own_cap] (push mode)
    PMCP(0, 0);
    if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) {  // complete before the dependents' wait
        if (init.n_pairs) *init.n_pairs = 0;
        if (init.best) *init.best = pp_best{-kInf, -1, -1};
        if (init.bad_cand) *init.bad_cand = 0;
    }
    asm volatile("griddepcontrol.launch_dependents;");
    constexpr unsigned FULL = 0xffffffffu;
    constexpr bool REG = K > 0 && K <= PMC_KREG;  // periods, masses and ranks in registers
    constexpr bool PACK = K > PMC_KREG;            // ranks packed 2 per register, blocks re-read
    constexpr int KR = REG ? K : 1;
    static_assert(K <= 2 * PMC_GRP, "packed ranks cover two load groups");
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r = blockIdx.x, p = blockIdx.y;
    const int32_t *as = assign + (size_t)p * B;
    const int KB = REG ? K : kk;
    const int base = (r * PMC_WARPS + warp) * (32 * KB);
    const unsigned lt = (1u << lane) - 1u;
    int tk[KR];
    double mk[KR];
    int pos[KR];
    int badl = 0;
    unsigned pk[PMC_GRP] = {};  // PACK: rank of block k in bits 16 (k & 1) of pk[k >> 1]
    if constexpr (REG) {
#pragma unroll
        for (int k = 0; k < K; k++) {
            const int b = base + k * 32 + lane;
            int t = -1;
            double m = 0.0;
            if (b < B) {
                t = __ldg(as + b);
                m = __ldg(mass + b);
            }
            tk[k] = ((unsigned)t < (unsigned)T) ? t : -1;
            badl |= (t < -1) | (t >= T);
            mk[k] = m;
        }
    }
    PMCS(0);
    for (int i = tid; i < PMC_WARPS * PMC_MAXT; i += PMC_THREADS) (&h.cnt[0][0])[i] = 0;
    __syncthreads();
    if constexpr (REG) {  // ranks inside (warp, period): match_any groups, running counts in shared memory
#pragma unroll
        for (int k = 0; k < K; k++) {
            const unsigned mt = match_period(tk[k]);
            const int lr = __popc(mt & lt);
            const int b0 = tk[k] >= 0 ? h.cnt[warp][tk[k]] : 0;
            pos[k] = b0 + lr;
            __syncwarp();
            if (tk[k] >= 0 && lr == 0) h.cnt[warp][tk[k]] = b0 + __popc(mt);
            __syncwarp();
        }
    } else if constexpr (PACK) {  // the same ranks, PMC_GRP loads in flight per lane, kept packed
#pragma unroll
        for (int k0 = 0; k0 < 2 * PMC_GRP; k0 += PMC_GRP) {
            if (k0 >= kk) break;
            int tq[PMC_GRP];
#pragma unroll
            for (int u = 0; u < PMC_GRP; u++) {
                const int b = base + (k0 + u) * 32 + lane;
                tq[u] = (k0 + u < kk && b < B) ? __ldg(as + b) : -1;
            }
#pragma unroll
            for (int u = 0; u < PMC_GRP; u++) {
                const int t = tq[u];
                badl |= (t < -1) | (t >= T);
                const int tv = ((unsigned)t < (unsigned)T) ? t : -1;
                const unsigned mt = match_period(tv);
                const int lr = __popc(mt & lt);
                const int b0 = tv >= 0 ? h.cnt[warp][tv] : 0;
                __syncwarp();
                if (tv >= 0 && lr == 0) h.cnt[warp][tv] = b0 + __popc(mt);
                __syncwarp();
                pk[(k0 + u) >> 1] |= (unsigned)(b0 + lr) << (16 * ((k0 + u) & 1));
            }
        }
    } else {  // count pass: PMC_GRP loads in flight per lane
        for (int k0 = 0; k0 < kk; k0 += PMC_GRP) {
            int tq[PMC_GRP];
#pragma unroll
            for (int u = 0; u < PMC_GRP; u++) {
                const int b = base + (k0 + u) * 32 + lane;
                tq[u] = (k0 + u < kk && b < B) ? __ldg(as + b) : -1;
            }
#pragma unroll
            for (int u = 0; u < PMC_GRP; u++) {
                const int t = tq[u];
                badl |= (t < -1) | (t >= T);
                const int tv = ((unsigned)t < (unsigned)T) ? t : -1;
                const unsigned mt = match_period(tv);
                if (tv >= 0 && __popc(mt & lt) == 0) h.cnt[warp][tv] += __popc(mt);
                __syncwarp();
            }
        }
    }
    const int anybad = __syncthreads_or(badl);  // (also the barrier after the ranks)
    if (bad && threadIdx.x == 0 && blockIdx.y == 0) bad[blockIdx.x] = anybad;  // every CTA writes its flag
    // per-period exclusive scan over the warps (warp j scans period j)
    if (warp < T) {
        const int v = h.cnt[lane][warp];
        int inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += y;
        }
        h.cnt[lane][warp] = inc - v;
        if (lane == 31) h.tot[warp] = inc;
    }
    cluster_sync_acqrel();  // totals published
    PMCS(1);
    if (warp < T) {  // cross-CTA scan of the totals through distributed shared memory
        const int v = lane < R ? ld_dsmem_i32(&h.tot[warp], lane) : 0;
        int inc = v;
#pragma unroll
        for (int o = 1; o < R; o <<= 1) {
            const int y = __shfl_up_sync(FULL, inc, o);
            if (lane >= o) inc += y;
        }
        const int off = __shfl_sync(FULL, inc - v, r);
        const int n = __shfl_sync(FULL, inc, R - 1);
        if (lane == 0) {
            h.off[warp] = off;
            h.n[warp] = n;
        }
    }
    __syncthreads();
    PMCS(2);
    // push mode (every period fits its slot; the same decision in every CTA): each mass goes
    // straight into the shared memory of the CTA that reduces its period; otherwise through L2
    bool push = true;
    for (int t = 0; t < T; t++) push &= h.n[t] <= own_cap;
    if constexpr (REG) {
#pragma unroll
        for (int k = 0; k < K; k++)
            if (tk[k] >= 0) {
                const int t = tk[k], at = h.off[t] + h.cnt[warp][t] + pos[k];
                PP_DCHECK(at >= 0 && at < h.n[t] && (!push || at < own_cap));
                if (push) st_dsmem_f64(pmc_own + (t / R) * own_cap + at, t % R, mk[k]);
                else compact[((size_t)p * T + t) * B + at] = mk[k];
            }
    } else if constexpr (PACK) {  // scatter pass: re-read the blocks (L2), ranks from the first pass
#pragma unroll
        for (int k0 = 0; k0 < 2 * PMC_GRP; k0 += PMC_GRP) {
            if (k0 >= kk) break;
            int tq[PMC_GRP];
            double mq[PMC_GRP];
#pragma unroll
            for (int u = 0; u < PMC_GRP; u++) {
                const int b = base + (k0 + u) * 32 + lane;
                const bool in = k0 + u < kk && b < B;
                const int t = in ? __ldg(as + b) : -1;
                tq[u] = ((unsigned)t < (unsigned)T) ? t : -1;
                mq[u] = in ? __ldg(mass + b) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < PMC_GRP; u++) {
                const int t = tq[u];
                if (t >= 0) {
                    const int at = h.off[t] + h.cnt[warp][t] + (int)((pk[(k0 + u) >> 1] >> (16 * ((k0 + u) & 1))) & 0xffffu);
                    PP_DCHECK(at >= 0 && at < h.n[t] && (!push || at < own_cap));
                    if (push) st_dsmem_f64(pmc_own + (t / R) * own_cap + at, t % R, mq[u]);
                    else compact[((size_t)p * T + t) * B + at] = mq[u];
                }
            }
        }
    } else {  // scatter pass: re-read, rank again (same groups), h.cnt[warp][t] is the running position
        for (int k0 = 0; k0 < kk; k0 += PMC_GRP) {
            int tq[PMC_GRP];
            double mq[PMC_GRP];
#pragma unroll
            for (int u = 0; u < PMC_GRP; u++) {
                const int b = base + (k0 + u) * 32 + lane;
                const bool in = k0 + u < kk && b < B;
                const int t = in ? __ldg(as + b) : -1;
                tq[u] = ((unsigned)t < (unsigned)T) ? t : -1;
                mq[u] = in ? __ldg(mass + b) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < PMC_GRP; u++) {
                const int t = tq[u];
                const unsigned mt = match_period(t);
                const int lr = __popc(mt & lt);
                const int w0 = t >= 0 ? h.cnt[warp][t] : 0;
                __syncwarp();
                if (t >= 0) {
                    const int at = h.off[t] + w0 + lr;
                    PP_DCHECK(at >= 0 && at < h.n[t] && (!push || at < own_cap));
                    if (push) st_dsmem_f64(pmc_own + (t / R) * own_cap + at, t % R, mq[u]);
                    else compact[((size_t)p * T + t) * B + at] = mq[u];
                    if (lr == 0) h.cnt[warp][t] = w0 + __popc(mt);
                }
                __syncwarp();
            }
        }
    }
    // the cluster barrier's release/acquire orders these stores (distributed shared memory or
    // global) for every thread of the cluster (no separate sequentially consistent fence)
    cluster_sync_acqrel();  // every block of the schedule is in place (remote totals no longer read)
    PMCP(0, 1);
    // depth-D nodes of this CTA's periods r, r + R, ...
    const int q = max(0, (T - r + R - 1) / R);
    int Dg[PMC_MAXQ], cntg[PMC_MAXQ];
    int nitems = 0;
#pragma unroll
    for (int g = 0; g < PMC_MAXQ; g++) {
        Dg[g] = 0;
        cntg[g] = 0;
        if (g < q) {
            // d = first depth whose rightmost node is a leaf: 8 ceil(m / 2^d) + rem <= 128, i.e.
            // 2^d >= ceil(m / thr) with thr = 16 when rem = 0, else 15
            const int n = h.n[r + R * g], m = n >> 3, rem = n & 7;
            const int thr = rem ? 15 : 16, qd = (m + thr - 1) / thr;
            const int d = qd <= 1 ? 0 : 32 - __clz(qd - 1);
            Dg[g] = max(d - 1, 0);
            cntg[g] = 1 << Dg[g];
        }
        nitems += cntg[g];
    }
    // node values: push mode in h.val; global mode in the (then unused) slot area, own_cap apart
    double *const nodes = push ? &h.val[0][0] : pmc_own;
    const int nstride = push ? PMC_PUSHNODE : own_cap;
    PMCS(4);
    const int sub = tid & 7, half = (tid >> 3) & 1;  // 16 lanes per node: half c sums child leaf c
    for (int it0 = 0; it0 < nitems; it0 += PMC_THREADS / 16) {
        const int it = it0 + (tid >> 4);
        if (it0 + 2 * warp >= nitems) continue;  // warp-uniform: this warp's two nodes are past the end
        const bool act = it < nitems;
        int g = 0, i = act ? it : 0, D = Dg[0];  // (unrolled selects: no local-memory indexing)
        bool fnd = false;
#pragma unroll
        for (int u = 0; u < PMC_MAXQ; u++)
            if (!fnd) {
                if (i < cntg[u] || u == PMC_MAXQ - 1) {
                    g = u;
                    D = Dg[u];
                    fnd = true;
                } else {
                    i -= cntg[u];
                }
            }
        const int t = r + R * g;
        const int n = act ? h.n[t] : 0, m = n >> 3, rem = n & 7;
        // half c walks to child 2i + c at depth D + 1; the node is the union of the two halves
        int s1, l1;
        pw_node(m, D + 1, 2 * i + half, s1, l1);
        const int s_sib = __shfl_xor_sync(FULL, s1, 8), l_sib = __shfl_xor_sync(FULL, l1, 8);
        const int s0 = half ? s_sib : s1, l0 = l1 + l_sib;
        const bool last = i == (1 << D) - 1;
        const int L = 8 * l0 + (last ? rem : 0);
        const bool split = L > 128;  // a node of depth D is one leaf or two
        int o = 8 * s0, len = L;
        if (split) {
            o = 8 * s1;
            len = 8 * l1 + ((last && half == 1) ? rem : 0);
        }
        const bool use = act && (split || half == 0);
        if (it0 == 0) PMCS(6);
        // every load of the leaf in flight: 16 accumulator elements per lane + one tail element
        // (separate shared / global paths: a pointer that may be either compiles to slow generic loads)
        const int nm = len >> 3, ntail = len & 7, e0 = len - ntail;
        double x[16], tailv;
        if (push) {
            const double *a = pmc_own + g * own_cap + o;
#pragma unroll
            for (int u = 0; u < 16; u++) x[u] = (use && u < nm) ? a[8 * u + sub] : 0.0;
            tailv = (use && sub < ntail) ? a[e0 + sub] : 0.0;
        } else {
            const double *a = compact + ((size_t)p * T + t) * B + o;
#pragma unroll
            for (int u = 0; u < 16; u++) x[u] = (use && u < nm) ? __ldcg(a + 8 * u + sub) : 0.0;
            tailv = (use && sub < ntail) ? __ldcg(a + e0 + sub) : 0.0;
        }
        double acc = x[0];
#pragma unroll
        for (int u = 1; u < 16; u++)
            if (u < nm) acc = f64_add(acc, x[u]);
        if (it0 == 0) PMCS(7);
        acc = f64_add(acc, __shfl_xor_sync(FULL, acc, 1));
        acc = f64_add(acc, __shfl_xor_sync(FULL, acc, 2));
        acc = f64_add(acc, __shfl_xor_sync(FULL, acc, 4));
        double res = len < 8 ? -0.0 : acc;
        const int lbase = lane & ~7;
        for (int e = 0; e < 7; e++) {  // uniform trip count (shuffles)
            const double y = __shfl_sync(FULL, tailv, lbase + e);
            if (e < ntail) res = f64_add(res, y);
        }
        if (it0 == 0) PMCS(8);
        const double other = __shfl_xor_sync(FULL, res, 8);  // the sibling leaf
        PP_DCHECK(!use || (i < nstride && o + len <= n && (!push || o + len <= own_cap)));
        if (use && sub == 0 && half == 0) nodes[g * nstride + i] = split ? f64_add(res, other) : res;
    }
    PMCS(5);
    __syncthreads();
    // periods above ~123k blocks have more than PMC_FOLD depth-D nodes: fold one level first
    // (pairs (2i, 2i + 1) are the perfect tree's lowest level)
    {
        double y[PMC_MAXQ];
#pragma unroll
        for (int g = 0; g < PMC_MAXQ; g++)
            y[g] = (cntg[g] > PMC_FOLD && tid < cntg[g] / 2)
                       ? f64_add(nodes[g * nstride + 2 * tid], nodes[g * nstride + 2 * tid + 1])
                       : 0.0;
        bool any = false;
#pragma unroll
        for (int g = 0; g < PMC_MAXQ; g++) any |= cntg[g] > PMC_FOLD;
        if (any) {  // uniform over the CTA
            __syncthreads();
#pragma unroll
            for (int g = 0; g < PMC_MAXQ; g++)
                if (cntg[g] > PMC_FOLD && tid < cntg[g] / 2) nodes[g * nstride + tid] = y[g];
            __syncthreads();
#pragma unroll
            for (int g = 0; g < PMC_MAXQ; g++)
                if (cntg[g] > PMC_FOLD) cntg[g] >>= 1;
        }
    }
    PMCS(3);
    // perfect-tree fold of the node values: warp g folds period slot g
    if (warp < q) {
        int cnt = cntg[0];
#pragma unroll
        for (int g = 1; g < PMC_MAXQ; g++)
            if (warp == g) cnt = cntg[g];
        const int g = warp;
        const int per = cnt > 32 ? cnt >> 5 : 1;  // consecutive values per lane (<= 16)
        double v = 0.0;
        if (lane * per < cnt) {
            double x[16];
#pragma unroll
            for (int u = 0; u < 16; u++) x[u] = (u < per) ? nodes[g * nstride + lane * per + u] : 0.0;
#pragma unroll
            for (int w = 1; w < 16; w <<= 1)
#pragma unroll
                for (int u = 0; u < 16; u += 2 * w)
                    if (u + w < per) x[u] = f64_add(x[u], x[u + w]);
            v = x[0];
        }
        const int lanes = cnt > 32 ? 32 : cnt;
        for (int o = 1; o < lanes; o <<= 1) v = f64_add(v, __shfl_xor_sync(FULL, v, o));
        if (lane == 0) {
            const int t = r + R * g;
            pm_out[(size_t)p * T + t] = f64_add(0.0, h.n[t] ? v : -0.0);
        }
    }
    PMCP(1, 1);
}

// dynamic shared memory of the push-mode slots: ceil(T / R) slots of own_cap doubles, each sized
// for twice the mean period (periods beyond it take the global path), within the 227 KB opt-in
static void pm_cluster_slots(int B, int T, int R, int *own_cap, size_t *smem) {
    const int q = (T + R - 1) / R;
    const size_t avail = PMC_SMEM_MAX - sizeof(PmcSmem) - 1024;
    const size_t want = std::min<size_t>(30720, std::max<size_t>(6144, 2 * (((size_t)B + T - 1) / T)));  // PMC_PUSHNODE
    const size_t cap = std::min(avail / (8 * (size_t)q), want);
    *own_cap = (int)cap;
    *smem = 8 * (size_t)q * cap;
}

template <int K, int R>
static int launch_pm_cluster_r(pp_ctx *c, const int32_t *d_assign, int np, double *d_pm, cudaStream_t st,
                               const EvalInit *init, int32_t *bad, int kk) {
    const EvalInit in = init ? *init : EvalInit{nullptr, nullptr, nullptr};
    int own_cap;
    size_t smem;
    pm_cluster_slots(c->B, c->T, R, &own_cap, &smem);
    TRY(ensure_max_smem(k_pm_cluster<K, R>, smem, c->device));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(R, np);
    cfg.blockDim = dim3(PMC_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = R;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k_pm_cluster<K, R>, d_assign, (const double *)c->mass.as<double>(),
                                             c->B, c->T, kk, own_cap, c->compact.as<double>(), d_pm, in, bad);
    if (e != cudaSuccess) return fail(PP_ERR_CUDA, "k_pm_cluster launch: %s", cudaGetErrorString(e));
    return PP_OK;
}

// 16-CTA clusters halve each CTA's share of the blocks (the kernel is latency-bound on 8 SMs);
// they need the non-portable opt-in and a GPC with 16 free SMs, probed once per device
template <int K>
static bool pm_r16_attr() {
    return cudaFuncSetAttribute(k_pm_cluster<K, PMC_R16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
           cudaSuccess;
}
static bool pm_use_r16(int device) {
    static int cached[64];  // 0 unknown, 1 yes, 2 no
    if (device < 0 || device >= 64) return false;
    if (!cached[device]) {
        bool ok = pm_r16_attr<0>() && pm_r16_attr<2 * PMC_GRP>() && pm_r16_attr<1>() && pm_r16_attr<2>() && pm_r16_attr<4>() && pm_r16_attr<8>();
        if (ok) {
            const size_t smem = PMC_SMEM_MAX - sizeof(PmcSmem) - 1024;  // the largest launch
            cudaFuncSetAttribute(k_pm_cluster<0, PMC_R16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(PMC_R16);
            cfg.blockDim = dim3(PMC_THREADS);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = PMC_R16;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            int n = 0;
            ok = cudaOccupancyMaxActiveClusters(&n, k_pm_cluster<0, PMC_R16>, &cfg) == cudaSuccess && n >= 1;
        }
        cudaGetLastError();
        cached[device] = ok ? 1 : 2;
    }
    return cached[device] == 1;
}

template <int R>
static int launch_pm_cluster(pp_ctx *c, const int32_t *d_assign, int np, double *d_pm, cudaStream_t st,
                             const EvalInit *init, int32_t *bad) {
    const int per_lane = (c->B + R * PMC_THREADS - 1) / (R * PMC_THREADS);  // blocks per lane
    if (per_lane <= 1) return launch_pm_cluster_r<1, R>(c, d_assign, np, d_pm, st, init, bad, 1);
    if (per_lane <= 2) return launch_pm_cluster_r<2, R>(c, d_assign, np, d_pm, st, init, bad, 2);
    if (per_lane <= 4) return launch_pm_cluster_r<4, R>(c, d_assign, np, d_pm, st, init, bad, 4);
    if (per_lane <= PMC_KREG) return launch_pm_cluster_r<8, R>(c, d_assign, np, d_pm, st, init, bad, 8);
    if (per_lane <= 2 * PMC_GRP) return launch_pm_cluster_r<2 * PMC_GRP, R>(c, d_assign, np, d_pm, st, init, bad, per_lane);
    return launch_pm_cluster_r<0, R>(c, d_assign, np, d_pm, st, init, bad, per_lane);
}

int run_period_mass(pp_ctx *c, const int32_t *d_assign, int P, double *d_pm, cudaStream_t st, const EvalInit *init) {
    const int B = c->B, T = c->T;
    const int nchunk = (B + PM_CH - 1) / PM_CH;
    // compacted masses: B doubles per (period, schedule); batches bounded to ~512 MiB
    const size_t per = (size_t)T * B * sizeof(double);
    const int pchunk = std::max(1, std::min(P, (int)std::max<size_t>(1, ((size_t)512 << 20) / per)));
    TRY(c->compact.ensure(per * pchunk));
    TRY(c->cnt.ensure(sizeof(int32_t) * (size_t)pchunk * nchunk * (T + 1)));
    const size_t nflags = (size_t)pchunk * nchunk + 2 * (size_t)pchunk;
    if (c->pm_flags_n < nflags) {
        TRY(c->pm_flags.ensure(sizeof(int32_t) * nflags));
        CUDA_TRY(dev_zero(c, c->pm_flags.ptr, sizeof(int32_t) * nflags));
        c->pm_flags_n = nflags;
    }
    if (pm_cluster_path(c)) {
        const bool r16 = pm_use_r16(c->device);
        for (int p0 = 0; p0 < P; p0 += pchunk) {
            const int np = std::min(pchunk, P - p0);
            const int32_t *a = d_assign + (size_t)p0 * B;
            double *o = d_pm + (size_t)p0 * T;
            const EvalInit *z = p0 == 0 ? init : nullptr;
            int32_t *bad = (P == 1 && d_assign == c->assign_ptr && c->bad_pending) ? c->pm_bad.as<int32_t>() : nullptr;
            if (r16) TRY(launch_pm_cluster<PMC_R16>(c, a, np, o, st, z, bad));
            else TRY(launch_pm_cluster<PMC_R>(c, a, np, o, st, z, bad));
        }
        return PP_OK;
    }
    if (init) TRY(init_eval_outputs(c, *init, st));
    const size_t smem = std::max(sizeof(PmTreeSmem), sizeof(int) * ((PM_THREADS / 32) * PM_MAXT + PM_MAXT));
    TRY(ensure_max_smem(k_period_mass, smem, c->device));
    int32_t *flags = c->pm_flags.as<int32_t>();
    unsigned int *done = reinterpret_cast<unsigned int *>(flags + (size_t)pchunk * nchunk);
    for (int p0 = 0; p0 < P; p0 += pchunk) {
        const int np = std::min(pchunk, P - p0);
        k_period_mass<<<dim3(nchunk + T, np), PM_THREADS, smem, st>>>(d_assign + (size_t)p0 * B, c->mass.as<double>(), B,
                                                                       T, nchunk, c->cnt.as<int32_t>(), flags, done,
                                                                       c->compact.as<double>(), d_pm + (size_t)p0 * T);
        CUDA_TRY(cudaGetLastError());
    }
    return PP_OK;
}

// recompute the current schedule's period masses if the schedule changed
bool pm_cluster_path(const pp_ctx *c) {
    static const bool off = getenv("PP_PM_NOCLUSTER") != nullptr;  // A/B timing of the chunk + tree kernel
    return c->T <= PMC_MAXT && c->B <= PMC_MAXN && !off;
}

int check_schedule_range(pp_ctx *c, bool copied) {
    if (!c->bad_pending || c->pm_dirty) return PP_OK;  // not range-checked yet
    c->bad_pending = false;
    if (!copied) CUDA_TRY(cudaMemcpy(c->h_bad, c->pm_bad.ptr, sizeof(int32_t) * PMC_R16, cudaMemcpyDeviceToHost));
    for (int r = 0; r < PMC_R16; r++)
        if (c->h_bad[r]) {
            c->have_sched = false;  // unusable until the next pp_set_schedule
            return fail(PP_ERR_INVALID_ARGS, "schedule has period indices out of range");
        }
    return PP_OK;
}

// the per-launch output state of an evaluation when no period-mass kernel precedes it: one tiny
// kernel (graph-capturable, no host staging) instead of memsets and a copy
__global__ void k_init_eval(int32_t *n_pairs, int32_t *bad_cand, pp_best *best) {
    asm volatile("griddepcontrol.launch_dependents;");
    if (threadIdx.x != 0) return;
    if (n_pairs) *n_pairs = 0;
    if (bad_cand) *bad_cand = 0;
    if (best) {
        best->value = -kInf;
        best->block = -1;
        best->period = -1;
    }
}

int init_eval_outputs(pp_ctx *c, const EvalInit &init, cudaStream_t st) {
    (void)c;
    if (!init.n_pairs && !init.bad_cand && !init.best) return PP_OK;
    k_init_eval<<<1, 32, 0, st>>>(init.n_pairs, init.bad_cand, init.best);
    CUDA_TRY(cudaGetLastError());
    return PP_OK;
}

int refresh_pm(pp_ctx *c, cudaStream_t st, bool *launched, const EvalInit *init) {
    *launched = false;
    if (!c->pm_dirty) {
        if (init) {
            TRY(init_eval_outputs(c, *init, st));
            // the evaluation may start under PDL: it touches the initialised state only after its
            // griddepcontrol.wait -- except the host-mode bad-candidate flag (set before the wait)
            *launched = !init->bad_cand && (init->n_pairs || init->best);
        }
        return PP_OK;
    }
    TRY(run_period_mass(c, c->assign_ptr, 1, c->pm.as<double>(), st, init));
    c->pm_dirty = false;
    *launched = true;
    return PP_OK;
}


static void plan_rec(PwPlan &p, int o, int n) {
    if (n <= 128) {
        p.start[p.nleaf] = o;
        p.len[p.nleaf] = n;
        p.adds[p.nleaf] = 0;
        p.nleaf++;
        return;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    plan_rec(p, o, n2);
    plan_rec(p, o + n2, n - n2);
    p.adds[p.nleaf - 1]++;
}

static int make_plan(int n, PwPlan *p) {
    // leaves hold 56..128 elements once n > 128
    if (n > 128 * (kMaxLeaves / 2)) return fail(PP_ERR_INVALID_ARGS, "too many scenarios (%d) for the pairwise plan", n);
    memset(p, 0, sizeof(*p));
    p->n = n;
    if (n > 0) plan_rec(*p, 0, n);
    return PP_OK;
}


static void plan_words(const PwPlan &p, int *w) {
    w[0] = p.n;
    w[1] = p.nleaf;
    for (int i = 0; i < kMaxLeaves; i++) {
        w[2 + i] = p.start[i];
        w[2 + kMaxLeaves + i] = p.len[i];
        w[2 + 2 * kMaxLeaves + i] = p.adds[i];
    }
}

extern "C" {

int pp_set_instance(pp_ctx *c, int32_t B, int32_t T, int64_t E, const int32_t *ei, const int32_t *ej,
                    const double *mass, const double *cost, const double *capacity, const double *discount) {
    if (!c) return fail(PP_ERR_INVALID_ARGS, "NULL context");
    if (B < 1 || T < 1) return fail(PP_ERR_INVALID_ARGS, "need n_blocks >= 1 and n_periods >= 1");
    if (T > PM_MAXT) return fail(PP_ERR_INVALID_ARGS, "n_periods %d exceeds the supported %d", T, PM_MAXT);
    if (E < 0 || (E > 0 && (!ei || !ej))) return fail(PP_ERR_INVALID_ARGS, "bad edge arrays");
    if (!mass || !cost || !capacity || !discount) return fail(PP_ERR_INVALID_ARGS, "NULL table");
    for (int64_t e = 0; e < E; e++)
        if (ei[e] < 0 || ei[e] >= B || ej[e] < 0 || ej[e] >= B)
            return fail(PP_ERR_VALIDATION, "precedence edge (%d, %d) references unknown block", ei[e], ej[e]);
    for (int t = 0; t < T; t++)
        if (!(capacity[t] > 0)) return fail(PP_ERR_VALIDATION, "mining capacity must be > 0 in every period");
    TRY(use_device(c));
    // adjacency: predecessors of b (edges (i, b) in list order) then successors (edges (b, j))
    std::vector<int> npred(B, 0), nsucc(B, 0);
    for (int64_t e = 0; e < E; e++) {
        npred[ej[e]]++;
        nsucc[ei[e]]++;
    }
    for (int b = 0; b < B; b++)
        if (npred[b] > 0xffff || nsucc[b] > 0x7fff)
            return fail(PP_ERR_INVALID_ARGS, "block %d has too many neighbours", b);
    std::vector<int> start(B + 1, 0);
    for (int b = 0; b < B; b++) start[b + 1] = start[b] + npred[b] + nsucc[b];
    std::vector<int> adj((size_t)std::max<long long>(start[B], 1));
    std::vector<int> fp(B), fs(B);
    for (int b = 0; b < B; b++) {
        fp[b] = start[b];
        fs[b] = start[b] + npred[b];
    }
    for (int64_t e = 0; e < E; e++) {
        adj[fp[ej[e]]++] = ei[e];
        adj[fs[ei[e]]++] = ej[e];
    }
    // topological levels (longest predecessor chain) by Kahn's algorithm; cycle check
    std::vector<int> indeg(npred), level(B, 0), queue;
    queue.reserve(B);
    for (int b = 0; b < B; b++)
        if (indeg[b] == 0) queue.push_back(b);
    for (size_t q = 0; q < queue.size(); q++) {
        int b = queue[q];
        for (int k = start[b] + npred[b]; k < start[b + 1]; k++) {
            int j = adj[k];
            level[j] = std::max(level[j], level[b] + 1);
            if (--indeg[j] == 0) queue.push_back(j);
        }
    }
    if ((int)queue.size() != B) return fail(PP_ERR_VALIDATION, "cycle in precedence graph");
    int nlev = 0;
    for (int b = 0; b < B; b++) nlev = std::max(nlev, level[b] + 1);
    std::vector<int> lptr(nlev + 1, 0), lblocks(B);
    for (int b = 0; b < B; b++) lptr[level[b] + 1]++;
    for (int l = 0; l < nlev; l++) lptr[l + 1] += lptr[l];
    {
        std::vector<int> fill(lptr.begin(), lptr.end() - 1);
        for (int b = 0; b < B; b++) lblocks[fill[level[b]]++] = b;
    }
    c->h_start = start;
    c->h_npred = npred;
    c->h_adj = adj;
    c->h_mass.assign(mass, mass + B);
    c->h_cap.assign(capacity, capacity + T);
    std::vector<BlockRow> rows(B);
    for (int b = 0; b < B; b++) {
        rows[b].mass = mass[b];
        rows[b].spatial = 0.0;
        rows[b].adj = start[b];
        rows[b].cnt = npred[b] | (nsucc[b] << 16);
        rows[b].level = level[b];
        rows[b].pad = 0;
    }
    TRY(c->rows.ensure(sizeof(BlockRow) * B));
    TRY(c->adj.ensure(sizeof(int) * adj.size()));
    TRY(c->cost.ensure(sizeof(double) * (size_t)B * T));
    TRY(c->cap.ensure(sizeof(double) * T));
    TRY(c->disc.ensure(sizeof(double) * T));
    TRY(c->ones_t.ensure(sizeof(double) * T));
    TRY(c->level_blocks.ensure(sizeof(int) * B));
    TRY(c->assign.ensure(sizeof(int) * B));
    TRY(c->mass.ensure(sizeof(double) * B));
    TRY(c->pm.ensure(sizeof(double) * T));
    std::vector<double> ones(T, 1.0);
    CUDA_TRY(dev_upload(c, c->rows.ptr, rows.data(), sizeof(BlockRow) * B));
    CUDA_TRY(dev_upload(c, c->adj.ptr, adj.data(), sizeof(int) * adj.size()));
    CUDA_TRY(dev_upload(c, c->cost.ptr, cost, sizeof(double) * (size_t)B * T));
    CUDA_TRY(dev_upload(c, c->mass.ptr, mass, sizeof(double) * B));
    CUDA_TRY(dev_upload(c, c->cap.ptr, capacity, sizeof(double) * T));
    CUDA_TRY(dev_upload(c, c->disc.ptr, discount, sizeof(double) * T));
    CUDA_TRY(dev_upload(c, c->ones_t.ptr, ones.data(), sizeof(double) * T));
    CUDA_TRY(dev_upload(c, c->level_blocks.ptr, lblocks.data(), sizeof(int) * B));
    c->B = B;
    c->T = T;
    c->E = E;
    c->n_levels = nlev;
    c->deg_max = 0;
    for (int b = 0; b < B; b++) c->deg_max = std::max(c->deg_max, npred[b] + nsucc[b]);
    // padded neighbour table for the warp evaluation kernel: one 128-byte row of 32 slots per
    // block, predecessors as ids, successors tagged with 1 << 30, padding -1
    c->nbr_stride = 32;
    if (c->deg_max <= 32) {
        std::vector<int> nbr((size_t)B * 32, -1);
        for (int b = 0; b < B; b++)
            for (int k = 0; k < npred[b] + nsucc[b]; k++)
                nbr[(size_t)b * 32 + k] = adj[start[b] + k] | (k < npred[b] ? 0 : (1 << 30));
        TRY(c->nbr.ensure(sizeof(int) * nbr.size()));
        CUDA_TRY(dev_upload(c, c->nbr.ptr, nbr.data(), sizeof(int) * nbr.size()));
    } else {
        c->nbr.release();
    }
    c->level_ptr = lptr;
    c->level_of = level;
    c->mean_cap = (0.0 + host_pairwise(capacity, T)) / (double)T;
    c->have_instance = true;
    c->npv_gen++;
    c->assign_ptr = c->assign.as<int32_t>();
    c->borrowed = false;
    c->pm_dirty = true;
    c->have_spatial = false;
    c->have_scen = false;
    c->have_sched = false;
    return PP_OK;
}

int pp_set_geology(pp_ctx *c, const double *alt, const double *strc, const double *dist, double w1, double w2,
                   double w3, double diameter) {
    if (!c || !c->have_instance) return fail(PP_ERR_STATE, "pp_set_instance first");
    if (!alt || !strc || !dist) return fail(PP_ERR_INVALID_ARGS, "NULL feature array");
    TRY(use_device(c));
    const int B = c->B;
    DevBuf tmp;
    int rc = tmp.ensure(sizeof(double) * 3 * (size_t)B);
    if (rc) return rc;
    double *d = tmp.as<double>();
    cudaError_t e = dev_upload(c, d, alt, sizeof(double) * B);
    if (e == cudaSuccess) e = dev_upload(c, d + B, strc, sizeof(double) * B);
    if (e == cudaSuccess) e = dev_upload(c, d + 2 * (size_t)B, dist, sizeof(double) * B);
    if (e == cudaSuccess) {
        k_spatial<<<(B + 255) / 256, 256, 0, c->stream>>>(c->rows.as<BlockRow>(), B, d, d + B, d + 2 * (size_t)B, w1,
                                                          w2, w3, diameter);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    tmp.release();
    if (e != cudaSuccess) return fail(PP_ERR_CUDA, "pp_set_geology: %s", cudaGetErrorString(e));
    c->have_spatial = true;
    return PP_OK;
}

}  // extern "C"

// common part of pp_set_scenarios / pp_set_scenarios_grades: `fill` writes c->vmax [B][Sp] and
// c->unit_mean on c->stream from host data
template <class Fill>
static int set_scenarios_common(pp_ctx *c, int32_t S, const double *sigma_st, Fill fill) {
    TRY(use_device(c));
    PwPlan plan;
    TRY(make_plan(S, &plan));
    const int B = c->B, T = c->T;
    const int Sp = (S + 3) & ~3;
    TRY(c->vmax.ensure(sizeof(double) * (size_t)B * Sp));
    TRY(c->unit_mean.ensure(sizeof(double) * B));
    TRY(c->sigma.ensure(sizeof(double) * (size_t)S * T));
    TRY(c->sigma_ts.ensure(sizeof(double) * (size_t)S * T));
    TRY(c->ones_st.ensure(sizeof(double) * (size_t)S * T));
    TRY(c->sig_mean.ensure(sizeof(double) * T));
    TRY(c->plan_dev.ensure(sizeof(int) * kPlanWords));
    cudaError_t e = fill(Sp);
    std::vector<double> ones((size_t)S * T, 1.0);
    int words[kPlanWords];
    plan_words(plan, words);
    if (e == cudaSuccess) e = dev_upload(c, c->plan_dev.ptr, words, sizeof(words));
    if (e == cudaSuccess) e = dev_upload(c, c->ones_st.ptr, ones.data(), sizeof(double) * ones.size());
    if (e == cudaSuccess && sigma_st) {
        e = dev_upload(c, c->sigma.ptr, sigma_st, sizeof(double) * (size_t)S * T);
        if (e == cudaSuccess) {
            std::vector<double> ts((size_t)S * T);
            for (int s_ = 0; s_ < S; s_++)
                for (int t = 0; t < T; t++) ts[(size_t)t * S + s_] = sigma_st[(size_t)s_ * T + t];
            e = dev_upload(c, c->sigma_ts.ptr, ts.data(), sizeof(double) * ts.size());
        }
        if (e == cudaSuccess) {
            k_sig_mean<<<(T + 127) / 128, 128, 0, c->stream>>>(c->sigma.as<double>(), S, T, c->sig_mean.as<double>());
            e = cudaGetLastError();
        }
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return fail(PP_ERR_CUDA, "pp_set_scenarios: %s", cudaGetErrorString(e));
    c->S = S;
    c->Sp = Sp;
    c->plan = plan;
    c->cvar_k = std::max(1, (int)std::ceil(0.1 * S));
    c->have_sigma = sigma_st != nullptr;
    c->have_scen = true;
    c->npv_gen++;
    return PP_OK;
}

extern "C" {

int pp_set_scenarios(pp_ctx *c, int32_t S, const double *vmax_sb, const double *sigma_st) {
    if (!c || !c->have_instance) return fail(PP_ERR_STATE, "pp_set_instance first");
    if (S < 1 || !vmax_sb) return fail(PP_ERR_INVALID_ARGS, "need n_scenarios >= 1 and a value table");
    const int B = c->B;
    DevBuf tmp;
    TRY(tmp.ensure(sizeof(double) * (size_t)S * B));
    const int rc = set_scenarios_common(c, S, sigma_st, [&](int Sp) {
        cudaError_t e = dev_upload(c, tmp.ptr, vmax_sb, sizeof(double) * (size_t)S * B);
        if (e == cudaSuccess) {
            k_scen_tables<<<(B + 255) / 256, 256, 0, c->stream>>>(tmp.as<double>(), S, B, Sp, c->vmax.as<double>(),
                                                                  c->unit_mean.as<double>());
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
        return e;
    });
    tmp.release();
    return rc;
}

int pp_set_scenarios_grades(pp_ctx *c, int32_t S, const double *grades_sb, int32_t n_modes, double price,
                            const double *recovery, int32_t n_recovery, const double *proc_cost, int32_t n_proc_cost,
                            const double *sigma_st) {
    if (!c || !c->have_instance) return fail(PP_ERR_STATE, "pp_set_instance first");
    if (S < 1 || !grades_sb) return fail(PP_ERR_INVALID_ARGS, "need n_scenarios >= 1 and a grade matrix");
    if (n_modes < 1 || !recovery || n_recovery < 1 || !proc_cost || n_proc_cost < 1)
        return fail(PP_ERR_INVALID_ARGS, "need at least one operating mode with recovery and processing cost");
    const int B = c->B;
    DevBuf tmp, par;
    TRY(tmp.ensure(sizeof(double) * (size_t)S * B));
    TRY(par.ensure(sizeof(double) * (size_t)(n_recovery + n_proc_cost)));
    const int rc = set_scenarios_common(c, S, sigma_st, [&](int Sp) {
        cudaError_t e = dev_upload(c, tmp.ptr, grades_sb, sizeof(double) * (size_t)S * B);
        if (e == cudaSuccess) e = dev_upload(c, par.ptr, recovery, sizeof(double) * n_recovery);
        if (e == cudaSuccess)
            e = dev_upload(c, par.as<double>() + n_recovery, proc_cost, sizeof(double) * n_proc_cost);
        if (e == cudaSuccess) {
            k_scen_from_grades<<<(B + 127) / 128, 128, 0, c->stream>>>(
                tmp.as<double>(), S, B, Sp, c->mass.as<double>(), price, par.as<double>(), n_recovery,
                par.as<double>() + n_recovery, n_proc_cost, n_modes, c->vmax.as<double>(), c->unit_mean.as<double>());
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
        return e;
    });
    tmp.release();
    par.release();
    return rc;
}

}  // extern "C"

// grades[S][B] already on the device (the VAE decode, pp_vae.cu) bound as the scenario set: the value
// table built by k_scen_from_grades exactly as pp_set_scenarios_grades does for host grades
int set_scenarios_from_device_grades(pp_ctx *c, int32_t S, const double *dgrades, int32_t n_modes, double price,
                                     const double *recovery, int32_t n_recovery, const double *proc_cost,
                                     int32_t n_proc_cost, const double *sigma_st) {
    if (!c || !c->have_instance) return fail(PP_ERR_STATE, "pp_set_instance first");
    if (S < 1 || !dgrades) return fail(PP_ERR_INVALID_ARGS, "need n_scenarios >= 1 and a grade matrix");
    if (n_modes < 1 || !recovery || n_recovery < 1 || !proc_cost || n_proc_cost < 1)
        return fail(PP_ERR_INVALID_ARGS, "need at least one operating mode with recovery and processing cost");
    const int B = c->B;
    DevBuf par;
    TRY(par.ensure(sizeof(double) * (size_t)(n_recovery + n_proc_cost)));
    const int rc = set_scenarios_common(c, S, sigma_st, [&](int Sp) {
        cudaError_t e = dev_upload(c, par.ptr, recovery, sizeof(double) * n_recovery);
        if (e == cudaSuccess) e = dev_upload(c, par.as<double>() + n_recovery, proc_cost, sizeof(double) * n_proc_cost);
        if (e == cudaSuccess) {
            k_scen_from_grades<<<(B + 127) / 128, 128, 0, c->stream>>>(
                dgrades, S, B, Sp, c->mass.as<double>(), price, par.as<double>(), n_recovery,
                par.as<double>() + n_recovery, n_proc_cost, n_modes, c->vmax.as<double>(), c->unit_mean.as<double>());
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
        return e;
    });
    par.release();
    return rc;
}

extern "C" {

int pp_get_scenario_values(pp_ctx *c, double *vmax_sb_out) {
    if (!c || !c->have_scen) return fail(PP_ERR_STATE, "pp_set_scenarios first");
    if (!vmax_sb_out) return fail(PP_ERR_INVALID_ARGS, "vmax_sb_out is NULL");
    TRY(use_device(c));
    const size_t n = (size_t)c->S * c->B;
    DevBuf tmp;
    TRY(tmp.ensure(sizeof(double) * n));
    k_scen_to_sb<<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(c->vmax.as<double>(), c->S, c->B, c->Sp,
                                                                    tmp.as<double>());
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(vmax_sb_out, tmp.ptr, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    tmp.release();
    if (e != cudaSuccess) return fail(PP_ERR_CUDA, "pp_get_scenario_values: %s", cudaGetErrorString(e));
    return PP_OK;
}

int pp_set_schedule(pp_ctx *c, const int32_t *assign, int32_t mem, void *stream) {
    HostTrace ht("pp_set_schedule");
    if (!c || !c->have_instance) return fail(PP_ERR_STATE, "pp_set_instance first");
    if (!assign) return fail(PP_ERR_INVALID_ARGS, "assign is NULL");
    if (mem != PP_MEM_HOST && mem != PP_MEM_DEVICE && mem != PP_MEM_DEVICE_BORROW)
        return fail(PP_ERR_INVALID_ARGS, "unknown memory kind %d", mem);
    TRY(use_device(c));
    cudaStream_t st = pick(c, stream);
    c->bad_pending = false;
    if (mem == PP_MEM_HOST && pm_cluster_path(c)) {  // range-checked by k_pm_cluster on the device
        if (!c->pm_bad.ptr) {
            TRY(c->pm_bad.ensure(sizeof(int32_t) * PMC_R16));
            CUDA_TRY(dev_zero(c, c->pm_bad.ptr, sizeof(int32_t) * PMC_R16));
            CUDA_TRY(cudaHostAlloc(reinterpret_cast<void **>(&c->h_bad), sizeof(int32_t) * PMC_R16,
                                   cudaHostAllocPortable | cudaHostAllocMapped));
        }
        c->bad_pending = true;
    } else if (mem == PP_MEM_HOST) {  // branch-free min/max (vectorises)
        int32_t lo = 0, hi = -1;
        for (int b = 0; b < c->B; b++) {
            lo = std::min(lo, assign[b]);
            hi = std::max(hi, assign[b]);
        }
        if (lo < -1 || hi >= c->T) return fail(PP_ERR_INVALID_ARGS, "schedule has period indices out of range");
        ht.mark("validate");
    }
    if (mem == PP_MEM_DEVICE_BORROW) {
        c->assign_ptr = assign;  // read in place until the next pp_set_schedule
        c->borrowed = true;
    } else {
        CUDA_TRY(cudaMemcpyAsync(c->assign.ptr, assign, sizeof(int32_t) * c->B,
                                 mem == PP_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
        c->assign_ptr = c->assign.as<int32_t>();
        c->borrowed = false;
    }
    c->pm_dirty = true;  // period masses are recomputed by the next evaluation launch (PDL-overlapped)
    c->have_sched = true;  // host copies are stream-ordered (see the header), no synchronisation here
    return PP_OK;
}

int pp_apply_moves(pp_ctx *c, const int32_t *blocks, const int32_t *periods, int32_t n, int32_t mem, void *stream) {
    if (!c || !c->have_sched) return fail(PP_ERR_STATE, "pp_set_schedule first");
    if (n < 0 || (n > 0 && (!blocks || !periods))) return fail(PP_ERR_INVALID_ARGS, "bad move arrays");
    TRY(use_device(c));
    cudaStream_t st = pick(c, stream);
    if (n == 0) return PP_OK;
    if (c->borrowed) {  // take a private copy before writing
        CUDA_TRY(cudaMemcpyAsync(c->assign.ptr, c->assign_ptr, sizeof(int32_t) * c->B, cudaMemcpyDeviceToDevice, st));
        c->assign_ptr = c->assign.as<int32_t>();
        c->borrowed = false;
    }
    const int32_t *db = blocks, *dp = periods;
    if (mem == PP_MEM_HOST) {
        for (int k = 0; k < n; k++)
            if (blocks[k] < 0 || blocks[k] >= c->B || periods[k] < -1 || periods[k] >= c->T)
                return fail(PP_ERR_INVALID_ARGS, "move (%d, %d) out of range", blocks[k], periods[k]);
        TRY(c->h_a.ensure(sizeof(int32_t) * n));
        TRY(c->h_b.ensure(sizeof(int32_t) * n));
        CUDA_TRY(cudaMemcpyAsync(c->h_a.ptr, blocks, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(c->h_b.ptr, periods, sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
        db = c->h_a.as<int32_t>();
        dp = c->h_b.as<int32_t>();
    }
    k_apply_moves<<<1, 32, 0, st>>>(c->assign.as<int32_t>(), c->B, c->T, db, dp, n);
    CUDA_TRY(cudaGetLastError());
    c->pm_dirty = true;
    if (mem == PP_MEM_HOST) CUDA_TRY(cudaStreamSynchronize(st));
    return PP_OK;
}

int pp_get_schedule(pp_ctx *c, int32_t *assign_out, double *pm_out, int32_t mem, void *stream) {
    if (!c || !c->have_sched) return fail(PP_ERR_STATE, "pp_set_schedule first");
    TRY(use_device(c));
    cudaStream_t st = pick(c, stream);
    bool launched;
    if (pm_out) TRY(refresh_pm(c, st, &launched));
    cudaMemcpyKind k = (mem == PP_MEM_HOST) ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    if (assign_out) CUDA_TRY(cudaMemcpyAsync(assign_out, c->assign_ptr, sizeof(int32_t) * c->B, k, st));
    if (pm_out) CUDA_TRY(cudaMemcpyAsync(pm_out, c->pm.ptr, sizeof(double) * c->T, k, st));
    if (mem == PP_MEM_HOST) {
        CUDA_TRY(cudaStreamSynchronize(st));
        TRY(check_schedule_range(c, false));
    }
    return PP_OK;
}

int pp_check_feasible(pp_ctx *c, const int32_t *assign, int32_t P, int64_t *pred_count, double *excess,
                      double *violation, double *period_mass, int32_t mem, void *stream) {
    if (!c || !c->have_instance) return fail(PP_ERR_STATE, "pp_set_instance first");
    if (P < 0 || (P > 0 && !assign) || !pred_count || !excess || !violation)
        return fail(PP_ERR_INVALID_ARGS, "bad arguments");
    if (P == 0) return PP_OK;
    TRY(use_device(c));
    cudaStream_t st = pick(c, stream);
    const int B = c->B, T = c->T;
    const int32_t *da = assign;
    int64_t *dcnt = pred_count;
    double *dex = excess, *dvi = violation, *dpm = period_mass;
    if (mem == PP_MEM_HOST) {
        TRY(c->h_assign.ensure(sizeof(int32_t) * (size_t)P * B));
        TRY(c->h_i64.ensure(sizeof(int64_t) * P));
        TRY(c->h_d1.ensure(sizeof(double) * P));
        TRY(c->h_d2.ensure(sizeof(double) * P));
        TRY(c->h_pm.ensure(sizeof(double) * (size_t)P * T));
        CUDA_TRY(cudaMemcpyAsync(c->h_assign.ptr, assign, sizeof(int32_t) * (size_t)P * B, cudaMemcpyHostToDevice, st));
        da = c->h_assign.as<int32_t>();
        dcnt = c->h_i64.as<int64_t>();
        dex = c->h_d1.as<double>();
        dvi = c->h_d2.as<double>();
        dpm = c->h_pm.as<double>();
    } else if (!dpm) {
        TRY(c->pm_batch.ensure(sizeof(double) * (size_t)P * T));
        dpm = c->pm_batch.as<double>();
    }
    TRY(c->predcnt.ensure(sizeof(unsigned long long) * P));
    CUDA_TRY(cudaMemsetAsync(c->predcnt.ptr, 0, sizeof(unsigned long long) * P, st));
    TRY(run_period_mass(c, da, P, dpm, st));
    k_pred_count<<<dim3((B + 255) / 256, P), 256, 0, st>>>(da, c->rows.as<BlockRow>(), c->adj.as<int32_t>(), B,
                                                           c->predcnt.as<unsigned long long>());
    k_feas_final<<<(P + 127) / 128, 128, 0, st>>>(dpm, c->cap.as<double>(), T, P, c->mean_cap,
                                                  c->predcnt.as<unsigned long long>(), dcnt, dex, dvi);
    CUDA_TRY(cudaGetLastError());
    if (mem == PP_MEM_HOST) {
        CUDA_TRY(cudaMemcpyAsync(pred_count, dcnt, sizeof(int64_t) * P, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(excess, dex, sizeof(double) * P, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(violation, dvi, sizeof(double) * P, cudaMemcpyDeviceToHost, st));
        if (period_mass)
            CUDA_TRY(cudaMemcpyAsync(period_mass, dpm, sizeof(double) * (size_t)P * T, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
    }
    return PP_OK;
}

int pp_repair(pp_ctx *c, int32_t *assign, int32_t P, int32_t mode, uint8_t *unmined_out, int32_t mem, void *stream) {
    if (!c || !c->have_instance) return fail(PP_ERR_STATE, "pp_set_instance first");
    if (P < 0 || (P > 0 && !assign)) return fail(PP_ERR_INVALID_ARGS, "bad arguments");
    if (mode != PP_REPAIR_PUSH_FORWARD && mode != PP_REPAIR_UNMINE) return fail(PP_ERR_INVALID_ARGS, "unknown repair mode %d", mode);
    if (P == 0) return PP_OK;
    TRY(use_device(c));
    cudaStream_t st = pick(c, stream);
    const int B = c->B;
    int32_t *da = assign;
    uint8_t *du = unmined_out;
    if (mem == PP_MEM_HOST) {
        TRY(c->h_assign.ensure(sizeof(int32_t) * (size_t)P * B));
        CUDA_TRY(cudaMemcpyAsync(c->h_assign.ptr, assign, sizeof(int32_t) * (size_t)P * B, cudaMemcpyHostToDevice, st));
        da = c->h_assign.as<int32_t>();
        if (unmined_out) {
            TRY(c->h_o5.ensure((size_t)P * B));
            du = c->h_o5.as<uint8_t>();
        }
    }
    if (du) CUDA_TRY(cudaMemsetAsync(du, 0, (size_t)P * B, st));
    for (int l = 1; l < c->n_levels; l++) {
        int ls = c->level_ptr[l], lc = c->level_ptr[l + 1] - ls;
        if (lc <= 0) continue;
        k_repair_level<<<dim3((lc + 255) / 256, P), 256, 0, st>>>(da, B, c->rows.as<BlockRow>(), c->adj.as<int32_t>(),
                                                                  c->level_blocks.as<int32_t>(), ls, lc, mode, du);
    }
    CUDA_TRY(cudaGetLastError());
    if (mem == PP_MEM_HOST) {
        CUDA_TRY(cudaMemcpyAsync(assign, da, sizeof(int32_t) * (size_t)P * B, cudaMemcpyDeviceToHost, st));
        if (unmined_out) CUDA_TRY(cudaMemcpyAsync(unmined_out, du, (size_t)P * B, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
    }
    return PP_OK;
}

int pp_eject(pp_ctx *c, int32_t *assign, int32_t P, const double *mean_grade, double destroy_fraction,
             uint8_t *ejected_out, int32_t mem, void *stream) {
    if (!c || !c->have_instance) return fail(PP_ERR_STATE, "pp_set_instance first");
    if (P < 0 || (P > 0 && (!assign || !mean_grade))) return fail(PP_ERR_INVALID_ARGS, "bad arguments");
    if (!(destroy_fraction >= 0.0)) return fail(PP_ERR_INVALID_ARGS, "destroy_fraction must be >= 0");
    if (P == 0) return PP_OK;
    TRY(use_device(c));
    cudaStream_t st = pick(c, stream);
    const int B = c->B, T = c->T;
    int32_t *da = assign;
    uint8_t *du = ejected_out;
    const double *dg = mean_grade;
    if (mem == PP_MEM_HOST) {
        TRY(c->h_assign.ensure(sizeof(int32_t) * (size_t)P * B));
        TRY(c->h_d2.ensure(sizeof(double) * (size_t)B));
        CUDA_TRY(cudaMemcpyAsync(c->h_assign.ptr, assign, sizeof(int32_t) * (size_t)P * B, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(c->h_d2.ptr, mean_grade, sizeof(double) * B, cudaMemcpyHostToDevice, st));
        da = c->h_assign.as<int32_t>();
        dg = c->h_d2.as<double>();
        if (ejected_out) {
            TRY(c->h_o5.ensure((size_t)P * B));
            du = c->h_o5.as<uint8_t>();
        }
    }
    if (du) CUDA_TRY(cudaMemsetAsync(du, 0, (size_t)P * B, st));
    TRY(c->pm_batch.ensure(sizeof(double) * (size_t)P * T));
    TRY(c->ej_count.ensure(sizeof(int32_t) * T));
    TRY(c->ej_key.ensure(sizeof(double) * (size_t)T * B));
    TRY(c->ej_blk.ensure(sizeof(int32_t) * (size_t)T * B));
    TRY(run_period_mass(c, da, P, c->pm_batch.as<double>(), st));
    for (int p = 0; p < P; p++) {  // one schedule at a time: the lists use [T][B] scratch
        int32_t *ap = da + (size_t)p * B;
        const double *pmp = c->pm_batch.as<double>() + (size_t)p * T;
        CUDA_TRY(cudaMemsetAsync(c->ej_count.ptr, 0, sizeof(int32_t) * T, st));
        k_eject_list<<<(B + 255) / 256, 256, 0, st>>>(ap, B, T, c->rows.as<BlockRow>(), c->adj.as<int32_t>(), pmp,
                                                      c->cap.as<double>(), dg, destroy_fraction,
                                                      c->ej_count.as<int32_t>(), c->ej_key.as<double>(),
                                                      c->ej_blk.as<int32_t>());
        k_eject_apply<<<T, 512, 0, st>>>(ap, B, c->mass.as<double>(), pmp, c->cap.as<double>(), destroy_fraction,
                                         c->ej_count.as<int32_t>(), c->ej_key.as<double>(), c->ej_blk.as<int32_t>(),
                                         du ? du + (size_t)p * B : nullptr);
    }
    CUDA_TRY(cudaGetLastError());
    if (mem == PP_MEM_HOST) {
        CUDA_TRY(cudaMemcpyAsync(assign, da, sizeof(int32_t) * (size_t)P * B, cudaMemcpyDeviceToHost, st));
        if (ejected_out) CUDA_TRY(cudaMemcpyAsync(ejected_out, du, (size_t)P * B, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(stream_wait(st));
    }
    return PP_OK;
}

int pp_get_spatial(pp_ctx *c, double *out, int32_t mem, void *stream) {
    if (!c || !c->have_instance || !c->have_spatial) return fail(PP_ERR_STATE, "pp_set_instance and pp_set_geology first");
    if (!out) return fail(PP_ERR_INVALID_ARGS, "out is NULL");
    TRY(use_device(c));
    cudaStream_t st = pick(c, stream);
    // BlockRow.spatial: one strided 2-D copy (pitch 32 bytes -> 8 bytes)
    const char *src = reinterpret_cast<const char *>(c->rows.ptr) + offsetof(BlockRow, spatial);
    CUDA_TRY(cudaMemcpy2DAsync(out, sizeof(double), src, sizeof(BlockRow), sizeof(double), c->B,
                               mem == PP_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, st));
    if (mem == PP_MEM_HOST) CUDA_TRY(stream_wait(st));
    return PP_OK;
}

int pp_reduce_best(pp_ctx *c, const pp_best *recs, int32_t n, pp_best *out, int32_t mem, void *stream) {
    if (!c || n < 0 || (n > 0 && !recs) || !out) return fail(PP_ERR_INVALID_ARGS, "bad arguments");
    TRY(use_device(c));
    cudaStream_t st = pick(c, stream);
    const pp_best *dr = recs;
    pp_best *dout = out;
    if (mem == PP_MEM_HOST) {
        TRY(c->h_d1.ensure(sizeof(pp_best) * (size_t)std::max(n, 1)));
        TRY(c->h_glob.ensure(sizeof(pp_best)));
        if (n > 0) CUDA_TRY(cudaMemcpyAsync(c->h_d1.ptr, recs, sizeof(pp_best) * n, cudaMemcpyHostToDevice, st));
        dr = c->h_d1.as<pp_best>();
        dout = c->h_glob.as<pp_best>();
    }
    k_reduce_best<<<1, 32, 0, st>>>(dr, n, dout);
    CUDA_TRY(cudaGetLastError());
    if (mem == PP_MEM_HOST) {
        CUDA_TRY(cudaMemcpyAsync(out, dout, sizeof(pp_best), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
    }
    return PP_OK;
}

int pp_enpv_table(pp_ctx *c, uint32_t flags, int32_t factored, double *out, int32_t mem, void *stream) {
    if (!c || !c->have_instance || !c->have_scen) return fail(PP_ERR_STATE, "pp_set_instance and pp_set_scenarios first");
    if (!out) return fail(PP_ERR_INVALID_ARGS, "out is NULL");
    if ((flags & PP_USE_SIGMA) && !c->have_sigma) return fail(PP_ERR_STATE, "PP_USE_SIGMA without an uploaded sigma");
    TRY(use_device(c));
    cudaStream_t st = pick(c, stream);
    const size_t n = (size_t)c->B * c->T;
    double *dout = out;
    if (mem == PP_MEM_HOST) {
        TRY(c->h_o4.ensure(sizeof(double) * n));
        dout = c->h_o4.as<double>();
    }
    const double *sig = (flags & PP_USE_SIGMA) ? c->sigma.as<double>() : c->ones_st.as<double>();
    k_enpv_table<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(c->vmax.as<double>(), c->Sp, c->S, c->B, c->T, sig,
                                                              c->disc.as<double>(), c->cost.as<double>(),
                                                              factored ? 1 : 0, dout);
    CUDA_TRY(cudaGetLastError());
    if (mem == PP_MEM_HOST) {
        CUDA_TRY(cudaMemcpyAsync(out, dout, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
    }
    return PP_OK;
}


int pp_get_levels(pp_ctx *c, int32_t *n_levels, int32_t *level_of_block) {
    if (!c || !c->have_instance) return fail(PP_ERR_STATE, "pp_set_instance first");
    if (n_levels) *n_levels = c->n_levels;
    if (level_of_block) memcpy(level_of_block, c->level_of.data(), sizeof(int32_t) * c->B);
    return PP_OK;
}

}  // extern "C"
