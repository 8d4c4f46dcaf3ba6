// pitplan_b200.cu -- sm_100a kernels and the C ABI of the move-evaluation engine.
//
// Hot path (reference: /root/reference/pkg/src/pitplan/evaluate.py:306-430):
//   k_pm_count / k_pm_scatter / k_pm_leaf   period_mass[t] = masses[assign == t].sum()
//                                           with numpy's pairwise tree, bit-exact
//   k_eval_candidates<G,PER,KC>             K1+K2+K3+K4 fused: one lane group per candidate,
//                                           lanes = periods; precedence window by segmented
//                                           shuffle max/min, capacity test, fp64 value in the
//                                           reference op order, per-scenario deltas with
//                                           expected (pairwise mean) and CVaR10, per-candidate
//                                           argmax, CTA argmax, last-CTA grid argmax
//   k_eval_moves<KC>                        explicit reassign / unmine / swap moves
//   k_pred_count / k_feas_final             check_feasible (evaluate.py:82-105)
//   k_repair_level                          topological-wave repair (hybrid.py:493-510, 199-211)
//
// All float arithmetic on the value path uses explicit round-to-nearest intrinsics and the
// file is compiled with -fmad=false: no multiply-add is ever contracted, so every double
// matches the reference's numpy/Python scalar evaluation bit for bit.

#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "pitplan_b200.h"

// ------------------------------------------------------------------------------------
// error plumbing
// ------------------------------------------------------------------------------------
static thread_local std::string g_last_error;

static int fail(int code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

#define CUDA_TRY(expr)                                                                     \
    do {                                                                                   \
        cudaError_t e_ = (expr);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return fail(PP_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                               \
    } while (0)

#define TRY(expr)                    \
    do {                             \
        int rc_ = (expr);            \
        if (rc_ != PP_OK) return rc_; \
    } while (0)

// ------------------------------------------------------------------------------------
// device helpers: IEEE binary64, round-to-nearest, never contracted
// ------------------------------------------------------------------------------------
__device__ __forceinline__ double f64_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double f64_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double f64_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double f64_div(double a, double b) { return __ddiv_rn(a, b); }

__device__ __forceinline__ double tree8(const double r[8]) {
    // ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7))   (numpy pairwise block combine)
    return f64_add(f64_add(f64_add(r[0], r[1]), f64_add(r[2], r[3])), f64_add(f64_add(r[4], r[5]), f64_add(r[6], r[7])));
}

constexpr double kInf = __builtin_huge_val();

// Per-block static record: one 32-byte load gives mass, spatial factor and adjacency.
struct __align__(16) BlockRow {
    double mass;
    double spatial;
    int32_t adj;  // offset into adj[]: predecessors then successors, reference order
    int32_t cnt;  // npred | nsucc << 16
    int32_t level;
    int32_t pad;
};

// numpy pairwise-sum plan for a fixed length n: leaves in order, plus the number of
// post-order additions that follow each leaf.
constexpr int kMaxLeaves = 32;
struct PwPlan {
    int n;
    int nleaf;
    int start[kMaxLeaves];
    int len[kMaxLeaves];
    int adds[kMaxLeaves];
};

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

// Device copy of a PwPlan: int words [n, nleaf, start[kMaxLeaves], len[kMaxLeaves], adds[kMaxLeaves]].
constexpr int kPlanWords = 2 + 3 * kMaxLeaves;
static void plan_words(const PwPlan &p, int *w) {
    w[0] = p.n;
    w[1] = p.nleaf;
    for (int i = 0; i < kMaxLeaves; i++) {
        w[2 + i] = p.start[i];
        w[2 + kMaxLeaves + i] = p.len[i];
        w[2 + 2 * kMaxLeaves + i] = p.adds[i];
    }
}

// Streaming numpy pairwise sum over x[0..n), fed 8 values at a time in order.  Every leaf
// of numpy's recursion starts at a multiple of 8 and all but the last end on one, and the
// 8-accumulator part of a leaf covers whole 8-blocks, so each 8-block is either entirely
// "main" (accumulator j gets element j of the block) or entirely remainder.
struct PwStream {
    double r[8];
    double res;
    double stk[8];
    int sp, leaf, nleaf, ls, le, lmain;

    __device__ __forceinline__ void set_leaf(const int *P) {
        ls = __ldg(P + 2 + leaf);
        int L = __ldg(P + 2 + kMaxLeaves + leaf);
        le = ls + L;
        lmain = (L >= 8) ? ls + L - (L & 7) : ls;
        res = -0.0;
    }
    __device__ __forceinline__ void begin(const int *P) {
        sp = 0;
        leaf = 0;
        nleaf = __ldg(P + 1);
        set_leaf(P);
    }
    // x[0..nvalid) are elements s8 .. s8+nvalid-1 (s8 a multiple of 8)
    __device__ __forceinline__ void block(int s8, const double x[8], int nvalid, const int *P) {
        if (s8 < lmain) {
            if (s8 == ls) {
#pragma unroll
                for (int j = 0; j < 8; j++) r[j] = x[j];
            } else {
#pragma unroll
                for (int j = 0; j < 8; j++) r[j] = f64_add(r[j], x[j]);
            }
            if (s8 + 8 == lmain) res = tree8(r);
        } else {
#pragma unroll
            for (int j = 0; j < 8; j++)
                if (j < nvalid) res = f64_add(res, x[j]);
        }
        if (s8 + 8 >= le) finish(P);
    }
    __device__ __forceinline__ void finish(const int *P) {
        stk[sp++] = res;
        const int nadd = __ldg(P + 2 + 2 * kMaxLeaves + leaf);
        for (int a = 0; a < nadd; a++) {
            double rhs = stk[--sp];
            double lhs = stk[--sp];
            stk[sp++] = f64_add(lhs, rhs);
        }
        leaf++;
        if (leaf < nleaf) set_leaf(P);
    }
    // float(np.mean(x)) = (0.0 + pairwise(x)) / n
    __device__ __forceinline__ double mean(const int *P) const { return f64_div(f64_add(0.0, stk[0]), (double)__ldg(P)); }
};

// k smallest values seen (ascending), for CVaR10 (saa.py:157-164).
template <int KC>
struct TopK {
    double a[KC];
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int j = 0; j < KC; j++) a[j] = kInf;
    }
    __device__ __forceinline__ void push(double x) {
        if (x < a[KC - 1]) {
            if constexpr (KC <= 8) {
#pragma unroll
                for (int j = KC - 1; j > 0; j--) a[j] = (x < a[j - 1]) ? a[j - 1] : ((x < a[j]) ? x : a[j]);
                a[0] = (x < a[0]) ? x : a[0];
            } else {  // insertion sort step in local memory
                int j = KC - 1;
                while (j > 0 && x < a[j - 1]) {
                    a[j] = a[j - 1];
                    j--;
                }
                a[j] = x;
            }
        }
    }
    // float(srt[:k].mean()) = (0.0 + pairwise(a[0..k))) / k,  k <= 128
    __device__ __forceinline__ double mean(int k) const {
        double s;
        if (k < 8) {
            s = -0.0;
#pragma unroll
            for (int j = 0; j < KC; j++)
                if (j < k) s = f64_add(s, a[j]);
        } else {
            double r[8];
#pragma unroll
            for (int j = 0; j < 8; j++) r[j] = a[j < KC ? j : 0];
            int main_ = k - (k & 7);
            for (int i = 8; i < main_; i += 8)
#pragma unroll
                for (int j = 0; j < 8; j++) r[j] = f64_add(r[j], a[(i + j) < KC ? (i + j) : 0]);
            s = tree8(r);
            for (int i = main_; i < k; i++) s = f64_add(s, a[i < KC ? i : 0]);
        }
        return f64_div(f64_add(0.0, s), (double)k);
    }
};
template <>
struct TopK<0> {
    __device__ __forceinline__ void init() {}
    __device__ __forceinline__ void push(double) {}
    __device__ __forceinline__ double mean(int) const { return 0.0; }
};

// selection order of evaluate.py:404-409: value desc, then block asc, then period asc
struct Best {
    double v;
    int b;
    int t;
};
__device__ __forceinline__ bool better(const Best &x, const Best &y) {
    return x.v > y.v || (x.v == y.v && (x.b < y.b || (x.b == y.b && x.t < y.t)));
}
__device__ __forceinline__ Best shfl_best(const Best &x, int off) {
    Best y;
    y.v = __shfl_xor_sync(0xffffffffu, x.v, off);
    y.b = __shfl_xor_sync(0xffffffffu, x.b, off);
    y.t = __shfl_xor_sync(0xffffffffu, x.t, off);
    return y;
}

// CTA argmax of per-thread candidates in smem, then the last CTA to finish reduces the
// per-CTA partials in index order.  Deterministic: `better` is a total order.
__device__ void grid_argmax(Best mine, Best *s_red, pp_best *partial, unsigned int *counter,
                            pp_best *global) {
    __shared__ bool s_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        Best o = shfl_best(mine, off);
        if (better(o, mine)) mine = o;
    }
    if (lane == 0) s_red[warp] = mine;
    __syncthreads();
    if (warp == 0) {
        Best x = (lane < nw) ? s_red[lane] : Best{-kInf, INT_MAX, INT_MAX};
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            Best o = shfl_best(x, off);
            if (better(o, x)) x = o;
        }
        if (lane == 0) {
            pp_best pb;
            pb.value = x.v;
            pb.block = x.b;
            pb.period = x.t;
            partial[blockIdx.x] = pb;
            __threadfence();
            unsigned int prev = atomicAdd(counter, 1u);
            s_last = (prev == gridDim.x - 1);
        }
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    Best x{-kInf, INT_MAX, INT_MAX};
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
        const pp_best *q = partial + i;
        Best o{__ldcg(&q->value), __ldcg(&q->block), __ldcg(&q->period)};
        if (better(o, x)) x = o;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        Best o = shfl_best(x, off);
        if (better(o, x)) x = o;
    }
    if (lane == 0) s_red[warp] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        Best y = s_red[0];
        for (int w = 1; w < nw; w++)
            if (better(s_red[w], y)) y = s_red[w];
        pp_best g;
        bool none = (y.b == INT_MAX);
        g.value = none ? -kInf : y.v;
        g.block = none ? -1 : y.b;
        g.period = none ? -1 : y.t;
        *global = g;
        *counter = 0u;  // re-arm for the next launch (graph replay safe)
    }
}

// ------------------------------------------------------------------------------------
// period mass, bit-exact numpy pairwise summation per period
// ------------------------------------------------------------------------------------
constexpr int PM_THREADS = 256;
constexpr int PM_ITEMS = 8;
constexpr int PM_CHUNK = PM_THREADS * PM_ITEMS;  // blocks per chunk
constexpr int PM_MAXT = 128;

// per-(schedule, chunk) count of blocks in each period
__global__ void __launch_bounds__(PM_THREADS) k_pm_count(const int32_t *__restrict__ assign, int B, int T,
                                                           int nchunk, int32_t *__restrict__ cnt) {
    __shared__ int h[PM_MAXT];
    const int p = blockIdx.y, chunk = blockIdx.x;
    for (int i = threadIdx.x; i < T; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const int32_t *a = assign + (size_t)p * B;
    const int base = chunk * PM_CHUNK;
#pragma unroll
    for (int k = 0; k < PM_ITEMS; k++) {
        int b = base + k * PM_THREADS + threadIdx.x;
        int t = (b < B) ? a[b] : -1;
        if (t < 0 || t >= T) t = -1;
        unsigned m = __match_any_sync(0xffffffffu, t);
        int leader = __ffs(m) - 1;
        if (t >= 0 && (threadIdx.x & 31) == leader) atomicAdd(&h[t], __popc(m));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < T; i += blockDim.x) cnt[((size_t)p * nchunk + chunk) * T + i] = h[i];
}

// stable compaction of masses by period (block order) into compact[p][start_t + rank]
__global__ void __launch_bounds__(PM_THREADS) k_pm_scatter(const int32_t *__restrict__ assign,
                                                             const BlockRow *__restrict__ rows, int B, int T,
                                                             int nchunk, const int32_t *__restrict__ cnt,
                                                             double *__restrict__ compact) {
    __shared__ int s_off[PM_MAXT];
    __shared__ int s_tot[PM_MAXT];
    __shared__ int s_wc[PM_THREADS / 32][PM_MAXT];
    const int p = blockIdx.y, chunk = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int t = threadIdx.x; t < T; t += blockDim.x) {
        int tot = 0, pre = 0;
        const int32_t *c = cnt + (size_t)p * nchunk * T + t;
        for (int k = 0; k < nchunk; k++) {
            int v = c[(size_t)k * T];
            tot += v;
            if (k < chunk) pre += v;
        }
        s_tot[t] = tot;
        s_off[t] = pre;
    }
    for (int i = threadIdx.x; i < (PM_THREADS / 32) * PM_MAXT; i += blockDim.x) (&s_wc[0][0])[i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
        int run = 0;
        for (int t = 0; t < T; t++) {
            int v = s_tot[t];
            s_off[t] += run;
            run += v;
        }
    }
    // warp w owns blocks [base + w*256, base + (w+1)*256), 8 steps of 32 consecutive blocks
    const int32_t *a = assign + (size_t)p * B;
    const int wbase = chunk * PM_CHUNK + warp * (32 * PM_ITEMS);
    int tt[PM_ITEMS], rk[PM_ITEMS];
#pragma unroll
    for (int k = 0; k < PM_ITEMS; k++) {
        int b = wbase + k * 32 + lane;
        int t = (b < B) ? a[b] : -1;
        if (t < 0 || t >= T) t = -1;
        unsigned m = __match_any_sync(0xffffffffu, t);
        int before = (t >= 0) ? s_wc[warp][t] : 0;
        rk[k] = before + __popc(m & ((1u << lane) - 1u));
        tt[k] = t;
        __syncwarp();
        if (t >= 0 && lane == __ffs(m) - 1) s_wc[warp][t] = before + __popc(m);
        __syncwarp();
    }
    __syncthreads();
    // exclusive prefix over warps per period
    for (int t = threadIdx.x; t < T; t += blockDim.x) {
        int run = s_off[t];
        for (int w = 0; w < PM_THREADS / 32; w++) {
            int v = s_wc[w][t];
            s_wc[w][t] = run;
            run += v;
        }
    }
    __syncthreads();
    double *out = compact + (size_t)p * B;
#pragma unroll
    for (int k = 0; k < PM_ITEMS; k++) {
        int t = tt[k];
        if (t >= 0) {
            int b = wbase + k * 32 + lane;
            out[s_wc[warp][t] + rk[k]] = rows[b].mass;
        }
    }
}

// one CTA per (period, schedule): pairwise sum of the compacted masses of that period
constexpr int PM_LEAF_CAP = 2048;
__global__ void __launch_bounds__(PM_THREADS) k_pm_leaf(const double *__restrict__ compact,
                                                          const int32_t *__restrict__ cnt, int B, int T,
                                                          int nchunk, double *__restrict__ pm_out) {
    __shared__ int s_tot[PM_MAXT];
    __shared__ int s_ls[PM_LEAF_CAP];
    __shared__ short s_ll[PM_LEAF_CAP];
    __shared__ unsigned char s_adds[PM_LEAF_CAP];
    __shared__ double s_sum[PM_LEAF_CAP];
    __shared__ int s_nleaf, s_start, s_n;
    const int t = blockIdx.x, p = blockIdx.y;
    for (int i = threadIdx.x; i < T; i += blockDim.x) {
        int tot = 0;
        const int32_t *c = cnt + (size_t)p * nchunk * T + i;
        for (int k = 0; k < nchunk; k++) tot += c[(size_t)k * T];
        s_tot[i] = tot;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int st = 0;
        for (int i = 0; i < t; i++) st += s_tot[i];
        s_start = st;
        s_n = s_tot[t];
        // iterative DFS: leaves in order, post-order add counts attached to the last leaf
        int stk_o[64], stk_n[64], sp = 0, nl = 0;
        int nleaf_overflow = 0;
        // emulate recursion plan_rec(o, n) with an explicit stack of frames
        // frame kinds: >=0 node to expand, marker -1 = "emit add after previous leaf"
        stk_o[sp] = 0;
        stk_n[sp] = s_n;
        sp++;
        while (sp > 0) {
            sp--;
            int o = stk_o[sp], n = stk_n[sp];
            if (n < 0) {  // add marker
                if (nl > 0 && nl <= PM_LEAF_CAP) s_adds[nl - 1]++;
                continue;
            }
            if (n <= 128) {
                if (nl < PM_LEAF_CAP) {
                    s_ls[nl] = o;
                    s_ll[nl] = (short)n;
                    s_adds[nl] = 0;
                } else {
                    nleaf_overflow = 1;
                }
                nl++;
                continue;
            }
            int n2 = n / 2;
            n2 -= n2 % 8;
            // push in reverse: add marker, right, left
            stk_o[sp] = 0;
            stk_n[sp] = -1;
            sp++;
            stk_o[sp] = o + n2;
            stk_n[sp] = n - n2;
            sp++;
            stk_o[sp] = o;
            stk_n[sp] = n2;
            sp++;
        }
        s_nleaf = nleaf_overflow ? -1 : nl;
    }
    __syncthreads();
    const int n = s_n;
    const double *a = compact + (size_t)p * B + s_start;
    if (s_nleaf < 0) {  // pathological size: serial evaluation (correct, slow)
        if (threadIdx.x == 0) {
            // recursive pairwise via explicit stack
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
            pm_out[(size_t)p * T + t] = f64_add(0.0, vp ? vst[0] : -0.0);
        }
        return;
    }
    const int nl = s_nleaf;
    // 8 lanes per leaf: lane j owns accumulator j
    const int sub = threadIdx.x & 7, grp = threadIdx.x >> 3, ngrp = blockDim.x >> 3;
    for (int l0 = 0; l0 < nl; l0 += ngrp) {
        int l = l0 + grp;
        bool act = l < nl;
        int o = act ? s_ls[l] : 0;
        int L = act ? s_ll[l] : 0;
        double r = 0.0;
        if (act && L >= 8) {
            int main_ = L - (L & 7);
            r = a[o + sub];
            for (int i = 8; i < main_; i += 8) r = f64_add(r, a[o + i + sub]);
        }
        // butterfly xor 1, 2, 4 == ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))
        double x1 = __shfl_xor_sync(0xffffffffu, r, 1);
        r = (sub & 1) ? f64_add(x1, r) : f64_add(r, x1);
        double x2 = __shfl_xor_sync(0xffffffffu, r, 2);
        r = (sub & 2) ? f64_add(x2, r) : f64_add(r, x2);
        double x4 = __shfl_xor_sync(0xffffffffu, r, 4);
        r = (sub & 4) ? f64_add(x4, r) : f64_add(r, x4);
        if (act && sub == 0) {
            double res;
            int i;
            if (L < 8) {
                res = -0.0;
                i = 0;
            } else {
                res = r;
                i = L - (L & 7);
            }
            for (; i < L; i++) res = f64_add(res, a[o + i]);
            s_sum[l] = res;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double vst[64];
        int vp = 0;
        for (int l = 0; l < nl; l++) {
            vst[vp++] = s_sum[l];
            for (int k = 0; k < s_adds[l]; k++) {
                double rhs = vst[--vp];
                double lhs = vst[--vp];
                vst[vp++] = f64_add(lhs, rhs);
            }
        }
        pm_out[(size_t)p * T + t] = f64_add(0.0, nl ? vst[0] : -0.0);
    }
}

// ------------------------------------------------------------------------------------
// candidate evaluation: K1 value, K2 precedence window, K3 capacity, K4 argmax
// ------------------------------------------------------------------------------------
struct EvalParams {
    const BlockRow *rows;
    const int32_t *adj;
    const int32_t *assign;
    const double *pm;
    const double *cap;
    const double *disc;
    const double *cost;      // [B][T]
    const double *vmax;      // [B][Sp]
    const double *unit_mean; // [B]
    const double *sig_row;   // [T] (ones / scenario mean / sigma[k])
    const double *sigma;     // [S][T] (ones if no sigma)
    const int32_t *cand;
    int C, B, T, S, Sp, scen, cvar_k;
    unsigned flags;
    const int *plan;
    int32_t *best_t;
    double *best_val;
    uint8_t *feas;
    double *trace_val;
    uint8_t *trace_feas;
    double *exp_delta;
    double *cvar;
    float *scen_delta;
    pp_best *partial;
    unsigned int *counter;
    pp_best *global;
};

constexpr int EV_THREADS = 256;

// Lane groups of G = pow2 >= T lanes (4..32, runtime) evaluate one candidate each; lane
// tl owns periods tl, tl+G, ... (PER slots, PER > 1 only when T > 32).
constexpr int EV_MAX_GPC = (EV_THREADS / 32) * 8;  // groups per CTA at G = 4

template <int PER, int KC>
__global__ void __launch_bounds__(EV_THREADS) k_eval_candidates(const EvalParams p, const int G) {
    __shared__ double s_old[EV_MAX_GPC][32];
    __shared__ Best s_red[EV_THREADS / 32];

    const int GPW = 32 / G, GPC = (EV_THREADS / 32) * GPW;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tl = lane & (G - 1);
    const int gl = warp * GPW + lane / G;  // group within CTA
    const int grp = blockIdx.x * GPC + gl;
    const int T = p.T;
    const bool net = p.flags & PP_NET_MINING_COST;
    int b = (grp < p.C) ? __ldg(p.cand + grp) : -1;
    const bool active = (b >= 0 && b < p.B);
    if (!active) b = 0;

    const BlockRow row = p.rows[b];
    const int ab = p.assign[b];
    double unit;
    if (p.flags & PP_LITERAL_VALUE) unit = f64_mul(row.mass, 100.0);
    else if (p.scen < 0) unit = __ldg(p.unit_mean + b);
    else unit = __ldg(p.vmax + (size_t)b * p.Sp + p.scen);

    double c_t[PER], pm_t[PER], cap_t[PER], d_t[PER], sr_t[PER];
#pragma unroll
    for (int k = 0; k < PER; k++) {
        const int t = tl + k * G;
        const int tc = (t < T) ? t : 0;
        c_t[k] = net ? __ldg(p.cost + (size_t)b * T + tc) : 0.0;
        pm_t[k] = p.pm[tc];
        cap_t[k] = __ldg(p.cap + tc);
        d_t[k] = __ldg(p.disc + tc);
        sr_t[k] = __ldg(p.sig_row + tc);
    }

    // K2: precedence window lo <= t <= hi over the CSR neighbourhood (evaluate.py:361-372)
    const int npred = row.cnt & 0xffff, nnb = npred + (row.cnt >> 16);
    int lo = 0, hi = INT_MAX;
    for (int k = tl; k < nnb; k += G) {
        const int nb = __ldg(p.adj + row.adj + k);
        const int tn = p.assign[nb];
        if (k < npred) lo = max(lo, tn < 0 ? INT_MAX : tn);
        else if (tn >= 0) hi = min(hi, tn);
    }
    for (int off = G >> 1; off > 0; off >>= 1) {
        lo = max(lo, __shfl_xor_sync(0xffffffffu, lo, off, G));
        hi = min(hi, __shfl_xor_sync(0xffffffffu, hi, off, G));
    }

    // K3 capacity (evaluate.py:373-378) + K1 value (evaluate.py:379-384), lowest-t argmax
    bool ok_t[PER];
    Best mine{-kInf, INT_MAX, INT_MAX};
#pragma unroll
    for (int k = 0; k < PER; k++) {
        const int t = tl + k * G;
        bool ok = active && t < T && lo <= t && t <= hi;
        if (ok) {
            double load = f64_add(pm_t[k], row.mass);
            if (ab == t) load = f64_sub(load, row.mass);
            if (load > cap_t[k]) ok = false;
        }
        double v = -kInf;
        if (ok) {
            v = f64_mul(f64_mul(f64_mul(unit, d_t[k]), sr_t[k]), row.spatial);
            if (net) v = f64_sub(v, f64_mul(d_t[k], c_t[k]));
        }
        ok_t[k] = ok;
        if (active && t < T) {
            const size_t m = (size_t)grp * T + t;
            if (p.trace_val) p.trace_val[m] = v;
            if (p.trace_feas) p.trace_feas[m] = ok ? 1 : 0;
        }
        if (ok && (v > mine.v || (v == mine.v && t < mine.t))) {
            mine.v = v;
            mine.t = t;
        }
    }
    for (int off = G >> 1; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, mine.v, off, G);
        const int ot = __shfl_xor_sync(0xffffffffu, mine.t, off, G);
        if (ov > mine.v || (ov == mine.v && ot < mine.t)) {
            mine.v = ov;
            mine.t = ot;
        }
    }
    const bool cand_ok = mine.t != INT_MAX;
    if (active && tl == 0) {
        p.best_t[grp] = cand_ok ? mine.t : -1;
        p.best_val[grp] = mine.v;
        p.feas[grp] = cand_ok ? 1 : 0;
    }

    // per-scenario deltas d_s = val_s(b,t) - val_s(b,a[b]): expected (np.mean) and CVaR10
    if constexpr (KC > 0) {
        if (p.exp_delta || p.cvar || p.scen_delta) {
            const int S = p.S;
            const double *vrow = p.vmax + (size_t)b * p.Sp;
            const int abc = (ab >= 0 && ab < T) ? ab : 0;
            const double d_ab = __ldg(p.disc + abc);
            const double dc_ab = net ? f64_mul(d_ab, __ldg(p.cost + (size_t)b * T + abc)) : 0.0;
#pragma unroll
            for (int k = 0; k < PER; k++) {
                const int t = tl + k * G;
                const int tc = (t < T) ? t : 0;
                const bool ok = ok_t[k];
                const double dc_t = net ? f64_mul(d_t[k], c_t[k]) : 0.0;
                PwStream acc;
                acc.begin(p.plan);
                TopK<KC> tk;
                tk.init();
                for (int s0 = 0; s0 < S; s0 += 32) {
                    __syncwarp();
                    if (ab >= 0) {
                        for (int j = tl; j < 32 && s0 + j < S; j += G) {
                            const int s = s0 + j;
                            double v = f64_mul(f64_mul(f64_mul(__ldg(vrow + s), d_ab), __ldg(p.sigma + (size_t)s * T + abc)),
                                               row.spatial);
                            if (net) v = f64_sub(v, dc_ab);
                            s_old[gl][j] = v;
                        }
                    }
                    __syncwarp();
                    if (ok) {
                        const int s_end = min(s0 + 32, S);
                        for (int s8 = s0; s8 < s_end; s8 += 8) {
                            double x[8];
#pragma unroll
                            for (int j = 0; j < 8; j++) {
                                const int s = s8 + j;
                                double dlt = 0.0;
                                if (s < s_end) {
                                    double v = f64_mul(f64_mul(f64_mul(__ldg(vrow + s), d_t[k]),
                                                               __ldg(p.sigma + (size_t)s * T + tc)),
                                                       row.spatial);
                                    if (net) v = f64_sub(v, dc_t);
                                    dlt = (ab >= 0) ? f64_sub(v, s_old[gl][s - s0]) : v;
                                    tk.push(dlt);
                                    if (p.scen_delta) p.scen_delta[((size_t)grp * S + s) * T + t] = (float)dlt;
                                }
                                x[j] = dlt;
                            }
                            acc.block(s8, x, min(8, s_end - s8), p.plan);
                        }
                    }
                }
                if (active && t < T) {
                    const size_t m = (size_t)grp * T + t;
                    if (ok) {
                        if (p.exp_delta) p.exp_delta[m] = acc.mean(p.plan);
                        if (p.cvar) p.cvar[m] = tk.mean(p.cvar_k);
                    } else {
                        if (p.exp_delta) p.exp_delta[m] = -kInf;
                        if (p.cvar) p.cvar[m] = -kInf;
                        if (p.scen_delta)
                            for (int s = 0; s < S; s++) p.scen_delta[((size_t)grp * S + s) * T + t] = -__int_as_float(0x7f800000);
                    }
                }
            }
        }
    }

    // K4: grid argmax over candidates (one entry per group, from its lane 0)
    Best cb{-kInf, INT_MAX, INT_MAX};
    if (active && tl == 0 && cand_ok) cb = Best{mine.v, b, mine.t};
    grid_argmax(cb, s_red, p.partial, p.counter, p.global);
}

// ------------------------------------------------------------------------------------
// explicit moves (reassign / unmine / swap), one thread per move
// ------------------------------------------------------------------------------------
struct MoveParams {
    const BlockRow *rows;
    const int32_t *adj;
    const int32_t *assign;
    const double *pm;
    const double *cap;
    const double *disc;
    const double *cost;
    const double *vmax;
    const double *unit_mean;
    const double *sig_row;
    const double *sigma;
    const int32_t *ma;
    const int32_t *mb;
    int M, B, T, S, Sp, scen, cvar_k, kind;
    unsigned flags;
    const int *plan;
    uint8_t *feas;
    double *delta;
    double *exp_delta;
    double *cvar;
    float *scen_delta;
    pp_best *partial;
    unsigned int *counter;
    pp_best *global;
};

__device__ __forceinline__ double kernel_value(const MoveParams &p, const BlockRow &r, int b, int t) {
    double unit;
    if (p.flags & PP_LITERAL_VALUE) unit = f64_mul(r.mass, 100.0);
    else if (p.scen < 0) unit = __ldg(p.unit_mean + b);
    else unit = __ldg(p.vmax + (size_t)b * p.Sp + p.scen);
    double d = __ldg(p.disc + t);
    double v = f64_mul(f64_mul(f64_mul(unit, d), __ldg(p.sig_row + t)), r.spatial);
    if (p.flags & PP_NET_MINING_COST) v = f64_sub(v, f64_mul(d, __ldg(p.cost + (size_t)b * p.T + t)));
    return v;
}

__device__ __forceinline__ double scen_value(const MoveParams &p, const BlockRow &r, int b, int t, int s) {
    double d = __ldg(p.disc + t);
    double v = f64_mul(f64_mul(f64_mul(__ldg(p.vmax + (size_t)b * p.Sp + s), d), __ldg(p.sigma + (size_t)s * p.T + t)),
                    r.spatial);
    if (p.flags & PP_NET_MINING_COST) v = f64_sub(v, f64_mul(d, __ldg(p.cost + (size_t)b * p.T + t)));
    return v;
}

// window(b) of hybrid.py:348-355 with block `ob` seen at period `ot`; lo = -2 encodes None
__device__ __forceinline__ void move_window(const MoveParams &p, const BlockRow &r, int ob, int ot, int &lo,
                                            int &hi) {
    const int npred = r.cnt & 0xffff, nnb = npred + (r.cnt >> 16);
    int l = 0, h = p.T - 1;
    bool none = false;
    for (int k = 0; k < nnb; k++) {
        int nb = __ldg(p.adj + r.adj + k);
        int tn = (nb == ob) ? ot : p.assign[nb];
        if (k < npred) {
            if (tn < 0) none = true;
            else l = max(l, tn);
        } else if (tn >= 0) {
            h = min(h, tn);
        }
    }
    lo = none ? -2 : l;
    hi = h;
}

template <int KC>
__global__ void __launch_bounds__(EV_THREADS) k_eval_moves(const MoveParams p) {
    __shared__ Best s_red[EV_THREADS / 32];
    const int i = blockIdx.x * EV_THREADS + threadIdx.x;
    const bool active = i < p.M;
    bool ok = false;
    double dl = -kInf;
    int b1 = 0, b2 = 0, t1 = -1, t2 = -1;
    BlockRow r1, r2;
    if (active) {
        const int x = p.ma[i], y = p.mb[i];
        if (p.kind == PP_MOVE_REASSIGN) {
            if (x >= 0 && x < p.B && y >= -1 && y < p.T) {
                b1 = x;
                r1 = p.rows[b1];
                t1 = p.assign[b1];  // old period
                t2 = y;             // new period
                const int npred = r1.cnt & 0xffff, nnb = npred + (r1.cnt >> 16);
                if (t2 == t1) {
                    ok = false;
                } else if (t2 < 0) {  // unmine: allowed iff mined and no mined successor
                    ok = true;
                    for (int k = npred; k < nnb; k++)
                        if (p.assign[__ldg(p.adj + r1.adj + k)] >= 0) ok = false;
                } else {
                    ok = true;
                    for (int k = 0; k < nnb; k++) {
                        int tn = p.assign[__ldg(p.adj + r1.adj + k)];
                        if (k < npred) {
                            if (tn < 0 || tn > t2) ok = false;
                        } else if (tn >= 0 && tn < t2) {
                            ok = false;
                        }
                    }
                    if (ok) {
                        double load = f64_add(p.pm[t2], r1.mass);
                        if (load > __ldg(p.cap + t2)) ok = false;
                    }
                }
                if (ok) {
                    double vn = (t2 >= 0) ? kernel_value(p, r1, b1, t2) : 0.0;
                    double vo = (t1 >= 0) ? kernel_value(p, r1, b1, t1) : 0.0;
                    dl = f64_sub(vn, vo);
                }
            }
        } else {
            if (x >= 0 && x < p.B && y >= 0 && y < p.B && x != y) {
                b1 = x;
                b2 = y;
                r1 = p.rows[b1];
                r2 = p.rows[b2];
                t1 = p.assign[b1];
                t2 = p.assign[b2];
                if (t1 >= 0 && t2 >= 0 && t1 != t2) {
                    double l1 = f64_add(f64_sub(p.pm[t1], r1.mass), r2.mass);
                    double l2 = f64_add(f64_sub(p.pm[t2], r2.mass), r1.mass);
                    if (!(l1 > __ldg(p.cap + t1)) && !(l2 > __ldg(p.cap + t2))) {
                        int lo1, hi1, lo2, hi2;
                        move_window(p, r1, b2, t1, lo1, hi1);
                        move_window(p, r2, b1, t2, lo2, hi2);
                        ok = lo1 != -2 && lo1 <= t2 && t2 <= hi1 && lo2 != -2 && lo2 <= t1 && t1 <= hi2;
                    }
                }
                if (ok) {
                    double v12 = kernel_value(p, r1, b1, t2), v11 = kernel_value(p, r1, b1, t1);
                    double v21 = kernel_value(p, r2, b2, t1), v22 = kernel_value(p, r2, b2, t2);
                    dl = f64_add(f64_sub(v12, v11), f64_sub(v21, v22));
                }
            }
        }
        p.feas[i] = ok ? 1 : 0;
        p.delta[i] = dl;
    }
    if constexpr (KC > 0) {
        if (active && (p.exp_delta || p.cvar || p.scen_delta)) {
            const int S = p.S;
            if (ok) {
                PwStream acc;
                acc.begin(p.plan);
                TopK<KC> tk;
                tk.init();
                for (int s8 = 0; s8 < S; s8 += 8) {
                    double x[8];
#pragma unroll
                    for (int j = 0; j < 8; j++) {
                        const int s = s8 + j;
                        double ds = 0.0;
                        if (s < S) {
                            if (p.kind == PP_MOVE_REASSIGN) {
                                ds = (t2 >= 0) ? scen_value(p, r1, b1, t2, s) : 0.0;
                                if (t1 >= 0) ds = f64_sub(ds, scen_value(p, r1, b1, t1, s));
                            } else {
                                ds = f64_add(f64_sub(scen_value(p, r1, b1, t2, s), scen_value(p, r1, b1, t1, s)),
                                             f64_sub(scen_value(p, r2, b2, t1, s), scen_value(p, r2, b2, t2, s)));
                            }
                            tk.push(ds);
                            if (p.scen_delta) p.scen_delta[(size_t)i * S + s] = (float)ds;
                        }
                        x[j] = ds;
                    }
                    acc.block(s8, x, min(8, S - s8), p.plan);
                }
                if (p.exp_delta) p.exp_delta[i] = acc.mean(p.plan);
                if (p.cvar) p.cvar[i] = tk.mean(p.cvar_k);
            } else {
                if (p.exp_delta) p.exp_delta[i] = -kInf;
                if (p.cvar) p.cvar[i] = -kInf;
                if (p.scen_delta)
                    for (int s = 0; s < S; s++) p.scen_delta[(size_t)i * S + s] = -__int_as_float(0x7f800000);
            }
        }
    }
    Best mine{-kInf, INT_MAX, INT_MAX};
    if (active && ok) mine = Best{dl, i, -1};
    grid_argmax(mine, s_red, p.partial, p.counter, p.global);
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

// sigma.mean(axis=0) sequentially over s (evaluate.py:351)
__global__ void k_sig_mean(const double *sigma, int S, int T, double *out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= T) return;
    double acc = 0.0;
    for (int s = 0; s < S; s++) acc = f64_add(acc, sigma[(size_t)s * T + t]);
    out[t] = f64_div(acc, (double)S);
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

// ------------------------------------------------------------------------------------
// host side: context
// ------------------------------------------------------------------------------------
struct DevBuf {
    void *ptr = nullptr;
    size_t bytes = 0;
    int ensure(size_t need) {
        if (need <= bytes) return PP_OK;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
        size_t n = std::max<size_t>(need, 256);
        CUDA_TRY(cudaMalloc(&ptr, n));
        bytes = n;
        return PP_OK;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
    }
    template <class T>
    T *as() const {
        return reinterpret_cast<T *>(ptr);
    }
};

struct pp_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int B = 0, T = 0, S = 0, Sp = 0, n_levels = 0;
    long long E = 0;
    bool have_instance = false, have_spatial = false, have_scen = false, have_sigma = false, have_sched = false;
    double mean_cap = 0.0;
    std::vector<int> level_ptr;  // host, n_levels + 1
    std::vector<int> level_of;   // host, B
    PwPlan plan{};
    int cvar_k = 1;
    // static tables
    DevBuf rows, adj, cost, cap, disc, level_blocks, ones_t;
    DevBuf vmax, unit_mean, sigma, sig_mean, ones_st, plan_dev;
    // schedule
    DevBuf assign, pm;
    // scratch
    DevBuf cnt, compact, pm_batch, predcnt, partial, counter;
    DevBuf h_cand, h_a, h_b, h_o1, h_o2, h_o3, h_o4, h_o5, h_o6, h_o7, h_o8, h_glob, h_assign, h_i64, h_d1, h_d2,
        h_pm;
    std::vector<DevBuf *> all() {
        return {&rows, &adj, &cost, &cap, &disc, &level_blocks, &ones_t, &vmax, &unit_mean, &sigma, &sig_mean,
                &ones_st, &plan_dev, &assign, &pm, &cnt, &compact, &pm_batch, &predcnt, &partial, &counter, &h_cand, &h_a,
                &h_b, &h_o1, &h_o2, &h_o3, &h_o4, &h_o5, &h_o6, &h_o7, &h_o8, &h_glob, &h_assign, &h_i64, &h_d1,
                &h_d2, &h_pm};
    }
};

static int use_device(pp_ctx *c) {
    CUDA_TRY(cudaSetDevice(c->device));
    return PP_OK;
}

static cudaStream_t pick(pp_ctx *c, void *stream) { return stream ? (cudaStream_t)stream : c->stream; }

// host copy of numpy's pairwise sum (for np.mean(capacity), evaluate.py:103)
static double host_pairwise(const double *a, long n) {
    if (n < 8) {
        double r = -0.0;
        for (long i = 0; i < n; i++) r += a[i];
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = a[j];
        long i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    }
    long n2 = n / 2;
    n2 -= n2 % 8;
    return host_pairwise(a, n2) + host_pairwise(a + n2, n - n2);
}

static int ensure_grid_scratch(pp_ctx *c, int grid) {
    TRY(c->partial.ensure(sizeof(pp_best) * (size_t)std::max(grid, 1)));
    if (c->counter.bytes == 0) {
        TRY(c->counter.ensure(sizeof(unsigned int) * 4));
        CUDA_TRY(cudaMemset(c->counter.ptr, 0, c->counter.bytes));
    }
    return PP_OK;
}

// period masses of P schedules (device pointers) into pm_out[P][T]
static int run_period_mass(pp_ctx *c, const int32_t *d_assign, int P, double *d_pm, cudaStream_t st) {
    const int B = c->B, T = c->T;
    const int nchunk = (B + PM_CHUNK - 1) / PM_CHUNK;
    TRY(c->cnt.ensure(sizeof(int32_t) * (size_t)P * nchunk * T));
    TRY(c->compact.ensure(sizeof(double) * (size_t)P * B));
    dim3 g(nchunk, P);
    k_pm_count<<<g, PM_THREADS, 0, st>>>(d_assign, B, T, nchunk, c->cnt.as<int32_t>());
    k_pm_scatter<<<g, PM_THREADS, 0, st>>>(d_assign, c->rows.as<BlockRow>(), B, T, nchunk, c->cnt.as<int32_t>(),
                                           c->compact.as<double>());
    k_pm_leaf<<<dim3(T, P), PM_THREADS, 0, st>>>(c->compact.as<double>(), c->cnt.as<int32_t>(), B, T, nchunk, d_pm);
    CUDA_TRY(cudaGetLastError());
    return PP_OK;
}

extern "C" {

int pp_abi_version(void) { return PP_ABI_VERSION; }

const char *pp_last_error(void) { return g_last_error.c_str(); }

int pp_device_count(int *count) {
    if (!count) return fail(PP_ERR_INVALID_ARGS, "count is NULL");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        *count = 0;
        return fail(PP_ERR_CUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
    }
    *count = n;
    return PP_OK;
}

int pp_ctx_create(int device, pp_ctx **out) {
    if (!out) return fail(PP_ERR_INVALID_ARGS, "out is NULL");
    *out = nullptr;
    int n = 0;
    TRY(pp_device_count(&n));
    if (device < 0 || device >= n) return fail(PP_ERR_INVALID_ARGS, "device %d out of range (%d devices)", device, n);
    pp_ctx *c = new (std::nothrow) pp_ctx();
    if (!c) return fail(PP_ERR_CUDA, "out of host memory");
    c->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return fail(PP_ERR_CUDA, "context init: %s", cudaGetErrorString(e));
    }
    *out = c;
    return PP_OK;
}

int pp_ctx_destroy(pp_ctx *c) {
    if (!c) return PP_OK;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (DevBuf *b : c->all()) b->release();
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
    return PP_OK;
}

int pp_ctx_stream(pp_ctx *c, void **stream) {
    if (!c || !stream) return fail(PP_ERR_INVALID_ARGS, "NULL argument");
    *stream = (void *)c->stream;
    return PP_OK;
}

int pp_synchronize(pp_ctx *c, void *stream) {
    if (!c) return fail(PP_ERR_INVALID_ARGS, "NULL context");
    TRY(use_device(c));
    CUDA_TRY(cudaStreamSynchronize(pick(c, stream)));
    return PP_OK;
}

int pp_host_alloc(size_t bytes, void **ptr) {
    if (!ptr) return fail(PP_ERR_INVALID_ARGS, "ptr is NULL");
    CUDA_TRY(cudaHostAlloc(ptr, std::max<size_t>(bytes, 1), cudaHostAllocPortable));
    return PP_OK;
}

int pp_host_free(void *ptr) {
    if (ptr) CUDA_TRY(cudaFreeHost(ptr));
    return PP_OK;
}

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
    TRY(c->pm.ensure(sizeof(double) * T));
    std::vector<double> ones(T, 1.0);
    CUDA_TRY(cudaMemcpy(c->rows.ptr, rows.data(), sizeof(BlockRow) * B, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(c->adj.ptr, adj.data(), sizeof(int) * adj.size(), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(c->cost.ptr, cost, sizeof(double) * (size_t)B * T, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(c->cap.ptr, capacity, sizeof(double) * T, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(c->disc.ptr, discount, sizeof(double) * T, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(c->ones_t.ptr, ones.data(), sizeof(double) * T, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(c->level_blocks.ptr, lblocks.data(), sizeof(int) * B, cudaMemcpyHostToDevice));
    c->B = B;
    c->T = T;
    c->E = E;
    c->n_levels = nlev;
    c->level_ptr = lptr;
    c->level_of = level;
    c->mean_cap = (0.0 + host_pairwise(capacity, T)) / (double)T;
    c->have_instance = true;
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
    cudaError_t e = cudaMemcpy(d, alt, sizeof(double) * B, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d + B, strc, sizeof(double) * B, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d + 2 * (size_t)B, dist, sizeof(double) * B, cudaMemcpyHostToDevice);
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

int pp_set_scenarios(pp_ctx *c, int32_t S, const double *vmax_sb, const double *sigma_st) {
    if (!c || !c->have_instance) return fail(PP_ERR_STATE, "pp_set_instance first");
    if (S < 1 || !vmax_sb) return fail(PP_ERR_INVALID_ARGS, "need n_scenarios >= 1 and a value table");
    TRY(use_device(c));
    PwPlan plan;
    TRY(make_plan(S, &plan));
    const int B = c->B, T = c->T;
    const int Sp = (S + 3) & ~3;
    TRY(c->vmax.ensure(sizeof(double) * (size_t)B * Sp));
    TRY(c->unit_mean.ensure(sizeof(double) * B));
    TRY(c->sigma.ensure(sizeof(double) * (size_t)S * T));
    TRY(c->ones_st.ensure(sizeof(double) * (size_t)S * T));
    TRY(c->sig_mean.ensure(sizeof(double) * T));
    TRY(c->plan_dev.ensure(sizeof(int) * kPlanWords));
    DevBuf tmp;
    TRY(tmp.ensure(sizeof(double) * (size_t)S * B));
    cudaError_t e = cudaMemcpy(tmp.ptr, vmax_sb, sizeof(double) * (size_t)S * B, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        k_scen_tables<<<(B + 255) / 256, 256, 0, c->stream>>>(tmp.as<double>(), S, B, Sp, c->vmax.as<double>(),
                                                              c->unit_mean.as<double>());
        e = cudaGetLastError();
    }
    std::vector<double> ones((size_t)S * T, 1.0);
    int words[kPlanWords];
    plan_words(plan, words);
    if (e == cudaSuccess) e = cudaMemcpy(c->plan_dev.ptr, words, sizeof(words), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(c->ones_st.ptr, ones.data(), sizeof(double) * ones.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && sigma_st) {
        e = cudaMemcpy(c->sigma.ptr, sigma_st, sizeof(double) * (size_t)S * T, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) {
            k_sig_mean<<<(T + 127) / 128, 128, 0, c->stream>>>(c->sigma.as<double>(), S, T, c->sig_mean.as<double>());
            e = cudaGetLastError();
        }
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    tmp.release();
    if (e != cudaSuccess) return fail(PP_ERR_CUDA, "pp_set_scenarios: %s", cudaGetErrorString(e));
    c->S = S;
    c->Sp = Sp;
    c->plan = plan;
    c->cvar_k = std::max(1, (int)std::ceil(0.1 * S));
    c->have_sigma = sigma_st != nullptr;
    c->have_scen = true;
    return PP_OK;
}

int pp_set_schedule(pp_ctx *c, const int32_t *assign, int32_t mem, void *stream) {
    if (!c || !c->have_instance) return fail(PP_ERR_STATE, "pp_set_instance first");
    if (!assign) return fail(PP_ERR_INVALID_ARGS, "assign is NULL");
    TRY(use_device(c));
    cudaStream_t st = pick(c, stream);
    CUDA_TRY(cudaMemcpyAsync(c->assign.ptr, assign, sizeof(int32_t) * c->B,
                             mem == PP_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
    TRY(run_period_mass(c, c->assign.as<int32_t>(), 1, c->pm.as<double>(), st));
    if (mem == PP_MEM_HOST) CUDA_TRY(cudaStreamSynchronize(st));
    c->have_sched = true;
    return PP_OK;
}

int pp_apply_moves(pp_ctx *c, const int32_t *blocks, const int32_t *periods, int32_t n, int32_t mem, void *stream) {
    if (!c || !c->have_sched) return fail(PP_ERR_STATE, "pp_set_schedule first");
    if (n < 0 || (n > 0 && (!blocks || !periods))) return fail(PP_ERR_INVALID_ARGS, "bad move arrays");
    TRY(use_device(c));
    cudaStream_t st = pick(c, stream);
    if (n == 0) return PP_OK;
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
    TRY(run_period_mass(c, c->assign.as<int32_t>(), 1, c->pm.as<double>(), st));
    if (mem == PP_MEM_HOST) CUDA_TRY(cudaStreamSynchronize(st));
    return PP_OK;
}

int pp_get_schedule(pp_ctx *c, int32_t *assign_out, double *pm_out, int32_t mem, void *stream) {
    if (!c || !c->have_sched) return fail(PP_ERR_STATE, "pp_set_schedule first");
    TRY(use_device(c));
    cudaStream_t st = pick(c, stream);
    cudaMemcpyKind k = (mem == PP_MEM_HOST) ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    if (assign_out) CUDA_TRY(cudaMemcpyAsync(assign_out, c->assign.ptr, sizeof(int32_t) * c->B, k, st));
    if (pm_out) CUDA_TRY(cudaMemcpyAsync(pm_out, c->pm.ptr, sizeof(double) * c->T, k, st));
    if (mem == PP_MEM_HOST) CUDA_TRY(cudaStreamSynchronize(st));
    return PP_OK;
}

}  // extern "C"

static int pick_kc(int k) {
    if (k <= 4) return 4;
    if (k <= 128) return 128;
    return -1;
}

template <int PER>
static void launch_cand_kc(int kc, int grid, int G, cudaStream_t st, const EvalParams &ep) {
    switch (kc) {
        case 0: k_eval_candidates<PER, 0><<<grid, EV_THREADS, 0, st>>>(ep, G); break;
        case 4: k_eval_candidates<PER, 4><<<grid, EV_THREADS, 0, st>>>(ep, G); break;
        default: k_eval_candidates<PER, 128><<<grid, EV_THREADS, 0, st>>>(ep, G); break;
    }
}

static int check_ready(pp_ctx *c, uint32_t flags, int scenario) {
    if (!c) return fail(PP_ERR_INVALID_ARGS, "NULL context");
    if (!c->have_instance || !c->have_spatial) return fail(PP_ERR_STATE, "pp_set_instance and pp_set_geology first");
    if (!c->have_sched) return fail(PP_ERR_STATE, "pp_set_schedule first");
    if (!c->have_scen && !(flags & PP_LITERAL_VALUE)) return fail(PP_ERR_STATE, "pp_set_scenarios first");
    if ((flags & PP_USE_SIGMA) && !c->have_sigma) return fail(PP_ERR_STATE, "PP_USE_SIGMA without an uploaded sigma");
    if (scenario < -1 || (c->have_scen && scenario >= c->S) || (!c->have_scen && scenario >= 0))
        return fail(PP_ERR_INVALID_ARGS, "scenario %d out of range", scenario);
    return PP_OK;
}

extern "C" {

int pp_eval_candidates(pp_ctx *c, const int32_t *cand, int32_t C, int32_t scenario, uint32_t flags,
                       const pp_cand_out *out, int32_t mem, void *stream) {
    TRY(check_ready(c, flags, scenario));
    if (C < 0 || (C > 0 && !cand)) return fail(PP_ERR_INVALID_ARGS, "bad candidate array");
    if (!out || !out->best_t || !out->best_val || !out->feasible || !out->global)
        return fail(PP_ERR_INVALID_ARGS, "best_t, best_val, feasible and global outputs are required");
    const bool stats = out->exp_delta || out->cvar || out->scen_delta;
    if (stats && !c->have_scen) return fail(PP_ERR_STATE, "scenario statistics need pp_set_scenarios");
    TRY(use_device(c));
    cudaStream_t st = pick(c, stream);
    const int T = c->T, S = c->S;
    int G, PER = 1;
    if (T <= 4) G = 4;
    else if (T <= 8) G = 8;
    else if (T <= 16) G = 16;
    else if (T <= 32) G = 32;
    else {
        G = 32;
        PER = 4;
    }
    const int gpc = (EV_THREADS / 32) * (32 / G);
    const int grid = std::max(1, (C + gpc - 1) / gpc);
    TRY(ensure_grid_scratch(c, grid));
    const int kc = stats ? pick_kc(c->cvar_k) : 0;
    if (kc < 0) return fail(PP_ERR_INVALID_ARGS, "CVaR sample count %d too large", c->cvar_k);

    pp_cand_out o = *out;
    const int32_t *dcand = cand;
    if (mem == PP_MEM_HOST) {
        for (int i = 0; i < C; i++)
            if (cand[i] < 0 || cand[i] >= c->B) return fail(PP_ERR_INVALID_ARGS, "candidate block %d out of range", cand[i]);
        const size_t Cs = (size_t)std::max(C, 1), CT = Cs * T;
        TRY(c->h_cand.ensure(sizeof(int32_t) * Cs));
        TRY(c->h_o1.ensure(sizeof(int32_t) * Cs));
        TRY(c->h_o2.ensure(sizeof(double) * Cs));
        TRY(c->h_o3.ensure(Cs));
        TRY(c->h_glob.ensure(sizeof(pp_best)));
        o.best_t = c->h_o1.as<int32_t>();
        o.best_val = c->h_o2.as<double>();
        o.feasible = c->h_o3.as<uint8_t>();
        o.global = c->h_glob.as<pp_best>();
        if (out->trace_val) { TRY(c->h_o4.ensure(sizeof(double) * CT)); o.trace_val = c->h_o4.as<double>(); }
        if (out->trace_feas) { TRY(c->h_o5.ensure(CT)); o.trace_feas = c->h_o5.as<uint8_t>(); }
        if (out->exp_delta) { TRY(c->h_o6.ensure(sizeof(double) * CT)); o.exp_delta = c->h_o6.as<double>(); }
        if (out->cvar) { TRY(c->h_o7.ensure(sizeof(double) * CT)); o.cvar = c->h_o7.as<double>(); }
        if (out->scen_delta) { TRY(c->h_o8.ensure(sizeof(float) * CT * std::max(S, 1))); o.scen_delta = c->h_o8.as<float>(); }
        if (C > 0) CUDA_TRY(cudaMemcpyAsync(c->h_cand.ptr, cand, sizeof(int32_t) * C, cudaMemcpyHostToDevice, st));
        dcand = c->h_cand.as<int32_t>();
    }

    EvalParams ep;
    memset(&ep, 0, sizeof(ep));
    ep.rows = c->rows.as<BlockRow>();
    ep.adj = c->adj.as<int32_t>();
    ep.assign = c->assign.as<int32_t>();
    ep.pm = c->pm.as<double>();
    ep.cap = c->cap.as<double>();
    ep.disc = c->disc.as<double>();
    ep.cost = c->cost.as<double>();
    ep.vmax = c->have_scen ? c->vmax.as<double>() : nullptr;
    ep.unit_mean = c->have_scen ? c->unit_mean.as<double>() : nullptr;
    if (!(flags & PP_USE_SIGMA)) ep.sig_row = c->ones_t.as<double>();
    else if (scenario < 0) ep.sig_row = c->sig_mean.as<double>();
    else ep.sig_row = c->sigma.as<double>() + (size_t)scenario * T;
    ep.sigma = (flags & PP_USE_SIGMA) ? c->sigma.as<double>() : c->ones_st.as<double>();
    ep.cand = dcand;
    ep.C = C;
    ep.B = c->B;
    ep.T = T;
    ep.S = S;
    ep.Sp = c->Sp;
    ep.scen = scenario;
    ep.cvar_k = c->cvar_k;
    ep.flags = flags;
    ep.plan = c->plan_dev.as<int>();
    ep.best_t = o.best_t;
    ep.best_val = o.best_val;
    ep.feas = o.feasible;
    ep.trace_val = o.trace_val;
    ep.trace_feas = o.trace_feas;
    ep.exp_delta = o.exp_delta;
    ep.cvar = o.cvar;
    ep.scen_delta = o.scen_delta;
    ep.partial = c->partial.as<pp_best>();
    ep.counter = c->counter.as<unsigned int>();
    ep.global = o.global;

    if (PER == 1) launch_cand_kc<1>(kc, grid, G, st, ep);
    else launch_cand_kc<4>(kc, grid, G, st, ep);
    CUDA_TRY(cudaGetLastError());

    if (mem == PP_MEM_HOST) {
        const size_t Cs = (size_t)C, CT = Cs * T;
        CUDA_TRY(cudaMemcpyAsync(out->global, o.global, sizeof(pp_best), cudaMemcpyDeviceToHost, st));
        if (C > 0) {
            CUDA_TRY(cudaMemcpyAsync(out->best_t, o.best_t, sizeof(int32_t) * Cs, cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaMemcpyAsync(out->best_val, o.best_val, sizeof(double) * Cs, cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaMemcpyAsync(out->feasible, o.feasible, Cs, cudaMemcpyDeviceToHost, st));
            if (out->trace_val) CUDA_TRY(cudaMemcpyAsync(out->trace_val, o.trace_val, sizeof(double) * CT, cudaMemcpyDeviceToHost, st));
            if (out->trace_feas) CUDA_TRY(cudaMemcpyAsync(out->trace_feas, o.trace_feas, CT, cudaMemcpyDeviceToHost, st));
            if (out->exp_delta) CUDA_TRY(cudaMemcpyAsync(out->exp_delta, o.exp_delta, sizeof(double) * CT, cudaMemcpyDeviceToHost, st));
            if (out->cvar) CUDA_TRY(cudaMemcpyAsync(out->cvar, o.cvar, sizeof(double) * CT, cudaMemcpyDeviceToHost, st));
            if (out->scen_delta)
                CUDA_TRY(cudaMemcpyAsync(out->scen_delta, o.scen_delta, sizeof(float) * CT * S, cudaMemcpyDeviceToHost, st));
        }
        CUDA_TRY(cudaStreamSynchronize(st));
    }
    return PP_OK;
}

int pp_eval_moves(pp_ctx *c, int32_t kind, const int32_t *a, const int32_t *b, int32_t M, int32_t scenario,
                  uint32_t flags, const pp_move_out *out, int32_t mem, void *stream) {
    TRY(check_ready(c, flags, scenario));
    if (kind != PP_MOVE_REASSIGN && kind != PP_MOVE_SWAP) return fail(PP_ERR_INVALID_ARGS, "unknown move kind %d", kind);
    if (M < 0 || (M > 0 && (!a || !b))) return fail(PP_ERR_INVALID_ARGS, "bad move arrays");
    if (!out || !out->feasible || !out->delta || !out->global)
        return fail(PP_ERR_INVALID_ARGS, "feasible, delta and global outputs are required");
    const bool stats = out->exp_delta || out->cvar || out->scen_delta;
    if (stats && !c->have_scen) return fail(PP_ERR_STATE, "scenario statistics need pp_set_scenarios");
    TRY(use_device(c));
    cudaStream_t st = pick(c, stream);
    const int T = c->T, S = c->S;
    const int grid = std::max(1, (M + EV_THREADS - 1) / EV_THREADS);
    TRY(ensure_grid_scratch(c, grid));
    const int kc = stats ? pick_kc(c->cvar_k) : 0;
    if (kc < 0) return fail(PP_ERR_INVALID_ARGS, "CVaR sample count %d too large", c->cvar_k);
    pp_move_out o = *out;
    const int32_t *da = a, *db = b;
    if (mem == PP_MEM_HOST) {
        const size_t Ms = (size_t)std::max(M, 1);
        TRY(c->h_a.ensure(sizeof(int32_t) * Ms));
        TRY(c->h_b.ensure(sizeof(int32_t) * Ms));
        TRY(c->h_o3.ensure(Ms));
        TRY(c->h_o2.ensure(sizeof(double) * Ms));
        TRY(c->h_glob.ensure(sizeof(pp_best)));
        o.feasible = c->h_o3.as<uint8_t>();
        o.delta = c->h_o2.as<double>();
        o.global = c->h_glob.as<pp_best>();
        if (out->exp_delta) { TRY(c->h_o6.ensure(sizeof(double) * Ms)); o.exp_delta = c->h_o6.as<double>(); }
        if (out->cvar) { TRY(c->h_o7.ensure(sizeof(double) * Ms)); o.cvar = c->h_o7.as<double>(); }
        if (out->scen_delta) { TRY(c->h_o8.ensure(sizeof(float) * Ms * std::max(S, 1))); o.scen_delta = c->h_o8.as<float>(); }
        if (M > 0) {
            CUDA_TRY(cudaMemcpyAsync(c->h_a.ptr, a, sizeof(int32_t) * M, cudaMemcpyHostToDevice, st));
            CUDA_TRY(cudaMemcpyAsync(c->h_b.ptr, b, sizeof(int32_t) * M, cudaMemcpyHostToDevice, st));
        }
        da = c->h_a.as<int32_t>();
        db = c->h_b.as<int32_t>();
    }
    MoveParams mp;
    memset(&mp, 0, sizeof(mp));
    mp.rows = c->rows.as<BlockRow>();
    mp.adj = c->adj.as<int32_t>();
    mp.assign = c->assign.as<int32_t>();
    mp.pm = c->pm.as<double>();
    mp.cap = c->cap.as<double>();
    mp.disc = c->disc.as<double>();
    mp.cost = c->cost.as<double>();
    mp.vmax = c->have_scen ? c->vmax.as<double>() : nullptr;
    mp.unit_mean = c->have_scen ? c->unit_mean.as<double>() : nullptr;
    if (!(flags & PP_USE_SIGMA)) mp.sig_row = c->ones_t.as<double>();
    else if (scenario < 0) mp.sig_row = c->sig_mean.as<double>();
    else mp.sig_row = c->sigma.as<double>() + (size_t)scenario * T;
    mp.sigma = (flags & PP_USE_SIGMA) ? c->sigma.as<double>() : c->ones_st.as<double>();
    mp.ma = da;
    mp.mb = db;
    mp.M = M;
    mp.B = c->B;
    mp.T = T;
    mp.S = S;
    mp.Sp = c->Sp;
    mp.scen = scenario;
    mp.cvar_k = c->cvar_k;
    mp.kind = kind;
    mp.flags = flags;
    mp.plan = c->plan_dev.as<int>();
    mp.feas = o.feasible;
    mp.delta = o.delta;
    mp.exp_delta = o.exp_delta;
    mp.cvar = o.cvar;
    mp.scen_delta = o.scen_delta;
    mp.partial = c->partial.as<pp_best>();
    mp.counter = c->counter.as<unsigned int>();
    mp.global = o.global;
    switch (kc) {
        case 0: k_eval_moves<0><<<grid, EV_THREADS, 0, st>>>(mp); break;
        case 4: k_eval_moves<4><<<grid, EV_THREADS, 0, st>>>(mp); break;
        default: k_eval_moves<128><<<grid, EV_THREADS, 0, st>>>(mp); break;
    }
    CUDA_TRY(cudaGetLastError());
    if (mem == PP_MEM_HOST) {
        const size_t Ms = (size_t)M;
        CUDA_TRY(cudaMemcpyAsync(out->global, o.global, sizeof(pp_best), cudaMemcpyDeviceToHost, st));
        if (M > 0) {
            CUDA_TRY(cudaMemcpyAsync(out->feasible, o.feasible, Ms, cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaMemcpyAsync(out->delta, o.delta, sizeof(double) * Ms, cudaMemcpyDeviceToHost, st));
            if (out->exp_delta) CUDA_TRY(cudaMemcpyAsync(out->exp_delta, o.exp_delta, sizeof(double) * Ms, cudaMemcpyDeviceToHost, st));
            if (out->cvar) CUDA_TRY(cudaMemcpyAsync(out->cvar, o.cvar, sizeof(double) * Ms, cudaMemcpyDeviceToHost, st));
            if (out->scen_delta)
                CUDA_TRY(cudaMemcpyAsync(out->scen_delta, o.scen_delta, sizeof(float) * Ms * S, cudaMemcpyDeviceToHost, st));
        }
        CUDA_TRY(cudaStreamSynchronize(st));
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

int pp_get_levels(pp_ctx *c, int32_t *n_levels, int32_t *level_of_block) {
    if (!c || !c->have_instance) return fail(PP_ERR_STATE, "pp_set_instance first");
    if (n_levels) *n_levels = c->n_levels;
    if (level_of_block) memcpy(level_of_block, c->level_of.data(), sizeof(int32_t) * c->B);
    return PP_OK;
}

}  // extern "C"
