// pp_internal.cuh -- shared device helpers, parameter blocks and the host context of the
// pitplan_b200 engine (included by every translation unit of the library).
#pragma once

#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "pitplan_b200.h"

// last-error channel of the C ABI (pp_context.cu)
int fail(int code, const char *fmt, ...);

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

// Device copy of a PwPlan: int words [n, nleaf, start[kMaxLeaves], len[kMaxLeaves], adds[kMaxLeaves]].
constexpr int kPlanWords = 2 + 3 * kMaxLeaves;

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
    // merge with the list of lane (lane ^ m): both lanes end with the KC smallest of the union,
    // ascending (values are only compared and moved, never combined)
    __device__ __forceinline__ void merge_xor(int m, unsigned mask = 0xffffffffu) {
        double o[KC];
#pragma unroll
        for (int j = 0; j < KC; j++) o[j] = __shfl_xor_sync(mask, a[j], m);
        double r[KC];
        int ia = 0, ib = 0;
#pragma unroll
        for (int j = 0; j < KC; j++) {
            double x = a[0], y = o[0];
#pragma unroll
            for (int u = 0; u < KC; u++) {
                if (u == ia) x = a[u];
                if (u == ib) y = o[u];
            }
            const bool ta = !(y < x);
            r[j] = ta ? x : y;
            ia += ta ? 1 : 0;
            ib += ta ? 0 : 1;
        }
#pragma unroll
        for (int j = 0; j < KC; j++) a[j] = r[j];
    }
    __device__ __forceinline__ void push(double x) {
        if constexpr (KC <= 8) {
            // branch-free (x >= a[KC-1], or NaN, leaves every entry as it was): straight-line code lets
            // the next scenario's value be formed while this push runs
            bool lt[KC];  // every comparison against the old list first: selects only, no branches
#pragma unroll
            for (int j = 0; j < KC; j++) lt[j] = x < a[j];
#pragma unroll
            for (int j = KC - 1; j > 0; j--) a[j] = lt[j - 1] ? a[j - 1] : (lt[j] ? x : a[j]);
            a[0] = lt[0] ? x : a[0];
        } else if (x < a[KC - 1]) {
            {  // insertion sort step in local memory
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
        } else if constexpr (KC <= 8) {  // k == 8 == KC: one block of eight; constant indices only,
                                          // so a[] stays in registers
            double r[8];
#pragma unroll
            for (int j = 0; j < 8; j++) r[j] = a[j < KC ? j : 0];
            s = tree8(r);
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
struct TopK<2> {  // k <= 2 (S <= 20): two registers, branch-free (lanes hold different moves)
    double a0, a1;
    __device__ __forceinline__ void init() { a0 = a1 = kInf; }
    __device__ __forceinline__ void merge_xor(int m, unsigned mask = 0xffffffffu) {
        const double b0 = __shfl_xor_sync(mask, a0, m), b1 = __shfl_xor_sync(mask, a1, m);
        // two smallest of {a0 <= a1} u {b0 <= b1}, ascending
        const bool ta = !(b0 < a0);
        const double lo = ta ? a0 : b0;
        const double n1 = ta ? a1 : a0, n2 = ta ? b0 : b1;  // the candidates for second place
        a0 = lo;
        a1 = (n2 < n1) ? n2 : n1;
    }
    __device__ __forceinline__ void push(double x) {
        // the same selections as "if (x < a1) { if (x < a0) { a1 = a0; a0 = x; } else a1 = x; }"
        const bool lt0 = x < a0;
        const double lo = lt0 ? x : a0, hi = lt0 ? a0 : x;
        a1 = (hi < a1) ? hi : a1;
        a0 = lo;
    }
    __device__ __forceinline__ double mean(int k) const {
        double s = f64_add(-0.0, a0);
        if (k > 1) s = f64_add(s, a1);
        // x / 1 and x / 2 are exact scalings: the multiply gives the same correctly rounded value
        return f64_mul(f64_add(0.0, s), k > 1 ? 0.5 : 1.0);
    }
};
template <>
struct TopK<0> {
    __device__ __forceinline__ void init() {}
    __device__ __forceinline__ void merge_xor(int, unsigned = 0xffffffffu) {}
    __device__ __forceinline__ void push(double) {}
    __device__ __forceinline__ double mean(int) const { return 0.0; }
};

// order-preserving map of a double onto u64 (NaN after +inf, as np.sort places it)
__device__ __forceinline__ unsigned long long f64_key(double v) {
    const unsigned long long u = (unsigned long long)__double_as_longlong(v);
    if (v != v) return ~0ull - 1ull;
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_f64(unsigned long long k) {
    return __longlong_as_double((long long)((k >> 63) ? (k ^ 0x8000000000000000ull) : ~k));
}
__device__ __forceinline__ void ce_u64(unsigned long long &a, unsigned long long &b) {
    const unsigned long long lo = a < b ? a : b, hi = a < b ? b : a;
    a = lo;
    b = hi;
}
// The k (<= 32) smallest of the warp's keys (lane l holds elements l + 32 r, r < npl <= 8; the
// rest are padding), ascending: a per-lane sorting network, then k rounds of a warp-wide minimum
// over the lane heads (redux.sync on the high word; the low word only on a tie) in which the
// winning lane pops its head (its sorted tail waits in scr, 32 x npl u64 of the warp's scratch).
// Returns the r-th smallest on lane r < k.
__device__ __forceinline__ double warp_k_smallest(unsigned long long (&k8)[8], int k, unsigned long long *scr,
                                                  int npl) {
    constexpr unsigned FULL = 0xffffffffu;
    ce_u64(k8[0], k8[1]); ce_u64(k8[2], k8[3]); ce_u64(k8[4], k8[5]); ce_u64(k8[6], k8[7]);
    ce_u64(k8[0], k8[2]); ce_u64(k8[1], k8[3]); ce_u64(k8[4], k8[6]); ce_u64(k8[5], k8[7]);
    ce_u64(k8[1], k8[2]); ce_u64(k8[5], k8[6]);
    ce_u64(k8[0], k8[4]); ce_u64(k8[1], k8[5]); ce_u64(k8[2], k8[6]); ce_u64(k8[3], k8[7]);
    ce_u64(k8[2], k8[4]); ce_u64(k8[3], k8[5]);
    ce_u64(k8[1], k8[2]); ce_u64(k8[3], k8[4]); ce_u64(k8[5], k8[6]);
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 2; i < 8; i++)
        if (i < npl) scr[i * 32 + lane] = k8[i];
    unsigned long long h0 = k8[0], h1 = k8[1], mine = ~0ull;
    int ptr = 2;
    for (int r = 0; r < k; r++) {
        const unsigned hi = (unsigned)(h0 >> 32), lo = (unsigned)h0;
        const unsigned mhi = __reduce_min_sync(FULL, hi);
        unsigned who = __ballot_sync(FULL, hi == mhi);
        if (__popc(who) > 1) {  // warp-uniform
            const unsigned mlo = __reduce_min_sync(FULL, hi == mhi ? lo : 0xffffffffu);
            who = __ballot_sync(FULL, hi == mhi && lo == mlo);
        }
        const int w = __ffs(who) - 1;
        const unsigned wlo = __shfl_sync(FULL, lo, w);
        if (lane == r) mine = ((unsigned long long)mhi << 32) | wlo;
        if (lane == w) {
            h0 = h1;
            h1 = ptr < npl ? scr[ptr * 32 + lane] : ~0ull;
            ptr++;
        }
    }
    return key_f64(mine);
}


// numpy pairwise mean over a warp's scratch vb[0..S) with the scenario plan P (<= kMaxLeaves leaves
// of <= 128 elements): eight lanes per leaf (accumulator j = lane & 7, xor butterfly = numpy's
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))), the leaf's tail in order, then lane 0 folds the leaves in
// the recursion's post-order.  lv: >= kMaxLeaves doubles of warp scratch.  Result on lane 0.
__device__ __forceinline__ double warp_pairwise_mean(const double *vb, const int *P, double *lv) {
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const int nleaf = __ldg(P + 1);
    for (int l0 = 0; l0 < nleaf; l0 += 4) {
        const int l = l0 + (lane >> 3), sub = lane & 7;
        const bool act = l < nleaf;
        const int ls = act ? __ldg(P + 2 + l) : 0, len = act ? __ldg(P + 2 + kMaxLeaves + l) : 0;
        const int nm = len >> 3;
        double acc = 0.0;
        if (nm > 0) {
            acc = vb[ls + sub];
            for (int u = 1; u < nm; u++) acc = f64_add(acc, vb[ls + 8 * u + sub]);
        }
        acc = f64_add(acc, __shfl_xor_sync(FULL, acc, 1));
        acc = f64_add(acc, __shfl_xor_sync(FULL, acc, 2));
        acc = f64_add(acc, __shfl_xor_sync(FULL, acc, 4));
        if (act && sub == 0) {
            double r = len >= 8 ? acc : -0.0;
            for (int i = len - (len & 7); i < len; i++) r = f64_add(r, vb[ls + i]);
            lv[l] = r;
        }
    }
    __syncwarp();
    double res = 0.0;
    if (lane == 0) {
        double stk[8];
        int sp_ = 0;
        for (int l = 0; l < nleaf; l++) {  // numpy's recursion, post-order
            stk[sp_++] = lv[l];
            const int nadd = __ldg(P + 2 + 2 * kMaxLeaves + l);
            for (int a = 0; a < nadd; a++) {
                const double rhs = stk[--sp_];
                const double lhs = stk[--sp_];
                stk[sp_++] = f64_add(lhs, rhs);
            }
        }
        res = f64_div(f64_add(0.0, stk[0]), (double)__ldg(P));
    }
    return res;
}

// CVaR10 (saa.py:157-164) of a warp's values vb[0..S) (S <= 32 * npl, npl <= 8): the mean of the
// kq <= 32 smallest in ascending order, numpy pairwise (8 accumulators, butterfly, tail).  `scr`:
// 32 * npl u64 of warp scratch (may alias nothing the caller still needs).  Result on every lane.
__device__ __forceinline__ double warp_cvar(const double *vb, int S, int kq, unsigned long long *scr, int npl) {
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    unsigned long long k8[8];
#pragma unroll
    for (int r = 0; r < 8; r++) {
        const int s_ = lane + 32 * r;
        k8[r] = (r < npl && s_ < S) ? f64_key(vb[s_]) : ~0ull;
    }
    __syncwarp();
    const double kv = warp_k_smallest(k8, kq, scr, npl);
    const int kn = kq >> 3;
    double cacc = (lane < 8 && kn > 0) ? kv : 0.0;  // lane l < 8: ranks l, 8 + l, ...
    for (int u = 1; u < kn; u++) {
        const double x = __shfl_sync(FULL, kv, (8 * u + lane) & 31);
        if (lane < 8) cacc = f64_add(cacc, x);
    }
    cacc = f64_add(cacc, __shfl_xor_sync(FULL, cacc, 1));
    cacc = f64_add(cacc, __shfl_xor_sync(FULL, cacc, 2));
    cacc = f64_add(cacc, __shfl_xor_sync(FULL, cacc, 4));
    double rc = kq >= 8 ? cacc : -0.0;
    for (int i = kq - (kq & 7); i < kq; i++) rc = f64_add(rc, __shfl_sync(FULL, kv, i));
    return f64_div(f64_add(0.0, rc), (double)kq);
}

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
static __device__ void grid_argmax(Best mine, Best *s_red, pp_best *partial, unsigned int *counter,
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


// Grid argmax when warp 0 already holds the CTA's candidates (lanes 0..31); every thread
// of the CTA must call it.  Same deterministic last-CTA reduction as grid_argmax.
static __device__ void grid_argmax_warp0(Best x, Best *s_red, pp_best *partial, unsigned int *counter,
                                         pp_best *global) {
    __shared__ bool s_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (warp == 0) {
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
    Best y{-kInf, INT_MAX, INT_MAX};
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
        const pp_best *q = partial + i;
        Best o{__ldcg(&q->value), __ldcg(&q->block), __ldcg(&q->period)};
        if (better(o, y)) y = o;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        Best o = shfl_best(y, off);
        if (better(o, y)) y = o;
    }
    if (lane == 0) s_red[warp] = y;
    __syncthreads();
    if (threadIdx.x == 0) {
        Best z = s_red[0];
        for (int w = 1; w < nw; w++)
            if (better(s_red[w], z)) z = s_red[w];
        pp_best g;
        bool none = (z.b == INT_MAX);
        g.value = none ? -kInf : z.v;
        g.block = none ? -1 : z.b;
        g.period = none ? -1 : z.t;
        *global = g;
        *counter = 0u;
    }
}

// ------------------------------------------------------------------------------------
// kernel parameter blocks
// ------------------------------------------------------------------------------------
struct EvalParams {
    const BlockRow *rows;
    const int32_t *adj;
    const int32_t *nbr;  // [B][nbr_stride]: predecessors then successors, padded to 16 bytes
    int nbr_stride;
    const int32_t *assign;
    const double *pm;
    const double *cap;
    const double *disc;
    const double *cost;      // [B][T]
    const double *vmax;      // [B][Sp]
    const double *unit_mean; // [B]
    const double *sig_row;   // [T] (ones / scenario mean / sigma[k])
    const double *sigma;     // [S][T] (ones if no sigma)
    const double *sigma_ts;  // [T][S]: sigma transposed (scenario-contiguous rows for lane = scenario)
    int wl[7];               // k_eval_warp: the per-warp shared-memory layout (host-computed)
    const int32_t *cand;
    int cand_host;           // cand is page-locked host memory (read once per CTA, k_eval_warp)
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
    int32_t *bad_cand;
    int32_t *pair_cand;
    int32_t *pair_period;
    double *pair_exp;
    double *pair_cvar;
    int32_t *n_pairs;
    pp_best *partial;
    unsigned int *counter;
    pp_best *global;
};

constexpr int EV_THREADS = 256;

struct MoveParams {
    const BlockRow *rows;
    const int32_t *adj;
    const int32_t *nbr;  // padded neighbour rows [B][32] (successors tagged 1 << 30), or null
    const int2 *bwin;    // every block's precedence window, 3 x int2 per block (k_block_windows), or null
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

// numpy pairwise sum of a[0..n) (pairwise.c: blocks of 8, leaves <= 128), whole CTA, result on
// thread 0: the leaves from the recursion on thread 0 (pre-order, i.e. element order) into
// ls/ll (capacity >= n/64 + 2), one thread per leaf with numpy's 8 accumulators into leafval[],
// the fold in post-order on thread 0.  `a`, ls, ll and leafval may live in shared or global memory.
template <class GF>
__device__ double s2_pairwise_f(GF a, int n, int *ls, int *ll, double *leafval) {
    __shared__ int s_nl;
    if (threadIdx.x == 0) {
        int stk_o[32], stk_n[32], sp = 0, nl = 0;
        stk_o[sp] = 0;
        stk_n[sp] = n;
        sp++;
        while (sp > 0) {
            sp--;
            const int o = stk_o[sp], ln = stk_n[sp];
            if (ln <= 128) {
                ls[nl] = o;
                ll[nl] = ln;
                nl++;
            } else {
                int n2 = ln / 2;
                n2 -= n2 % 8;
                stk_o[sp] = o + n2;  // right pushed first, popped after the left subtree
                stk_n[sp] = ln - n2;
                sp++;
                stk_o[sp] = o;
                stk_n[sp] = n2;
                sp++;
            }
        }
        s_nl = nl;
    }
    __syncthreads();
    const int nl = s_nl;
    // leaf sums, eight lanes per leaf: lane j is numpy's accumulator j over the leaf's blocks of 8
    // (reads of consecutive elements by consecutive lanes), the xor butterfly over the eight lanes
    // is ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), the remainder is added in order by the group's lane 0
    const int grp = threadIdx.x >> 3, jl = threadIdx.x & 7, ngrp = blockDim.x >> 3;
    for (int l0 = 0; l0 < nl; l0 += ngrp) {
        const int l = l0 + grp;
        const bool act = l < nl;
        const int o = act ? ls[l] : 0, len = act ? ll[l] : 0;
        const int main_ = len >= 8 ? len - (len & 7) : 0;
        double acc = 0.0;
        if (main_) {  // all (<= 16) loads of the accumulator issued before its sequential adds
            double x[16];
#pragma unroll
            for (int u = 0; u < 16; u++) x[u] = (8 * u < main_) ? a(o + 8 * u + jl) : 0.0;
            acc = x[0];
#pragma unroll
            for (int u = 1; u < 16; u++)
                if (8 * u < main_) acc = f64_add(acc, x[u]);
        }
        acc = f64_add(acc, __shfl_xor_sync(0xffffffffu, acc, 1));
        acc = f64_add(acc, __shfl_xor_sync(0xffffffffu, acc, 2));
        acc = f64_add(acc, __shfl_xor_sync(0xffffffffu, acc, 4));
        if (act && jl == 0) {
            double r = main_ ? acc : -0.0;
            for (int i = main_; i < len; i++) r = f64_add(r, a(o + i));
            leafval[l] = r;
        }
    }
    __syncthreads();
    double res = 0.0;
    if (threadIdx.x == 0) {
        // fold: re-run the recursion over leaf indices (post-order)
        int stk_n[32], stk_state[32], sp = 0, leaf = 0;
        double val[32];
        stk_n[0] = n;
        stk_state[0] = 0;
        sp = 1;
        int vsp = 0;
        while (sp > 0) {
            const int ln = stk_n[sp - 1];
            if (ln <= 128) {
                val[vsp++] = leafval[leaf++];
                sp--;
                continue;
            }
            int n2 = ln / 2;
            n2 -= n2 % 8;
            if (stk_state[sp - 1] == 0) {
                stk_state[sp - 1] = 1;
                stk_n[sp] = n2;
                stk_state[sp] = 0;
                sp++;
            } else if (stk_state[sp - 1] == 1) {
                stk_state[sp - 1] = 2;
                stk_n[sp] = ln - n2;
                stk_state[sp] = 0;
                sp++;
            } else {
                const double rhs = val[--vsp];
                const double lhs = val[--vsp];
                val[vsp++] = f64_add(lhs, rhs);
                sp--;
            }
        }
        res = f64_add(0.0, n ? val[0] : -0.0);
    }
    return res;
}

__device__ inline double s2_pairwise(const double *a, int n, int *ls, int *ll, double *leafval) {
    return s2_pairwise_f([&](int k) { return a[k]; }, n, ls, ll, leafval);
}

// ------------------------------------------------------------------------------------
// host side: context
// ------------------------------------------------------------------------------------
// Checked builds (-DPP_CHECKED, __graft_entry__.build_checked(): libpitplan_b200_checked.so) stand
// in for compute-sanitizer memcheck, which this GPU pool does not offer: every device buffer gets
// 512-byte guard zones on both sides (pattern 0xA5) whose bytes are verified when the buffer is
// freed or re-allocated and by pp_debug_check_guards; fresh payloads are filled with 0xFF (NaN /
// -1) so reads of never-written memory surface as parity failures; PP_DCHECK traps on a failed
// device-side index check.
#ifdef PP_CHECKED
constexpr size_t PP_GUARD = 512;
struct DevBuf;
void guard_register(DevBuf *b);
void guard_unregister(DevBuf *b);
bool guard_intact(const DevBuf *b);  // false: the guard bytes were overwritten (reported once)
#define PP_DCHECK(c)                                                                                      \
    do {                                                                                                  \
        if (!(c)) {                                                                                       \
            printf("PP_DCHECK failed %s:%d: %s (block %d,%d thread %d)\n", __FILE__, __LINE__, #c,           \
                   (int)blockIdx.x, (int)blockIdx.y, (int)threadIdx.x);                                     \
            __trap();                                                                                     \
        }                                                                                                 \
    } while (0)
#else
#define PP_DCHECK(c) \
    do {             \
    } while (0)
#endif

struct DevBuf {
    void *ptr = nullptr;
    size_t bytes = 0;
    uint64_t gen = 0;  // bumped on every (re)allocation: caches keyed on a buffer compare this, not ptr
#ifdef PP_CHECKED
    void *base = nullptr;  // allocation start: [guard][payload: bytes][guard]
    DevBuf() { guard_register(this); }
    ~DevBuf() { guard_unregister(this); }
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
#endif
    int ensure(size_t need) {
        if (need <= bytes) return PP_OK;
        release();
        gen++;
        size_t n = std::max<size_t>(need, 256);
#ifdef PP_CHECKED
        CUDA_TRY(cudaMalloc(&base, n + 2 * PP_GUARD));
        ptr = static_cast<unsigned char *>(base) + PP_GUARD;
        CUDA_TRY(cudaMemset(base, 0xA5, PP_GUARD));
        CUDA_TRY(cudaMemset(static_cast<unsigned char *>(ptr) + n, 0xA5, PP_GUARD));
        CUDA_TRY(cudaMemset(ptr, 0xFF, n));
        CUDA_TRY(cudaDeviceSynchronize());
#else
        CUDA_TRY(cudaMalloc(&ptr, n));
#endif
        bytes = n;
        return PP_OK;
    }
    void release() {
#ifdef PP_CHECKED
        if (base) {
            guard_intact(this);
            cudaFree(base);
        }
        base = nullptr;
#else
        if (ptr) cudaFree(ptr);
#endif
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
    cudaStream_t side = nullptr;                        // second stream (ensure_side_stream)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;   // fork / join between stream and side
    int n_sms = 148;
    int B = 0, T = 0, S = 0, Sp = 0, n_levels = 0, deg_max = 0;
    long long E = 0;
    bool have_instance = false, have_spatial = false, have_scen = false, have_sigma = false, have_sched = false;
    bool have_plant = false;  // pp_set_plant (relaxed NPV)
    double rate = 0.0;
    double mean_cap = 0.0;
    std::vector<int> level_ptr;  // host, n_levels + 1
    std::vector<int> level_of;   // host, B
    // host copies of the instance for host-side drivers (pp_polish_sweep): adjacency (predecessors
    // then successors per block), masses, capacities
    std::vector<int> h_start, h_npred, h_adj;
    std::vector<double> h_mass, h_cap;
    PwPlan plan{};
    int cvar_k = 1;
    // static tables
    DevBuf rows, adj, cost, cap, disc, level_blocks, ones_t, mass;
    DevBuf nbr;        // padded neighbour table [B][nbr_stride] (staged kernel)
    int nbr_stride = 0;
    const int32_t *assign_ptr = nullptr;  // current schedule (own buffer or a borrowed device buffer)
    bool borrowed = false;
    bool pm_dirty = true;
    DevBuf vmax, unit_mean, sigma, sigma_ts, sig_mean, ones_st, plan_dev;
    // schedule
    DevBuf assign, pm;
    // scratch
    DevBuf cnt, compact, pm_batch, predcnt, partial, counter, pm_flags;
    size_t pm_flags_n = 0;
    size_t last_pairs = 0;  // sparse pair count of the previous host-mode evaluation
    DevBuf best_none;       // one pp_best {-inf, -1, -1}
    // host-mode schedules on the cluster path are range-checked on the device by k_pm_cluster
    // (one flag per CTA) and reported by the next host-mode call that synchronises
    DevBuf pm_bad;
    DevBuf mv_win;  // pp_eval_moves: per-block precedence windows of the current schedule
    int32_t *h_bad = nullptr;  // page-locked mirror [8]
    unsigned char *h_bounce = nullptr;  // page-locked bounce buffer for small host-mode results
    unsigned char *h_stage = nullptr;   // page-locked staging for packed host-mode uploads/results
    // pp_npv_moves: the base schedule's stage-2 results stay in npv_raw/_cost/_n between calls;
    // reused while the tables (npv_gen), the buffers and the base assignment are unchanged
    uint64_t npv_gen = 0, npvm_gen = ~0ull;
    std::vector<int32_t> npvm_base;
    std::vector<int32_t> npvm_cnt;  // mined blocks per period of npvm_base
    uint64_t npvm_bufgen[3] = {0, 0, 0};  // DevBuf::gen of npv_raw / npv_cost / npv_n when cached
    size_t h_stage_bytes = 0;
    DevBuf bad_cand;                    // int32: out-of-range candidate id seen (host-mode check)
    DevBuf ej_count, ej_key, ej_blk;    // ejection lists [T][B] (pp_eject)
    DevBuf hours, npv_raw, npv_cost, npv_n;  // relaxed NPV (pp_npv.cu)
    DevBuf s2_items, s2_scratch;  // large-period stage-2: work list [S*T*P | S*2*M] and per-CTA scratch
    DevBuf s2_rec;                // pp_npv_moves: the base schedule's per-(s, t) greedy structure
    DevBuf s2_assign;             // pp_npv_moves: the device copy of the cached base schedule
    DevBuf npvm_flags;            // pp_npv_moves: progress flags of the concurrent one-block update
    uint64_t npvm_flags_gen = 0;
    uint32_t npvm_epoch = 0;
    unsigned long long npvm_vc = 0;  // cost-sum CTAs launched as dependents of an update (cumulative)
    DevBuf pr_score, pr_cap, pr_assign, pr_elig;       // pricing greedy (pp_price.cu)
    // device-resident lns insertion loop (pp_lns.cu): rook CSR (pp_set_rook), mean grades, the pool
    // (unordered list + positions), ranking keys, control block, per-round candidates and results
    DevBuf lns_rptr, lns_ridx, lns_mg, lns_pool, lns_pos, lns_keys, lns_ctl, lns_out;
    DevBuf lns_rpi;  // the first block of every directed rook pair (Moran's I, pp_uncert.cu)
    int rook_pairs = 0;
    bool have_rook = false;
    // VAE decoder (pp_vae.cu): layer widths, packed W/b per layer, norm_mean | norm_std, scratch
    std::vector<int32_t> vae_widths;
    DevBuf vae_params, vae_norm, vae_h, vae_io;
    // host-mode pp_eval_candidates repeated with identical arguments (page-locked ids and outputs):
    // its launches (period masses or output init, evaluation, copy-out) replayed as one graph
    struct EvalGraphKey {
        const void *cand;
        int32_t C, scenario;
        uint32_t flags;
        int32_t pm_dirty, bad_pending, cvar_k, S, T, B, Sp;
        pp_cand_out out;
        const void *assign_ptr;
        uint64_t gensum, pinned_gen;
    };
    struct EvalBounce {
        void *user;  // nullptr: the call's own bad-candidate flag
        size_t off, bytes;
    };
    EvalGraphKey ev_key{}, ev_seen{};
    bool ev_have_seen = false, ev_bad_copy = false;
    cudaGraph_t ev_graph = nullptr;
    cudaGraphExec_t ev_exec = nullptr;
    EvalBounce ev_bounce[4]{};
    int ev_nb = 0;
    cudaGraph_t lns_graph = nullptr;      // the cached insertion-loop graph (pp_lns_insert)
    cudaGraphExec_t lns_exec = nullptr;
    uint64_t lns_key[3] = {0, 0, 0};      // width, flags, sum of the buffers' allocation generations
    bool bad_pending = false;
    DevBuf h_cand, h_a, h_b, h_o1, h_o2, h_o3, h_o4, h_o5, h_o6, h_o7, h_o8, h_glob, h_assign, h_i64, h_d1, h_d2,
        h_pm, h_p;
    std::vector<DevBuf *> all() {
        return {&rows, &adj, &nbr, &cost, &cap, &disc, &level_blocks, &ones_t, &mass, &vmax, &unit_mean, &sigma, &sigma_ts, &sig_mean,
                &ones_st, &plan_dev, &assign, &pm, &cnt, &compact, &pm_batch, &predcnt, &partial, &counter, &pm_flags, &h_cand, &h_a,
                &h_b, &h_o1, &h_o2, &h_o3, &h_o4, &h_o5, &h_o6, &h_o7, &h_o8, &h_glob, &h_assign, &h_i64, &h_d1,
                &h_d2, &h_pm, &h_p, &best_none, &bad_cand, &ej_count, &ej_key, &ej_blk, &hours, &npv_raw,
                &npv_cost, &npv_n, &s2_items, &s2_scratch, &s2_rec, &s2_assign, &pr_score, &pr_cap, &pr_assign, &pr_elig,
                &pm_bad, &mv_win, &npvm_flags, &vae_params, &vae_norm, &vae_h, &vae_io, &lns_rptr, &lns_ridx, &lns_rpi, &lns_mg, &lns_pool, &lns_pos, &lns_keys, &lns_ctl, &lns_out};
    }
};

// PP_TRACE_HOST=1: per-phase host time of the C-ABI calls on stderr (diagnostics only)
struct HostTrace {
    const char *name;
    bool on;
    std::chrono::steady_clock::time_point t0, t;
    static bool enabled() {
        static const bool on_ = std::getenv("PP_TRACE_HOST") != nullptr;
        return on_;
    }
    explicit HostTrace(const char *n) : name(n), on(enabled()) {
        if (on) t0 = t = std::chrono::steady_clock::now();
    }
    void mark(const char *what) {  // (the print is not charged to the next phase)
        if (!on) return;
        const auto n = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[%s] %-12s %7.1f us\n", name, what, std::chrono::duration<double, std::micro>(n - t).count());
        t = std::chrono::steady_clock::now();
    }
    ~HostTrace() {
        if (on)
            std::fprintf(stderr, "[%s] total        %7.1f us\n", name,
                         std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
    }
};

// Host-mode completion wait: spin on the stream (the results are usually ~20-40 us away, below a
// blocking synchronisation's wake-up latency).
inline cudaError_t stream_wait(cudaStream_t st) {
    cudaError_t e;
    while ((e = cudaStreamQuery(st)) == cudaErrorNotReady) {
    }
    return e;
}

// page-locked staging of at least `bytes` (grown on demand, kept for the context's lifetime)
inline int host_stage(pp_ctx *c, size_t bytes, unsigned char **out) {
    if (c->h_stage_bytes < bytes) {
        if (c->h_stage) CUDA_TRY(cudaFreeHost(c->h_stage));
        c->h_stage = nullptr;
        c->h_stage_bytes = 0;
        const size_t n = std::max<size_t>(bytes, 4096);
        CUDA_TRY(cudaHostAlloc(reinterpret_cast<void **>(&c->h_stage), n, cudaHostAllocPortable));
        c->h_stage_bytes = n;
    }
    *out = c->h_stage;
    return PP_OK;
}

inline int use_device(pp_ctx *c) {
    CUDA_TRY(cudaSetDevice(c->device));
    return PP_OK;
}

inline cudaStream_t pick(pp_ctx *c, void *stream) { return stream ? (cudaStream_t)stream : c->stream; }

// Setup-time upload / clear, complete on return.  Every table goes through the context stream:
// c->stream is non-blocking, so a plain cudaMemcpy / cudaMemset (legacy default stream) is NOT
// ordered before kernels on it, and a pageable cudaMemcpy may return before its DMA lands.
inline cudaError_t dev_upload(pp_ctx *c, void *dst, const void *src, size_t bytes) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream);
    return e == cudaSuccess ? cudaStreamSynchronize(c->stream) : e;
}
inline cudaError_t dev_zero(pp_ctx *c, void *dst, size_t bytes) {
    cudaError_t e = cudaMemsetAsync(dst, 0, bytes, c->stream);
    return e == cudaSuccess ? cudaStreamSynchronize(c->stream) : e;
}

// host copy of numpy's pairwise sum (for np.mean(capacity), evaluate.py:103)
inline double host_pairwise(const double *a, long n) {
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

// launch with programmatic stream serialization (PDL) when a period-mass kernel precedes
template <typename... KArgs, typename... Args>
inline int launch_eval(void (*kern)(KArgs...), int grid, size_t smem, cudaStream_t st, bool pdl, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(EV_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    static const bool no_pdl = std::getenv("PP_NO_PDL") != nullptr;  // diagnostics: serialise the launches
    cfg.numAttrs = (pdl && !no_pdl) ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args...);
    if (e != cudaSuccess) return fail(PP_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(e));
    return PP_OK;
}
template <typename... KArgs, typename... Args>
inline int launch_eval_n(void (*kern)(KArgs...), dim3 grid, int threads, size_t smem, cudaStream_t st, bool pdl,
                         Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    static const bool no_pdl = std::getenv("PP_NO_PDL") != nullptr;  // diagnostics: serialise the launches
    cfg.numAttrs = (pdl && !no_pdl) ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args...);
    if (e != cudaSuccess) return fail(PP_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(e));
    return PP_OK;
}


// ---- shared host helpers (pp_context.cu, pp_schedule.cu) ----
// page-locked buffers from pp_host_alloc: host range -> device mapping (nullptr if not one of them)
void pinned_register(void *host, size_t bytes, void *dev);
void pinned_unregister(void *host);
void *pinned_lookup(const void *host);
uint64_t pinned_generation();  // changes whenever a pp_host_alloc buffer is registered or freed
int ensure_grid_scratch(pp_ctx *c, int grid);
int check_ready(pp_ctx *c, uint32_t flags, int scenario);
int pick_kc(int k);
// Per-launch output state the evaluation kernel accumulates into with atomics: the period-mass
// launch ahead of it initialises it (n_pairs = 0, best = none), otherwise a copy node does.
struct EvalInit {
    int32_t *n_pairs;
    pp_best *best;
    int32_t *bad_cand;  // set to 0; the evaluation stores 1 on an out-of-range candidate id
};
int run_period_mass(pp_ctx *c, const int32_t *d_assign, int P, double *d_pm, cudaStream_t st,
                    const EvalInit *init = nullptr);
int refresh_pm(pp_ctx *c, cudaStream_t st, bool *launched, const EvalInit *init = nullptr);
int init_eval_outputs(pp_ctx *c, const EvalInit &init, cudaStream_t st);
bool pm_cluster_path(const pp_ctx *c);
void *mapped_host(const void *p);  // device alias of page-locked host memory, or nullptr
int ensure_side_stream(pp_ctx *c);  // c->side + fork/join events, created on first use
// after the stream was synchronised: PP_ERR_INVALID_ARGS if the pending host schedule had
// period indices out of range (h_bad already copied when `copied`)
int check_schedule_range(pp_ctx *c, bool copied);
int launch_general_candidates(int PER, int kc, bool scen, int C, int G, int S, int Sp, int T, bool stats,
                              cudaStream_t st, bool pdl, int device, const EvalParams &ep);

// cudaFuncSetAttribute(kern, MaxDynamicSharedMemorySize) once per (kernel, device): the attribute is
// per device, and one process may drive several devices (evaluate.set_device)
int smem_attr_needed(const void *kern, int device, size_t bytes);  // pp_context.cu (keyed by kernel)
template <typename K>
inline int ensure_max_smem(K kern, size_t bytes, int device) {
    if (!smem_attr_needed(reinterpret_cast<const void *>(kern), device, bytes)) return PP_OK;
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    return PP_OK;
}

// the 48 KB default covers static + dynamic; opt in (once per kernel and device) with room for the
// kernels' static arrays
template <typename K>
inline int set_smem_attr(K kern, size_t bytes, int device) {
    return bytes > 32 * 1024 ? ensure_max_smem(kern, bytes, device) : PP_OK;
}

// resident CTAs of a kernel at this smem size (cached per instantiation)
template <typename K>
inline int resident_ctas(K kern, size_t smem, int device) {
    int per_sm = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, EV_THREADS, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || sms < 1) sms = 148;
    return per_sm * sms;
}

