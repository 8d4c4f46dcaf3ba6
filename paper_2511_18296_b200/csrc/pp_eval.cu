// pp_eval.cu -- evaluate_candidates_parallel (evaluate.py:306-430): the staged fast-path kernel
// and pp_eval_candidates (which dispatches to pp_eval_general.cu otherwise).
#include "pp_internal.cuh"

// ------------------------------------------------------------------------------------
// k_eval_staged: the fast path of pp_eval_candidates (T <= 32, S <= 128, degree <= 32).
// A CTA takes NB consecutive candidates and stages everything they need in shared
// memory with a handful of dependent round trips for the whole batch (instead of one
// chain per candidate): ids; BlockRow / assign / unit / mining-cost row / vmax row via
// cp.async; adjacency ids then neighbour periods (precedence window reduced per warp).
// Groups of G lanes (lanes = periods) then compute from shared memory.  Everything
// before griddepcontrol.wait is independent of the period masses, so it overlaps the
// period-mass kernels under programmatic dependent launch.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void *s, const void *g) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async8(void *s, const void *g) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async4(void *s, const void *g) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

struct StagedLayout {  // byte offsets into dynamic shared memory
    int sig, tab, vrow, cost, nbr, ex, cv, row, unit, pair, b, ab, lo, hi, npair, okbits, total;
};

static __host__ __device__ inline int align16(int x) { return (x + 15) & ~15; }

static __host__ __device__ inline StagedLayout staged_layout(int NB, int T, int S, int Sp, int nbr_stride, bool stats,
                                                             bool need_vrow, bool net) {
    StagedLayout L;
    int o = 0;
    L.sig = o;  // sigma [S][T] (statistics)
    o += stats ? align16(8 * S * T) : 0;
    L.tab = o;  // cap, disc, sig_row, pm: [4][T]
    o += align16(8 * 4 * T);
    L.vrow = o;
    o += need_vrow ? align16(8 * NB * Sp) : 0;
    L.cost = o;
    o += net ? align16(8 * NB * T) : 0;
    L.nbr = o;
    o += align16(4 * NB * nbr_stride);
    L.ex = o;
    o += stats ? align16(8 * NB * T) : 0;
    L.cv = o;
    o += stats ? align16(8 * NB * T) : 0;
    L.row = o;
    o += align16(32 * NB);
    L.unit = o;
    o += align16(8 * NB);
    L.pair = o;
    o += stats ? align16(4 * NB * T) : 0;
    L.b = o;
    o += align16(4 * NB);
    L.ab = o;
    o += align16(4 * NB);
    L.lo = o;
    o += align16(4 * NB);
    L.hi = o;
    o += align16(4 * NB);
    L.npair = o;
    o += align16(4 * (NB + 1));
    L.okbits = o;  // one 32-bit mask of feasible periods per candidate (T <= 32)
    o += align16(4 * NB);
    L.total = o;
    return L;
}

// One (candidate, period) pair: per-scenario deltas d_s = val_s(b,t) - val_s(b,a[b])
// (evaluate.py:380-382 with s=k), expected = np.mean(d) (a single numpy pairwise leaf,
// S <= 128), CVaR10 = mean of the k smallest (saa.py:157-164); raw d_s optionally.
template <int KC, bool SCEN>
__device__ __forceinline__ void pair_stats(const EvalParams &p, int S, int T, const double *sg, const double *rowb,
                                           int t, int abc,
                                           double d_t, double dc_t, double d_ab, double dc_ab, double sp, bool mined,
                                           double *ex, double *cv, float *sd) {
    const int main_ = S & ~7;  // sg: sigma [S][T] staged in shared memory
    double acc[8];
#pragma unroll
    for (int j = 0; j < 8; j++) acc[j] = -0.0;
    TopK<KC> tk;
    tk.init();
    for (int s8 = 0; s8 < main_; s8 += 8) {
#pragma unroll
        for (int j = 0; j < 8; j++) {
            const int s = s8 + j;
            const double x = rowb[s];
            const double vn = f64_sub(f64_mul(f64_mul(f64_mul(x, d_t), sg[s * T + t]), sp), dc_t);
            const double vo =
                mined ? f64_sub(f64_mul(f64_mul(f64_mul(x, d_ab), sg[s * T + abc]), sp), dc_ab) : 0.0;
            const double v = f64_sub(vn, vo);  // vn - 0.0 == vn exactly
            acc[j] = f64_add(acc[j], v);
            tk.push(v);
            if constexpr (SCEN) sd[(size_t)s * T] = (float)v;
        }
    }
    double res = main_ ? tree8(acc) : -0.0;
    for (int s = main_; s < S; s++) {
        const double x = rowb[s];
        const double vn = f64_sub(f64_mul(f64_mul(f64_mul(x, d_t), sg[s * T + t]), sp), dc_t);
        const double vo =
            mined ? f64_sub(f64_mul(f64_mul(f64_mul(x, d_ab), sg[s * T + abc]), sp), dc_ab) : 0.0;
        const double v = f64_sub(vn, vo);
        res = f64_add(res, v);
        tk.push(v);
        if constexpr (SCEN) sd[(size_t)s * T] = (float)v;
    }
    *ex = f64_div(f64_add(0.0, res), (double)S);
    *cv = tk.mean(p.cvar_k);
}

// ------------------------------------------------------------------------------------
// k_eval_staged: the fast path of pp_eval_candidates (T <= 32, S <= 128, degree <= 32).
// Sized for the sparsity of the problem (at C2 a candidate's precedence window holds 1.2
// of 15 periods on average, 8% of the moves are feasible), NB candidates per CTA:
//   stage 1  candidate ids
//   stage 2  one warp per candidate: BlockRow, assign, unit, padded neighbour row,
//            mining-cost row, vmax row via cp.async -- one round trip for the batch
//   stage 3  one thread per candidate: neighbour periods -> precedence window
//            (evaluate.py:361-372); then the list of precedence-feasible (candidate, t)
//   B        one thread per feasible pair: per-scenario statistics into shared memory
//   C        griddepcontrol.wait; one thread per candidate walks its window: capacity
//            (evaluate.py:373-378), parity value (379-384), lowest-t argmax (387-388)
//   out      one thread per (candidate, period): coalesced writes of the [NB][T] block
//   K4       warp argmax of the CTA's candidates, deterministic grid argmax
// Stages 1-3 and B never read the period masses: under programmatic dependent launch
// they overlap k_pm_chunks / k_pm_tree.
// ------------------------------------------------------------------------------------
#ifdef PP_EVAL_PROBE
__device__ unsigned long long g_ev_probe[4096][8];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define EV_PROBE(k) do { if (threadIdx.x == 0 && blockIdx.x < 4096) g_ev_probe[blockIdx.x][k] = gtimer(); } while (0)
#else
#define EV_PROBE(k) do { } while (0)
#endif

template <int KC, bool SCEN>
__global__ void __launch_bounds__(EV_THREADS, 4) k_eval_staged(const EvalParams p, const int NB) {
    extern __shared__ __align__(16) unsigned char st_dyn[];
    __shared__ Best s_red[EV_THREADS / 32];
    constexpr int NW = EV_THREADS / 32;
    const int T = p.T, S = p.S, Sp = p.Sp, NS = p.nbr_stride;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
    const bool net = p.flags & PP_NET_MINING_COST;
    const bool literal = p.flags & PP_LITERAL_VALUE;
    constexpr bool STATS_T = KC > 0;
    const bool stats = STATS_T && (SCEN || p.exp_delta || p.cvar);
    const bool need_vrow = stats || (!literal && p.scen >= 0);
    const StagedLayout L = staged_layout(NB, T, S, Sp, NS, stats, need_vrow, net);
    double *s_sig = reinterpret_cast<double *>(st_dyn + L.sig);
    double *s_cap = reinterpret_cast<double *>(st_dyn + L.tab);
    double *s_disc = s_cap + T, *s_srow = s_cap + 2 * T, *s_pm = s_cap + 3 * T;
    double *s_vrow = reinterpret_cast<double *>(st_dyn + L.vrow);
    double *s_cost = reinterpret_cast<double *>(st_dyn + L.cost);
    int *s_nbr = reinterpret_cast<int *>(st_dyn + L.nbr);
    double *s_ex = reinterpret_cast<double *>(st_dyn + L.ex);
    double *s_cv = reinterpret_cast<double *>(st_dyn + L.cv);
    BlockRow *s_row = reinterpret_cast<BlockRow *>(st_dyn + L.row);
    double *s_unit = reinterpret_cast<double *>(st_dyn + L.unit);
    int *s_pair = reinterpret_cast<int *>(st_dyn + L.pair);
    int *s_b = reinterpret_cast<int *>(st_dyn + L.b);
    int *s_ab = reinterpret_cast<int *>(st_dyn + L.ab);
    int *s_lo = reinterpret_cast<int *>(st_dyn + L.lo);
    int *s_hi = reinterpret_cast<int *>(st_dyn + L.hi);
    int *s_np = reinterpret_cast<int *>(st_dyn + L.npair);
    unsigned *s_ok = reinterpret_cast<unsigned *>(st_dyn + L.okbits);
    const int c0 = blockIdx.x * NB;
    EV_PROBE(0);

    // ---- stage 1 ----
    for (int i = tid; i < NB; i += EV_THREADS) {
        const int g = c0 + i;
        int b = (g < p.C) ? __ldg(p.cand + g) : -1;
        if (b >= p.B) b = -1;
        s_b[i] = b;
    }
    for (int t = tid; t < T; t += EV_THREADS) {
        s_cap[t] = __ldg(p.cap + t);
        s_disc[t] = __ldg(p.disc + t);
        s_srow[t] = __ldg(p.sig_row + t);
    }
    if (stats) {  // sigma [S][T] (S*T*8 is a multiple of 8; copy 8-byte pieces)
        for (int e = tid; e < S * T; e += EV_THREADS) cp_async8(s_sig + e, p.sigma + e);
    }
    __syncthreads();
    EV_PROBE(1);

    // ---- stage 2: every row of every candidate in one cp.async round trip ----
    {
        const bool want_unit = !literal && p.scen < 0;
        const int nv = need_vrow ? (Sp >> 1) : 0, nn = NS >> 2;
        for (int i = warp; i < NB; i += NW) {
            const int b = max(s_b[i], 0);
            if (lane < 2)
                cp_async16(reinterpret_cast<char *>(s_row + i) + 16 * lane,
                           reinterpret_cast<const char *>(p.rows + b) + 16 * lane);
            if (lane == 2) cp_async4(s_ab + i, p.assign + b);
            if (lane == 3 && want_unit) cp_async8(s_unit + i, p.unit_mean + b);
            if (lane < nn) cp_async16(s_nbr + (size_t)i * NS + 4 * lane, p.nbr + (size_t)b * NS + 4 * lane);
            if (net && lane < T) cp_async8(s_cost + (size_t)i * T + lane, p.cost + (size_t)b * T + lane);
            for (int q = lane; q < nv; q += 32)
                cp_async16(s_vrow + (size_t)i * Sp + 2 * q, p.vmax + (size_t)b * Sp + 2 * q);
        }
        cp_async_wait_all();
    }
    __syncthreads();
    EV_PROBE(2);

    // ---- stage 3: precedence window, one thread per candidate ----
    for (int i = tid; i < NB; i += EV_THREADS) {
        const BlockRow r = s_row[i];
        const int npred = r.cnt & 0xffff, nnb = npred + (r.cnt >> 16);
        const int *nb = s_nbr + (size_t)i * NS;
        int lo = 0, hi = INT_MAX;
        int tn[32];
#pragma unroll
        for (int k = 0; k < 32; k++)  // independent gathers first (assign is L2-resident)
            if (k < nnb) tn[k] = p.assign[nb[k]];
#pragma unroll
        for (int k = 0; k < 32; k++) {
            if (k < npred) lo = max(lo, tn[k] < 0 ? INT_MAX : tn[k]);
            else if (k < nnb && tn[k] >= 0) hi = min(hi, tn[k]);
        }
        if (s_b[i] < 0) lo = INT_MAX;  // inactive slot: nothing feasible
        s_lo[i] = lo;
        s_hi[i] = hi;
        if (!literal && p.scen >= 0) s_unit[i] = s_vrow[(size_t)i * Sp + p.scen];
        if (literal) s_unit[i] = f64_mul(r.mass, 100.0);
    }
    EV_PROBE(3);

    // ---- C: capacity (evaluate.py:373-378), parity value (379-384), lowest-t argmax
    //      (387-388), one thread per candidate.  Everything above overlapped the
    //      period-mass kernels (PDL); the period masses are needed from here on.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int t = tid; t < T; t += EV_THREADS) s_pm[t] = __ldcg(p.pm + t);
    __syncthreads();
    EV_PROBE(4);
    Best mine{-kInf, INT_MAX, INT_MAX};
    for (int i = tid; i < NB; i += EV_THREADS) {
        const int b = s_b[i];
        const BlockRow r = s_row[i];
        const int ab = s_ab[i];
        const int lo = s_lo[i], z = min(s_hi[i], T - 1);
        unsigned okb = 0u;
        double bv = -kInf;
        int bt = INT_MAX;
        for (int t = lo; t <= z; t++) {
            double load = f64_add(s_pm[t], r.mass);
            if (ab == t) load = f64_sub(load, r.mass);
            if (load > s_cap[t]) continue;
            okb |= 1u << t;
            const double d = s_disc[t];
            double v = f64_mul(f64_mul(f64_mul(s_unit[i], d), s_srow[t]), r.spatial);
            if (net) v = f64_sub(v, f64_mul(d, s_cost[(size_t)i * T + t]));
            if (v > bv) {  // strict: the lowest period wins ties (evaluate.py:387-388)
                bv = v;
                bt = t;
            }
        }
        s_ok[i] = okb;
        s_np[i] = __popc(okb);
        if (b >= 0) {
            const int grp = c0 + i;
            const bool cand_ok = bt != INT_MAX;
            p.best_t[grp] = cand_ok ? bt : -1;
            p.best_val[grp] = bv;
            p.feas[grp] = cand_ok ? 1 : 0;
            if (cand_ok) {
                Best cb{bv, b, bt};
                if (better(cb, mine)) mine = cb;
            }
        }
    }
    __syncthreads();
    EV_PROBE(5);

    // ---- B: statistics of the feasible (candidate, period) pairs (~8% of moves at C2) ----
    if constexpr (STATS_T) {
        if (stats) {
            if (warp == 0) {  // exclusive scan of the pair counts
                int carry = 0;
                for (int i0 = 0; i0 < NB; i0 += 32) {
                    const int v = (i0 + lane < NB) ? s_np[i0 + lane] : 0;
                    int incl = v;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += y;
                    }
                    if (i0 + lane < NB) s_np[i0 + lane] = carry + incl - v;
                    carry += __shfl_sync(0xffffffffu, incl, 31);
                }
                if (lane == 0) s_np[NB] = carry;
            }
            __syncthreads();
            for (int i = tid; i < NB; i += EV_THREADS) {  // pair list: (candidate << 8) | period
                unsigned okb = s_ok[i];
                int o = s_np[i];
                while (okb) {
                    const int t = __ffs(okb) - 1;
                    okb &= okb - 1;
                    s_pair[o++] = (i << 8) | t;
                }
            }
            __syncthreads();
            const int npairs = s_np[NB];
            if constexpr (KC <= 2) {
                // 8 lanes per pair; lane j owns numpy's accumulator j (scenarios s = j mod 8),
                // the butterfly xor 1,2,4 is ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), the <8-element
                // tail is added in order; per-lane two smallest merged by butterfly (CVaR, k <= 2)
                const int sub = lane & 7, sgi = tid >> 3, nsg = EV_THREADS >> 3;
                const int main_ = S & ~7, nrem = S - main_;
                for (int k0 = 0; k0 < npairs; k0 += nsg) {
                    const int k = k0 + sgi;
                    const bool act = k < npairs;
                    const int pr = act ? s_pair[k] : 0;
                    const int i = pr >> 8, t = pr & 0xff;
                    const int ab = s_ab[i];
                    const bool mined = ab >= 0;
                    const int abc = mined ? ab : 0;
                    const double d_t = s_disc[t], d_ab = s_disc[abc], sp = s_row[i].spatial;
                    const double dc_t = net ? f64_mul(d_t, s_cost[(size_t)i * T + t]) : 0.0;
                    const double dc_ab = net ? f64_mul(d_ab, s_cost[(size_t)i * T + abc]) : 0.0;
                    const double *rowb = s_vrow + (size_t)i * Sp;
                    float *sd = SCEN ? p.scen_delta + (size_t)(c0 + i) * S * T + t : nullptr;
                    double acc = -0.0, a0 = kInf, a1 = kInf, remv = 0.0;
                    if (act) {
                        for (int s_ = sub; s_ < S; s_ += 8) {
                            const double x = rowb[s_];
                            const double vn = f64_sub(f64_mul(f64_mul(f64_mul(x, d_t), s_sig[s_ * T + t]), sp), dc_t);
                            const double vo =
                                mined ? f64_sub(f64_mul(f64_mul(f64_mul(x, d_ab), s_sig[s_ * T + abc]), sp), dc_ab) : 0.0;
                            const double v = f64_sub(vn, vo);  // vn - 0.0 == vn exactly
                            if (s_ < main_) acc = f64_add(acc, v);
                            else remv = v;
                            if (v < a1) {
                                if (v < a0) {
                                    a1 = a0;
                                    a0 = v;
                                } else {
                                    a1 = v;
                                }
                            }
                            if constexpr (SCEN) sd[(size_t)s_ * T] = (float)v;
                        }
                    }
                    acc = f64_add(acc, __shfl_xor_sync(0xffffffffu, acc, 1));
                    acc = f64_add(acc, __shfl_xor_sync(0xffffffffu, acc, 2));
                    acc = f64_add(acc, __shfl_xor_sync(0xffffffffu, acc, 4));
                    double res = main_ ? acc : -0.0;
                    for (int j = 0; j < nrem; j++) res = f64_add(res, __shfl_sync(0xffffffffu, remv, (lane & ~7) + j));
#pragma unroll
                    for (int o = 1; o < 8; o <<= 1) {
                        const double b0 = __shfl_xor_sync(0xffffffffu, a0, o);
                        const double b1 = __shfl_xor_sync(0xffffffffu, a1, o);
                        const double lo = (b0 < a0) ? b0 : a0, hi = (b0 < a0) ? a0 : b0;
                        const double m1 = (b1 < a1) ? b1 : a1;
                        a0 = lo;
                        a1 = (m1 < hi) ? m1 : hi;
                    }
                    if (act && sub == 0) {
                        s_ex[(size_t)i * T + t] = f64_div(f64_add(0.0, res), (double)S);
                        double c = f64_add(-0.0, a0);
                        if (p.cvar_k > 1) c = f64_add(c, a1);
                        s_cv[(size_t)i * T + t] = f64_mul(f64_add(0.0, c), p.cvar_k > 1 ? 0.5 : 1.0);
                    }
                }
            } else {
                for (int k = tid; k < npairs; k += EV_THREADS) {  // one thread per pair
                    const int i = s_pair[k] >> 8, t = s_pair[k] & 0xff;
                    const int ab = s_ab[i];
                    const int abc = (ab >= 0 && ab < T) ? ab : 0;
                    const double d_t = s_disc[t], d_ab = s_disc[abc];
                    const double dc_t = net ? f64_mul(d_t, s_cost[(size_t)i * T + t]) : 0.0;
                    const double dc_ab = net ? f64_mul(d_ab, s_cost[(size_t)i * T + abc]) : 0.0;
                    float *sd = SCEN ? p.scen_delta + (size_t)(c0 + i) * S * T + t : nullptr;
                    pair_stats<KC, SCEN>(p, S, T, s_sig, s_vrow + (size_t)i * Sp, t, abc, d_t, dc_t, d_ab, dc_ab,
                                         s_row[i].spatial, ab >= 0, s_ex + (size_t)i * T + t, s_cv + (size_t)i * T + t,
                                         sd);
                }
            }
            __syncthreads();
        }
    }
    EV_PROBE(6);

    // ---- per-(candidate, period) outputs: the CTA's [NB][T] block, coalesced ----
    const bool want_trace = p.trace_val || p.trace_feas;
    if (want_trace || stats) {
        const int nvalid = min(NB, p.C - c0);
        for (int e = tid; e < nvalid * T; e += EV_THREADS) {
            const int i = e / T, t = e - i * T;
            const size_t m = (size_t)c0 * T + e;
            const bool ok = (s_ok[i] >> t) & 1u;
            if (want_trace) {
                double v = -kInf;
                if (ok) {
                    const double d = s_disc[t];
                    const BlockRow &r = s_row[i];
                    v = f64_mul(f64_mul(f64_mul(s_unit[i], d), s_srow[t]), r.spatial);
                    if (net) v = f64_sub(v, f64_mul(d, s_cost[(size_t)i * T + t]));
                }
                if (p.trace_val) p.trace_val[m] = v;
                if (p.trace_feas) p.trace_feas[m] = ok ? 1 : 0;
            }
            if constexpr (STATS_T) {
                if (stats) {
                    if (p.exp_delta) p.exp_delta[m] = ok ? s_ex[e] : -kInf;
                    if (p.cvar) p.cvar[m] = ok ? s_cv[e] : -kInf;
                    if constexpr (SCEN) {
                        if (!ok)  // infeasible: raw deltas are -inf (also overwrites capacity-infeasible pairs)
                            for (int s = 0; s < S; s++)
                                p.scen_delta[((size_t)(c0 + i) * S + s) * T + t] = -__int_as_float(0x7f800000);
                    }
                }
            }
        }
    }

    // ---- K4: CTA argmax (candidates are one per thread of warp 0 when NB <= 32) ----
    if (NB > 32) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            Best o = shfl_best(mine, off);
            if (better(o, mine)) mine = o;
        }
        if (lane == 0) s_red[warp] = mine;
        __syncthreads();
        if (warp == 0) mine = (lane < NW) ? s_red[lane] : Best{-kInf, INT_MAX, INT_MAX};
        __syncthreads();
    }
    grid_argmax_warp0(mine, s_red, p.partial, p.counter, p.global);
    EV_PROBE(7);
}

#ifdef PP_EVAL_PROBE
extern "C" PP_API int pp_debug_eval_probe(unsigned long long *out) {
    return cudaMemcpyFromSymbol(out, g_ev_probe, sizeof(unsigned long long) * 4096 * 8) == cudaSuccess ? 0 : 3;
}
#endif

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
    ep.nbr = c->nbr.as<int32_t>();
    ep.nbr_stride = c->nbr_stride;
    ep.assign = c->assign_ptr;
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

    // fast path: whole candidate batches staged in shared memory
    if (T <= 32 && (!stats || S <= 128) && c->deg_max <= 32 && c->nbr.ptr) {
        const int NB = 32;
        const bool need_vrow = stats || (!(flags & PP_LITERAL_VALUE) && scenario >= 0);
        const StagedLayout Ls =
            staged_layout(NB, T, S, c->Sp, c->nbr_stride, stats, need_vrow, (flags & PP_NET_MINING_COST) != 0);
        if (Ls.total <= 200 * 1024) {
            const int sgrid = std::max(1, (C + NB - 1) / NB);
            TRY(ensure_grid_scratch(c, sgrid));
            bool pdl;
            TRY(refresh_pm(c, st, &pdl));
            const bool scen = o.scen_delta != nullptr;
            const size_t smem_s = (size_t)Ls.total;
#define PP_STAGED(KC, SC)                                                              \
    {                                                                                  \
        TRY(set_smem_attr(k_eval_staged<KC, SC>, smem_s));                             \
        TRY(launch_eval(k_eval_staged<KC, SC>, sgrid, smem_s, st, pdl, ep, NB));       \
    }
            if (kc == 0) PP_STAGED(0, false)
            else if (kc == 2) { if (scen) PP_STAGED(2, true) else PP_STAGED(2, false) }
            else if (kc == 8) { if (scen) PP_STAGED(8, true) else PP_STAGED(8, false) }
            else { if (scen) PP_STAGED(128, true) else PP_STAGED(128, false) }
#undef PP_STAGED
            goto copy_out;
        }
    }
    {
        bool pdl;
        TRY(refresh_pm(c, st, &pdl));
        TRY(launch_general_candidates(PER, kc, o.scen_delta != nullptr, C, G, S, c->Sp, T, stats, st, pdl, c->device,
                                      ep));
    }
copy_out:

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

}  // extern "C"
