// pp_eval.cu -- candidate evaluation kernels (evaluate_candidates_parallel, evaluate.py:306-430)
// and pp_eval_candidates.
#include "pp_internal.cuh"

// ------------------------------------------------------------------------------------
// candidate evaluation: K1 value, K2 precedence window, K3 capacity, K4 argmax
// ------------------------------------------------------------------------------------

// Persistent grid: each lane group of G = pow2 >= T lanes (4..32) walks candidates
// grp, grp + total_groups, ...; lane tl owns periods tl, tl+G, ... (PER slots, PER > 1
// only when T > 32).  Per candidate:
//   A  loads + precedence window (K2), no dependency on the period masses
//   B  per-scenario deltas for every precedence-feasible period (K1 statistics), still
//      independent of the period masses -- this overlaps k_period_mass under PDL
//   C  griddepcontrol.wait, capacity (K3), parity value, lowest-t argmax, outputs; K4
//      grid argmax after the loop.
// Shared memory (stats only): sigma staged once per CTA as [T][SS] (SS = S | 1, odd
// stride: conflict-free for lanes = periods), then per group the candidate's vmax row and
// its current-period values.
template <int PER, int KC, bool BIGS, bool SCEN>
__global__ void __launch_bounds__(EV_THREADS) k_eval_candidates(const EvalParams p, const int G,
                                                                const int total_groups) {
    extern __shared__ __align__(16) double ev_dyn[];
    __shared__ Best s_red[EV_THREADS / 32];

    const int GPW = 32 / G, GPC = (EV_THREADS / 32) * GPW;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tl = lane & (G - 1);
    const int gl = warp * GPW + lane / G;  // group within CTA
    const int T = p.T, S = p.S;
    const bool net = p.flags & PP_NET_MINING_COST;
    constexpr bool STATS_T = KC > 0;
    const bool stats = STATS_T && (SCEN || p.exp_delta || p.cvar);
    const int SS = S | 1;
    const int SB = BIGS ? 32 : p.Sp;
    double *s_sig = ev_dyn;  // [T][SS] (not BIGS)
    double *rowb = ev_dyn + (BIGS ? 0 : (size_t)T * SS) + (size_t)gl * 2 * SB;
    double *oldb = rowb + SB;
    if (!BIGS && stats) {
        for (int i = threadIdx.x; i < S * T; i += EV_THREADS) {
            const int s = i / T, t = i - s * T;
            s_sig[t * SS + s] = __ldg(p.sigma + i);
        }
        __syncthreads();
    }

    Best best_all{-kInf, INT_MAX, INT_MAX};
    const int warp_first = blockIdx.x * GPC + warp * GPW;
    for (int base = warp_first; base < p.C; base += total_groups) {
        const int grp = base + lane / G;
        int b = (grp < p.C) ? __ldg(p.cand + grp) : -1;
        const bool active = (b >= 0 && b < p.B);
        if (!active) b = 0;

        // ---- A: loads and precedence window (evaluate.py:361-372) ----
        const BlockRow row = p.rows[b];
        const int ab = p.assign[b];
        double unit;
        if (p.flags & PP_LITERAL_VALUE) unit = f64_mul(row.mass, 100.0);
        else if (p.scen < 0) unit = __ldg(p.unit_mean + b);
        else unit = __ldg(p.vmax + (size_t)b * p.Sp + p.scen);
        double c_t[PER], d_t[PER];
#pragma unroll
        for (int k = 0; k < PER; k++) {
            const int t = tl + k * G;
            const int tc = (t < T) ? t : 0;
            c_t[k] = net ? __ldg(p.cost + (size_t)b * T + tc) : 0.0;
            d_t[k] = __ldg(p.disc + tc);
        }
        const int npred = row.cnt & 0xffff, nnb = npred + (row.cnt >> 16);
        int lo = 0, hi = INT_MAX;
        for (int k = tl; k < nnb; k += G) {
            const int tn = p.assign[__ldg(p.adj + row.adj + k)];
            if (k < npred) lo = max(lo, tn < 0 ? INT_MAX : tn);
            else if (tn >= 0) hi = min(hi, tn);
        }
        for (int off = G >> 1; off > 0; off >>= 1) {
            lo = max(lo, __shfl_xor_sync(0xffffffffu, lo, off, G));
            hi = min(hi, __shfl_xor_sync(0xffffffffu, hi, off, G));
        }
        bool pok[PER];
#pragma unroll
        for (int k = 0; k < PER; k++) {
            const int t = tl + k * G;
            pok[k] = active && t < T && lo <= t && t <= hi;
        }

        // ---- B: per-scenario deltas d_s = val_s(b,t) - val_s(b,a[b]) (evaluate.py:380-382
        //      with s=k): expected = np.mean(d), CVaR10 (saa.py:157-164), raw d_s ----
        double ex_t[PER], cv_t[PER];
        if constexpr (STATS_T) {
            if (stats) {
                const double *vrow = p.vmax + (size_t)b * p.Sp;
                const int abc = (ab >= 0 && ab < T) ? ab : 0;
                const double d_ab = __ldg(p.disc + abc);
                const double dc_ab = net ? f64_mul(d_ab, __ldg(p.cost + (size_t)b * T + abc)) : 0.0;
                const bool mined = ab >= 0;
                if constexpr (!BIGS) {
                    __syncwarp();
                    const double *sg_ab = s_sig + (size_t)abc * SS;
                    for (int j = tl; j < S; j += G) {
                        const double x = __ldg(vrow + j);
                        rowb[j] = x;
                        const double v = f64_sub(f64_mul(f64_mul(f64_mul(x, d_ab), sg_ab[j]), row.spatial), dc_ab);
                        oldb[j] = mined ? v : 0.0;  // x - 0.0 == x: subtracting it is exact
                    }
                    __syncwarp();
                    const int main_ = S & ~7;
#pragma unroll
                    for (int k = 0; k < PER; k++) {
                        ex_t[k] = -kInf;
                        cv_t[k] = -kInf;
                        if (!pok[k]) continue;
                        const int t = tl + k * G;
                        const double dk = d_t[k], sp = row.spatial;
                        const double dc = net ? f64_mul(dk, c_t[k]) : 0.0;
                        const double *sg = s_sig + (size_t)t * SS;
                        float *sd = SCEN ? p.scen_delta + (size_t)grp * S * T + t : nullptr;
                        double r[8];
#pragma unroll
                        for (int j = 0; j < 8; j++) r[j] = -0.0;
                        TopK<KC> tk;
                        tk.init();
                        // numpy pairwise, single leaf (S <= 128): accumulator j takes s = j (mod 8)
                        for (int s8 = 0; s8 < main_; s8 += 8) {
#pragma unroll
                            for (int j = 0; j < 8; j++) {
                                const int s = s8 + j;
                                const double v = f64_sub(
                                    f64_sub(f64_mul(f64_mul(f64_mul(rowb[s], dk), sg[s]), sp), dc), oldb[s]);
                                r[j] = f64_add(r[j], v);
                                tk.push(v);
                                if constexpr (SCEN) sd[(size_t)s * T] = (float)v;
                            }
                        }
                        double res = main_ ? tree8(r) : -0.0;
                        for (int s = main_; s < S; s++) {
                            const double v =
                                f64_sub(f64_sub(f64_mul(f64_mul(f64_mul(rowb[s], dk), sg[s]), sp), dc), oldb[s]);
                            res = f64_add(res, v);
                            tk.push(v);
                            if constexpr (SCEN) sd[(size_t)s * T] = (float)v;
                        }
                        ex_t[k] = f64_div(f64_add(0.0, res), (double)S);
                        cv_t[k] = tk.mean(p.cvar_k);
                    }
                } else {
                    // S > 128: numpy's multi-leaf recursion, rows staged 32 scenarios at a time,
                    // sigma read from global [S][T]
#pragma unroll
                    for (int k = 0; k < PER; k++) {
                        ex_t[k] = -kInf;
                        cv_t[k] = -kInf;
                    }
#pragma unroll
                    for (int k = 0; k < PER; k++) {
                        const int t = tl + k * G;
                        const int tc = (t < T) ? t : 0;
                        const bool ok = pok[k];
                        const double dc_t = net ? f64_mul(d_t[k], c_t[k]) : 0.0;
                        PwStream acc;
                        acc.begin(p.plan);
                        TopK<KC> tk;
                        tk.init();
                        for (int s0 = 0; s0 < S; s0 += 32) {
                            __syncwarp();
                            for (int j = tl; j < 32 && s0 + j < S; j += G) {
                                const int s = s0 + j;
                                const double x = __ldg(vrow + s);
                                rowb[j] = x;
                                const double v = f64_sub(
                                    f64_mul(f64_mul(f64_mul(x, d_ab), __ldg(p.sigma + (size_t)s * T + abc)), row.spatial),
                                    dc_ab);
                                oldb[j] = mined ? v : 0.0;
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
                                            dlt = f64_sub(
                                                f64_sub(f64_mul(f64_mul(f64_mul(rowb[s - s0], d_t[k]),
                                                                        __ldg(p.sigma + (size_t)s * T + tc)),
                                                                row.spatial),
                                                        dc_t),
                                                oldb[s - s0]);
                                            tk.push(dlt);
                                            if constexpr (SCEN)
                                                p.scen_delta[((size_t)grp * S + s) * T + t] = (float)dlt;
                                        }
                                        x[j] = dlt;
                                    }
                                    acc.block(s8, x, min(8, s_end - s8), p.plan);
                                }
                            }
                        }
                        if (ok) {
                            ex_t[k] = acc.mean(p.plan);
                            cv_t[k] = tk.mean(p.cvar_k);
                        }
                    }
                }
            }
        }

        // ---- C: capacity against the period masses (evaluate.py:373-378) ----
        asm volatile("griddepcontrol.wait;" ::: "memory");
        Best mine{-kInf, INT_MAX, INT_MAX};
#pragma unroll
        for (int k = 0; k < PER; k++) {
            const int t = tl + k * G;
            const int tc = (t < T) ? t : 0;
            bool ok = pok[k];
            if (ok) {
                double load = f64_add(__ldcg(p.pm + tc), row.mass);
                if (ab == t) load = f64_sub(load, row.mass);
                if (load > __ldg(p.cap + tc)) ok = false;
            }
            double v = -kInf;
            if (ok) {
                v = f64_mul(f64_mul(f64_mul(unit, d_t[k]), __ldg(p.sig_row + tc)), row.spatial);
                if (net) v = f64_sub(v, f64_mul(d_t[k], c_t[k]));
            }
            if (active && t < T) {
                const size_t m = (size_t)grp * T + t;
                if (p.trace_val) p.trace_val[m] = v;
                if (p.trace_feas) p.trace_feas[m] = ok ? 1 : 0;
                if constexpr (STATS_T) {
                    if (stats) {
                        if (p.exp_delta) p.exp_delta[m] = ok ? ex_t[k] : -kInf;
                        if (p.cvar) p.cvar[m] = ok ? cv_t[k] : -kInf;
                        if constexpr (SCEN) {
                            if (!ok)  // infeasible: overwrite (or fill) the raw deltas with -inf
                                for (int s = 0; s < S; s++)
                                    p.scen_delta[((size_t)grp * S + s) * T + t] = -__int_as_float(0x7f800000);
                        }
                    }
                }
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
            if (cand_ok) {
                Best cb{mine.v, b, mine.t};
                if (better(cb, best_all)) best_all = cb;
            }
        }
    }
    // K4: grid argmax over candidates (evaluate.py:404-421 order)
    grid_argmax(best_all, s_red, p.partial, p.counter, p.global);
}

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
    int sig, vrow, old, cost, row, unit, ex, cv, b, ab, lo, hi, total;
};

static __host__ __device__ inline int align16(int x) { return (x + 15) & ~15; }

static __host__ __device__ inline StagedLayout staged_layout(int NB, int T, int S, int Sp, int GPC, bool stats,
                                                             bool need_vrow, bool net) {
    StagedLayout L;
    int o = 0;
    const int SS = S | 1;
    L.sig = o;
    o += stats ? align16(8 * T * SS) : 0;
    L.vrow = o;
    o += need_vrow ? align16(8 * NB * Sp) : 0;
    L.old = o;
    o += stats ? align16(8 * GPC * Sp) : 0;
    L.cost = o;
    o += net ? align16(8 * NB * T) : 0;
    L.row = o;
    o += align16(32 * NB);
    L.unit = o;
    o += align16(8 * NB);
    L.ex = o;
    o += stats ? align16(8 * NB * T) : 0;
    L.cv = o;
    o += stats ? align16(8 * NB * T) : 0;
    L.b = o;
    o += align16(4 * NB);
    L.ab = o;
    o += align16(4 * NB);
    L.lo = o;
    o += align16(4 * NB);
    L.hi = o;
    o += align16(4 * NB);
    L.total = o;
    return L;
}

template <int KC, bool SCEN>
__global__ void __launch_bounds__(EV_THREADS) k_eval_staged(const EvalParams p, const int G, const int NB) {
    extern __shared__ __align__(16) unsigned char st_dyn[];
    __shared__ Best s_red[EV_THREADS / 32];
    const int T = p.T, S = p.S, Sp = p.Sp, SS = S | 1;
    const int GPW = 32 / G, GPC = (EV_THREADS / 32) * GPW;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
    const int tl = lane & (G - 1);
    const int gl = warp * GPW + lane / G;
    const bool net = p.flags & PP_NET_MINING_COST;
    const bool literal = p.flags & PP_LITERAL_VALUE;
    constexpr bool STATS_T = KC > 0;
    const bool stats = STATS_T && (SCEN || p.exp_delta || p.cvar);
    const bool need_vrow = stats || (!literal && p.scen >= 0);
    const StagedLayout L = staged_layout(NB, T, S, Sp, GPC, stats, need_vrow, net);
    double *s_sig = reinterpret_cast<double *>(st_dyn + L.sig);
    double *s_vrow = reinterpret_cast<double *>(st_dyn + L.vrow);
    double *s_old = reinterpret_cast<double *>(st_dyn + L.old);
    double *s_cost = reinterpret_cast<double *>(st_dyn + L.cost);
    BlockRow *s_row = reinterpret_cast<BlockRow *>(st_dyn + L.row);
    double *s_unit = reinterpret_cast<double *>(st_dyn + L.unit);
    double *s_ex = reinterpret_cast<double *>(st_dyn + L.ex);
    double *s_cv = reinterpret_cast<double *>(st_dyn + L.cv);
    int *s_b = reinterpret_cast<int *>(st_dyn + L.b);
    int *s_ab = reinterpret_cast<int *>(st_dyn + L.ab);
    int *s_lo = reinterpret_cast<int *>(st_dyn + L.lo);
    int *s_hi = reinterpret_cast<int *>(st_dyn + L.hi);
    const int c0 = blockIdx.x * NB;

    // ---- stage 1: candidate ids (and sigma, transposed to [T][SS]) ----
    for (int i = tid; i < NB; i += EV_THREADS) {
        const int g = c0 + i;
        int b = (g < p.C) ? __ldg(p.cand + g) : -1;
        if (b >= p.B) b = -1;
        s_b[i] = b;
    }
    if (stats)
        for (int i = tid; i < S * T; i += EV_THREADS) {
            const int s = i / T, t = i - s * T;
            s_sig[t * SS + s] = __ldg(p.sigma + i);
        }
    __syncthreads();

    // ---- stage 2: per-candidate rows, one warp per candidate, lanes over 4..16-byte pieces ----
    {
        const int n_cost = net ? T : 0;
        const int n_vrow = need_vrow ? (Sp >> 1) : 0;
        const bool want_unit = !literal && p.scen < 0;
        const int nops = 3 + (want_unit ? 1 : 0) + n_cost + n_vrow;
        for (int i = warp; i < NB; i += EV_THREADS / 32) {
            const int bb = s_b[i];
            const int b = bb < 0 ? 0 : bb;
            for (int op = lane; op < nops; op += 32) {
                if (op < 2) {
                    cp_async16(reinterpret_cast<char *>(s_row + i) + 16 * op,
                               reinterpret_cast<const char *>(p.rows + b) + 16 * op);
                } else if (op == 2) {
                    cp_async4(s_ab + i, p.assign + b);
                } else {
                    int q = op - 3;
                    if (want_unit) {
                        if (q == 0) {
                            cp_async8(s_unit + i, p.unit_mean + b);
                            continue;
                        }
                        q -= 1;
                    }
                    if (q < n_cost) cp_async8(s_cost + (size_t)i * T + q, p.cost + (size_t)b * T + q);
                    else {
                        q -= n_cost;
                        cp_async16(s_vrow + (size_t)i * Sp + 2 * q, p.vmax + (size_t)b * Sp + 2 * q);
                    }
                }
            }
        }
        cp_async_wait_all();
    }
    __syncthreads();

    // ---- stage 3: precedence window per candidate (evaluate.py:361-372), one warp each ----
    for (int i = warp; i < NB; i += EV_THREADS / 32) {
        const BlockRow r = s_row[i];
        const int npred = r.cnt & 0xffff, nnb = npred + (r.cnt >> 16);
        int lo = 0, hi = INT_MAX;
        if (lane < nnb) {
            const int tn = p.assign[__ldg(p.adj + r.adj + lane)];
            if (lane < npred) lo = (tn < 0) ? INT_MAX : tn;
            else if (tn >= 0) hi = tn;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = max(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = min(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) {
            s_lo[i] = lo;
            s_hi[i] = hi;
            if (s_b[i] < 0) s_lo[i] = INT_MAX;  // inactive slot: nothing feasible
            if (!literal && p.scen >= 0) s_unit[i] = s_vrow[(size_t)i * Sp + p.scen];
            if (literal) s_unit[i] = f64_mul(r.mass, 100.0);
        }
    }
    __syncthreads();

    // ---- B: per-scenario deltas for precedence-feasible periods (no period masses needed) ----
    const int t = tl;
    const bool lane_t = t < T;
    const double d_t = __ldg(p.disc + (lane_t ? t : 0));
    if constexpr (STATS_T) {
        if (stats) {
            double *oldb = s_old + (size_t)gl * Sp;
            const int main_ = S & ~7;
            for (int i = gl; i < NB; i += GPC) {
                const int b = s_b[i];
                const BlockRow r = s_row[i];
                const int ab = s_ab[i];
                const bool mined = ab >= 0;
                const int abc = (ab >= 0 && ab < T) ? ab : 0;
                const double *rowb = s_vrow + (size_t)i * Sp;
                const double d_ab = __ldg(p.disc + abc);
                const double dc_ab = net ? f64_mul(d_ab, s_cost[(size_t)i * T + abc]) : 0.0;
                const double *sg_ab = s_sig + (size_t)abc * SS;
                __syncwarp();
                for (int j = tl; j < S; j += G) {
                    const double v = f64_sub(f64_mul(f64_mul(f64_mul(rowb[j], d_ab), sg_ab[j]), r.spatial), dc_ab);
                    oldb[j] = mined ? v : 0.0;  // x - 0.0 == x
                }
                __syncwarp();
                const bool pok = lane_t && b >= 0 && s_lo[i] <= t && t <= s_hi[i];
                if (!pok) continue;
                const double dc = net ? f64_mul(d_t, s_cost[(size_t)i * T + t]) : 0.0;
                const double sp = r.spatial;
                const double *sg = s_sig + (size_t)t * SS;
                float *sd = SCEN ? p.scen_delta + (size_t)(c0 + i) * S * T + t : nullptr;
                double acc[8];
#pragma unroll
                for (int j = 0; j < 8; j++) acc[j] = -0.0;
                TopK<KC> tk;
                tk.init();
                for (int s8 = 0; s8 < main_; s8 += 8) {
#pragma unroll
                    for (int j = 0; j < 8; j++) {
                        const int s = s8 + j;
                        const double v =
                            f64_sub(f64_sub(f64_mul(f64_mul(f64_mul(rowb[s], d_t), sg[s]), sp), dc), oldb[s]);
                        acc[j] = f64_add(acc[j], v);
                        tk.push(v);
                        if constexpr (SCEN) sd[(size_t)s * T] = (float)v;
                    }
                }
                double res = main_ ? tree8(acc) : -0.0;
                for (int s = main_; s < S; s++) {
                    const double v = f64_sub(f64_sub(f64_mul(f64_mul(f64_mul(rowb[s], d_t), sg[s]), sp), dc), oldb[s]);
                    res = f64_add(res, v);
                    tk.push(v);
                    if constexpr (SCEN) sd[(size_t)s * T] = (float)v;
                }
                s_ex[(size_t)i * T + t] = f64_div(f64_add(0.0, res), (double)S);
                s_cv[(size_t)i * T + t] = tk.mean(p.cvar_k);
            }
        }
    }

    // ---- C: capacity (evaluate.py:373-378), parity value, outputs, argmax ----
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const double pm_t = lane_t ? __ldcg(p.pm + t) : 0.0;
    const double cap_t = __ldg(p.cap + (lane_t ? t : 0));
    const double sr_t = __ldg(p.sig_row + (lane_t ? t : 0));
    Best best_all{-kInf, INT_MAX, INT_MAX};
    for (int i = gl; i < NB; i += GPC) {
        const int b = s_b[i];
        const int grp = c0 + i;
        const bool active = b >= 0;
        const BlockRow r = s_row[i];
        const int ab = s_ab[i];
        bool ok = active && lane_t && s_lo[i] <= t && t <= s_hi[i];
        if (ok) {
            double load = f64_add(pm_t, r.mass);
            if (ab == t) load = f64_sub(load, r.mass);
            if (load > cap_t) ok = false;
        }
        double v = -kInf;
        if (ok) {
            v = f64_mul(f64_mul(f64_mul(s_unit[i], d_t), sr_t), r.spatial);
            if (net) v = f64_sub(v, f64_mul(d_t, s_cost[(size_t)i * T + t]));
        }
        if (active && lane_t) {
            const size_t m = (size_t)grp * T + t;
            if (p.trace_val) p.trace_val[m] = v;
            if (p.trace_feas) p.trace_feas[m] = ok ? 1 : 0;
            if constexpr (STATS_T) {
                if (stats) {
                    if (p.exp_delta) p.exp_delta[m] = ok ? s_ex[(size_t)i * T + t] : -kInf;
                    if (p.cvar) p.cvar[m] = ok ? s_cv[(size_t)i * T + t] : -kInf;
                    if constexpr (SCEN) {
                        if (!ok)
                            for (int s = 0; s < S; s++)
                                p.scen_delta[((size_t)grp * S + s) * T + t] = -__int_as_float(0x7f800000);
                    }
                }
            }
        }
        Best mine{-kInf, INT_MAX, INT_MAX};
        if (ok) {
            mine.v = v;
            mine.t = t;
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
            if (cand_ok) {
                Best cb{mine.v, b, mine.t};
                if (better(cb, best_all)) best_all = cb;
            }
        }
    }
    grid_argmax(best_all, s_red, p.partial, p.counter, p.global);
}



// dynamic shared memory of k_eval_candidates: sigma [T][S|1] + per-group row buffers
static size_t eval_smem(int S, int Sp, int T, int G, bool stats, bool bigs) {
    if (!stats) return 0;
    const int gpc = (EV_THREADS / 32) * (32 / G);
    size_t rows = sizeof(double) * (size_t)gpc * 2 * (bigs ? 32 : Sp);
    size_t sig = bigs ? 0 : sizeof(double) * (size_t)T * (S | 1);
    return rows + sig;
}

template <typename K>
static int set_smem_attr(K kern, size_t bytes) {
    if (bytes > 48 * 1024) CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    return PP_OK;
}

// resident CTAs of a kernel at this smem size (cached per instantiation)
template <typename K>
static int resident_ctas(K kern, size_t smem, int device) {
    int per_sm = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, EV_THREADS, smem) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || sms < 1) sms = 148;
    return per_sm * sms;
}

template <int PER, int KC, bool BIGS, bool SCEN>
static int launch_cand1(int ngroups, int G, size_t smem, cudaStream_t st, bool pdl, int device, const EvalParams &ep) {
    auto kern = k_eval_candidates<PER, KC, BIGS, SCEN>;
    TRY(set_smem_attr(kern, smem));
    const int gpc = (EV_THREADS / 32) * (32 / G);
    const int need = std::max(1, (ngroups + gpc - 1) / gpc);
    const int grid = std::min(need, resident_ctas(kern, smem, device));
    return launch_eval(kern, grid, smem, st, pdl, ep, G, grid * gpc);
}

// general path (T > 32, S > 128 or degree > 32): the 128-slot top-k covers every k
template <int PER>
static int launch_cand_kc(int kc, bool bigs, bool scen, int ngroups, int G, size_t smem, cudaStream_t st, bool pdl,
                          int device, const EvalParams &ep) {
    if (kc == 0) return launch_cand1<PER, 0, false, false>(ngroups, G, smem, st, pdl, device, ep);
    if (bigs)
        return scen ? launch_cand1<PER, 128, true, true>(ngroups, G, smem, st, pdl, device, ep)
                    : launch_cand1<PER, 128, true, false>(ngroups, G, smem, st, pdl, device, ep);
    return scen ? launch_cand1<PER, 128, false, true>(ngroups, G, smem, st, pdl, device, ep)
                : launch_cand1<PER, 128, false, false>(ngroups, G, smem, st, pdl, device, ep);
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
    if (T <= 32 && (!stats || S <= 128) && c->deg_max <= 32) {
        const int gpc_s = (EV_THREADS / 32) * (32 / G);
        const int NB = std::max(32, gpc_s);
        const bool need_vrow = stats || (!(flags & PP_LITERAL_VALUE) && scenario >= 0);
        const StagedLayout Ls = staged_layout(NB, T, S, c->Sp, gpc_s, stats, need_vrow, (flags & PP_NET_MINING_COST) != 0);
        if (Ls.total <= 200 * 1024) {
            const int sgrid = std::max(1, (C + NB - 1) / NB);
            TRY(ensure_grid_scratch(c, sgrid));
            bool pdl;
            TRY(refresh_pm(c, st, &pdl));
            const bool scen = o.scen_delta != nullptr;
            const size_t smem_s = (size_t)Ls.total;
#define PP_STAGED(KC, SC)                                                                  \
    {                                                                                      \
        TRY(set_smem_attr(k_eval_staged<KC, SC>, smem_s));                                 \
        TRY(launch_eval(k_eval_staged<KC, SC>, sgrid, smem_s, st, pdl, ep, G, NB));        \
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
    const bool bigs = S > 128;
    const size_t smem = eval_smem(S, c->Sp, T, G, stats, bigs);
    if (smem > 227 * 1024) return fail(PP_ERR_INVALID_ARGS, "n_periods x n_scenarios too large for shared staging");
    bool pdl;
    TRY(refresh_pm(c, st, &pdl));
    const bool scen = o.scen_delta != nullptr;
    if (PER == 1) TRY(launch_cand_kc<1>(kc, bigs, scen, C, G, smem, st, pdl, c->device, ep));
    else TRY(launch_cand_kc<4>(kc, bigs, scen, C, G, smem, st, pdl, c->device, ep));
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
