// pp_eval_general.cu -- general candidate-evaluation kernel (any T <= 128, S <= 2048, degree):
// persistent lane groups with per-candidate global gathers.  The fast path is in pp_eval.cu.
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
    const bool stats = STATS_T && (SCEN || p.exp_delta || p.cvar || p.n_pairs);
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
                        if (p.n_pairs && ok) {
                            const int q = atomicAdd(p.n_pairs, 1);
                            p.pair_cand[q] = grp;
                            p.pair_period[q] = t;
                            p.pair_exp[q] = ex_t[k];
                            p.pair_cvar[q] = cv_t[k];
                        }
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

// dynamic shared memory of k_eval_candidates: sigma [T][S|1] + per-group row buffers
static size_t eval_smem(int S, int Sp, int T, int G, bool stats, bool bigs) {
    if (!stats) return 0;
    const int gpc = (EV_THREADS / 32) * (32 / G);
    size_t rows = sizeof(double) * (size_t)gpc * 2 * (bigs ? 32 : Sp);
    size_t sig = bigs ? 0 : sizeof(double) * (size_t)T * (S | 1);
    return rows + sig;
}

template <int PER, int KC, bool BIGS, bool SCEN>
static int launch_cand1(int ngroups, int G, size_t smem, cudaStream_t st, bool pdl, int device, const EvalParams &ep) {
    auto kern = k_eval_candidates<PER, KC, BIGS, SCEN>;
    TRY(set_smem_attr(kern, smem, device));
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


// entry point used by pp_eval_candidates for the general path
int launch_general_candidates(int PER, int kc, bool scen, int C, int G, int S, int Sp, int T, bool stats,
                              cudaStream_t st, bool pdl, int device, const EvalParams &ep) {
    const bool bigs = S > 128;
    const size_t smem = eval_smem(S, Sp, T, G, stats, bigs);
    if (smem > 227 * 1024) return fail(PP_ERR_INVALID_ARGS, "n_periods x n_scenarios too large for shared staging");
    if (PER == 1) return launch_cand_kc<1>(kc, bigs, scen, C, G, smem, st, pdl, device, ep);
    return launch_cand_kc<4>(kc, bigs, scen, C, G, smem, st, pdl, device, ep);
}
