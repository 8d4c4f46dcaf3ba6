// pp_moves.cu -- explicit reassign / unmine / swap move evaluation and pp_eval_moves.
#include "pp_internal.cuh"

// ------------------------------------------------------------------------------------
// explicit moves (reassign / unmine / swap), one thread per move
// ------------------------------------------------------------------------------------

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

// The precedence windows of the warp's 32 moves, the warp together (the padded neighbour rows: lane k
// = neighbour k, coalesced), eight moves per round with every row load and then every period load
// issued before use -- two memory round trips per eight moves instead of a dependent chain of
// loads per neighbour in each lane.  Move m of the warp asks for block bw (lane m's value; -1:
// none), with block sub (if it is a neighbour) seen at period subt; lane m gets lo = the latest
// predecessor period (-2: an unmined predecessor) and hi = the earliest mined successor period
// (INT_MAX: none) -- the quantities of move_window / hybrid.py:348-355.
constexpr int MV_NBR_W = 32, MV_NBR_SUCC = 1 << 30;
__device__ __forceinline__ void warp_windows(const MoveParams &p, int bw, int sub, int subt, int &lo_out, int &hi_out) {
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    lo_out = 0;
    hi_out = INT_MAX;
#pragma unroll 1
    for (int m0 = 0; m0 < 32; m0 += 8) {
        int nb[8], bb[8], sb[8], st[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            bb[u] = __shfl_sync(FULL, bw, m0 + u);
            sb[u] = __shfl_sync(FULL, sub, m0 + u);
            st[u] = __shfl_sync(FULL, subt, m0 + u);
            nb[u] = bb[u] >= 0 ? __ldg(p.nbr + (size_t)bb[u] * MV_NBR_W + lane) : -1;
        }
        int tn[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const int b = nb[u] >= 0 ? (nb[u] & (MV_NBR_SUCC - 1)) : 0;
            tn[u] = nb[u] >= 0 ? (b == sb[u] ? st[u] : p.assign[b]) : 0;
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const bool pred = nb[u] >= 0 && !(nb[u] & MV_NBR_SUCC), succ = nb[u] >= 0 && (nb[u] & MV_NBR_SUCC);
            const unsigned lc = pred ? (tn[u] < 0 ? 0x7fffffffu : (unsigned)tn[u]) : 0u;
            const unsigned hc = (succ && tn[u] >= 0) ? (unsigned)tn[u] : 0x7fffffffu;
            const int lo = (int)__reduce_max_sync(FULL, lc);
            const int hi = (int)__reduce_min_sync(FULL, hc);
            if (lane == m0 + u) {
                lo_out = lo == 0x7fffffff ? -2 : lo;
                hi_out = hi;
            }
        }
    }
}

// Every block's precedence window under the current schedule, a warp per 32 blocks: batches hold
// several moves per block (250k moves over 50k blocks at C2), so one window per block replaces one
// (or, for swaps, two) per move.  Per block, three int2: {lo, hi} raw (lo = the latest predecessor
// period, 0x7fffffff when a predecessor is unmined; hi = the earliest mined successor period,
// 0x7fffffff when none), {lob, hib} = a neighbour block attaining each, {lo2, hi2} = the same
// extremes without that one neighbour -- so a swap can re-form the window with its partner seen at
// another period.  Launched behind the period masses under PDL; it completes only after them, so
// the moves kernel's griddepcontrol.wait covers both.
constexpr int BW_NONE = 0x7fffffff;
__global__ void __launch_bounds__(256) k_block_windows(const MoveParams p, int2 *__restrict__ win) {
    asm volatile("griddepcontrol.launch_dependents;");
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    for (int base = (blockIdx.x * 8 + (threadIdx.x >> 5)) * 32; base < p.B; base += gridDim.x * 256) {
        int2 w0 = make_int2(0, BW_NONE), w1 = make_int2(-1, -1), w2 = make_int2(0, BW_NONE);
#pragma unroll 1
        for (int m0 = 0; m0 < 32; m0 += 8) {
            int nb[8], tn[8];
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const int b = base + m0 + u;
                nb[u] = b < p.B ? __ldg(p.nbr + (size_t)b * MV_NBR_W + lane) : -1;
            }
#pragma unroll
            for (int u = 0; u < 8; u++) tn[u] = nb[u] >= 0 ? p.assign[nb[u] & (MV_NBR_SUCC - 1)] : 0;
#pragma unroll
            for (int u = 0; u < 8; u++) {
                const bool pred = nb[u] >= 0 && !(nb[u] & MV_NBR_SUCC), succ = nb[u] >= 0 && (nb[u] & MV_NBR_SUCC);
                const int blk = nb[u] & (MV_NBR_SUCC - 1);
                const unsigned lc = pred ? (tn[u] < 0 ? (unsigned)BW_NONE : (unsigned)tn[u]) : 0u;
                const unsigned hc = (succ && tn[u] >= 0) ? (unsigned)tn[u] : (unsigned)BW_NONE;
                const unsigned lo = __reduce_max_sync(FULL, lc), hi = __reduce_min_sync(FULL, hc);
                const unsigned ml = __ballot_sync(FULL, pred && lc == lo);
                const unsigned mh = __ballot_sync(FULL, succ && tn[u] >= 0 && hc == hi);
                const int ll = ml ? __ffs(ml) - 1 : -1, lh = mh ? __ffs(mh) - 1 : -1;
                const int lob = __shfl_sync(FULL, blk, ll < 0 ? 0 : ll), hib = __shfl_sync(FULL, blk, lh < 0 ? 0 : lh);
                const unsigned lo2 = __reduce_max_sync(FULL, lane == ll ? 0u : lc);
                const unsigned hi2 = __reduce_min_sync(FULL, lane == lh ? (unsigned)BW_NONE : hc);
                if (lane == m0 + u) {
                    w0 = make_int2((int)lo, (int)hi);
                    w1 = make_int2(ll < 0 ? -1 : lob, lh < 0 ? -1 : hib);
                    w2 = make_int2((int)lo2, (int)hi2);
                }
            }
        }
        const int b = base + lane;
        if (b < p.B) {
            win[3 * (size_t)b] = w0;
            win[3 * (size_t)b + 1] = w1;
            win[3 * (size_t)b + 2] = w2;
        }
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Swaps: where block sub sits in bw's neighbour row (lane m asks for its own pair): 1 = a
// predecessor of bw, 2 = a successor, 0 = neither; eight rows per round, one memory round trip
__device__ __forceinline__ int warp_relation(const MoveParams &p, int bw, int sub) {
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    int rel = 0;
#pragma unroll 1
    for (int m0 = 0; m0 < 32; m0 += 8) {
        int nb[8], sb[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const int bb = __shfl_sync(FULL, bw, m0 + u);
            sb[u] = __shfl_sync(FULL, sub, m0 + u);
            nb[u] = bb >= 0 ? __ldg(p.nbr + (size_t)bb * MV_NBR_W + lane) : -1;
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const bool hit = nb[u] >= 0 && (nb[u] & (MV_NBR_SUCC - 1)) == sb[u];
            const unsigned m = __ballot_sync(FULL, hit), ms = __ballot_sync(FULL, hit && (nb[u] & MV_NBR_SUCC));
            if (lane == m0 + u) rel = ms ? 2 : (m ? 1 : 0);
        }
    }
    return rel;
}
// block b's window (k_block_windows) with neighbour o (relation rel: 1 pred, 2 succ) seen at period
// to, in warp_windows' convention (lo -2 when a predecessor is unmined, hi INT_MAX when none)
__device__ __forceinline__ void window_with(const int2 *win, int b, int o, int rel, int to, int &lo, int &hi) {
    const int2 w0 = __ldcg(win + 3 * (size_t)b);
    int l = w0.x, h = w0.y;
    if (rel != 0) {  // (only then the attaining neighbours and the runners-up)
        const int2 w1 = __ldcg(win + 3 * (size_t)b + 1), w2 = __ldcg(win + 3 * (size_t)b + 2);
        if (rel == 1) {
            const int lw = o == w1.x ? w2.x : w0.x;
            l = lw == BW_NONE ? BW_NONE : max(lw, to);
        } else {
            const int hw = o == w1.y ? w2.y : w0.y;
            h = min(hw, to);
        }
    }
    lo = l == BW_NONE ? -2 : l;
    hi = h;  // BW_NONE == INT_MAX
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
    asm volatile("griddepcontrol.wait;" ::: "memory");
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
                        double load = f64_add(__ldcg(p.pm + t2), r1.mass);
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
                    double l1 = f64_add(f64_sub(__ldcg(p.pm + t1), r1.mass), r2.mass);
                    double l2 = f64_add(f64_sub(__ldcg(p.pm + t2), r2.mass), r1.mass);
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
// k_moves_warp: explicit moves (north_star (1)), persistent warps.
//   feasibility  a lane per move, 32 moves per warp step (coalesced move ids): the window of
//                hybrid.py:348-355 over the block's adjacency (a swap sees its partner at its new
//                period), capacity of the destination periods (hybrid.py:370, 396-399), and the
//                kernel-value delta (the parity key, evaluate.py:379-382 at both periods)
//   statistics   then a warp per FEASIBLE move (the step's ballot, in lane order): lanes own
//                scenarios two at a time, the scenario-major value rows read with 128-bit loads
//                (double2), sigma[S][T] and the T-tables in shared memory; the per-scenario deltas go
//                to the warp's slice, their numpy pairwise mean (8 lanes per leaf) and CVaR10 (warp
//                k-smallest) follow.  Infeasible moves (most of a random batch) cost one lane.
//   argmax       lane -> warp -> CTA -> grid (move index order on ties), one atomic per CTA
// For S <= 256 (CVaR k <= 25); k_eval_moves covers larger scenario sets.
// ------------------------------------------------------------------------------------
constexpr int MW_THREADS = 256;
constexpr int MW_NW = MW_THREADS / 32;

template <bool STATS>
__global__ void __launch_bounds__(MW_THREADS) k_moves_warp(const MoveParams p) {
    extern __shared__ __align__(16) unsigned char mw_dyn[];
    __shared__ Best s_red[MW_NW];
    __shared__ double s_tab[3][32];  // disc, cap, sig_row
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int T = p.T, S = p.S, Sp = p.Sp;
    const int P2 = S <= 32 ? 32 : S <= 64 ? 64 : S <= 128 ? 128 : 256;
    double *s_sig = reinterpret_cast<double *>(mw_dyn);                                   // [S][T]
    double *vb = s_sig + (size_t)(STATS ? S * T : 0) + (size_t)warp * (P2 + kMaxLeaves);  // warp slice
    double *lv = vb + P2;
    if (threadIdx.x < T) {
        s_tab[0][threadIdx.x] = __ldg(p.disc + threadIdx.x);
        s_tab[1][threadIdx.x] = __ldg(p.cap + threadIdx.x);
        s_tab[2][threadIdx.x] = __ldg(p.sig_row + threadIdx.x);
    }
    if (STATS)
        for (int e = threadIdx.x; e < S * T; e += MW_THREADS) s_sig[e] = __ldg(p.sigma + e);
    __syncthreads();
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the period masses (pm) may be in flight
    const bool net = p.flags & PP_NET_MINING_COST;
    Best mine{-kInf, INT_MAX, INT_MAX};
    for (int base = (blockIdx.x * MW_NW + warp) * 32; base < p.M; base += gridDim.x * MW_NW * 32) {
        const int i = base + lane;
        bool ok = false;
        double dl = -kInf;
        int b1 = 0, b2 = -1, t1 = -1, t2 = -1;
        // the warp's windows together (warp-uniform: every lane reaches these shuffles)
        int wlo = 0, whi = INT_MAX, wlo2 = 0, whi2 = INT_MAX;
        if (p.bwin) {  // the blocks' windows, computed once per block
            int bw = -1, sub = -1;
            if (i < p.M) {
                const int x = __ldg(p.ma + i), y = __ldg(p.mb + i);
                if (p.kind == PP_MOVE_REASSIGN) {
                    if (x >= 0 && x < p.B && y >= -1 && y < p.T) window_with(p.bwin, x, -1, 0, 0, wlo, whi);
                } else if (x >= 0 && x < p.B && y >= 0 && y < p.B && x != y) {
                    bw = x;
                    sub = y;
                }
            }
            if (p.kind == PP_MOVE_SWAP) {  // b1's window with b2 at b1's period, and the other way round
                const int rel = warp_relation(p, bw, sub);
                if (bw >= 0) {
                    window_with(p.bwin, bw, sub, rel, p.assign[bw], wlo, whi);
                    window_with(p.bwin, sub, bw, rel == 1 ? 2 : rel == 2 ? 1 : 0, p.assign[sub], wlo2, whi2);
                }
            }
        } else if (p.nbr) {
            int bw = -1, sub = -1, subt = 0, bw2 = -1, sub2 = -1, subt2 = 0;
            if (i < p.M) {
                const int x = __ldg(p.ma + i), y = __ldg(p.mb + i);
                if (p.kind == PP_MOVE_REASSIGN) {
                    if (x >= 0 && x < p.B && y >= -1 && y < p.T) bw = x;
                } else if (x >= 0 && x < p.B && y >= 0 && y < p.B && x != y) {
                    bw = x;  // b1's window with b2 at b1's period, and the other way round
                    sub = y;
                    subt = p.assign[x];
                    bw2 = y;
                    sub2 = x;
                    subt2 = p.assign[y];
                }
            }
            warp_windows(p, bw, sub, subt, wlo, whi);
            if (p.kind == PP_MOVE_SWAP) warp_windows(p, bw2, sub2, subt2, wlo2, whi2);
        }
        if (i < p.M) {
            const int x = __ldg(p.ma + i), y = __ldg(p.mb + i);
            if (p.kind == PP_MOVE_REASSIGN) {
                if (x >= 0 && x < p.B && y >= -1 && y < p.T) {
                    b1 = x;
                    const BlockRow r1 = p.rows[b1];
                    t1 = p.assign[b1];
                    t2 = y;
                    const int npred = r1.cnt & 0xffff, nnb = npred + (r1.cnt >> 16);
                    if (t2 == t1) {
                        ok = false;
                    } else if (p.nbr || p.bwin) {  // from the warp's windows / the block windows
                        ok = t2 < 0 ? whi == INT_MAX : (wlo != -2 && wlo <= t2 && t2 <= whi);
                        if (ok && t2 >= 0 && f64_add(__ldcg(p.pm + t2), r1.mass) > s_tab[1][t2]) ok = false;
                    } else if (t2 < 0) {  // unmine: allowed iff no mined successor
                        ok = true;
                        for (int k = npred; k < nnb; k++)
                            if (p.assign[__ldg(p.adj + r1.adj + k)] >= 0) ok = false;
                    } else {
                        ok = true;
                        for (int k = 0; k < nnb; k++) {
                            const int tn = p.assign[__ldg(p.adj + r1.adj + k)];
                            if (k < npred) {
                                if (tn < 0 || tn > t2) ok = false;
                            } else if (tn >= 0 && tn < t2) {
                                ok = false;
                            }
                        }
                        if (ok && f64_add(__ldcg(p.pm + t2), r1.mass) > s_tab[1][t2]) ok = false;
                    }
                    if (ok) {
                        const double vn = (t2 >= 0) ? kernel_value(p, r1, b1, t2) : 0.0;
                        const double vo = (t1 >= 0) ? kernel_value(p, r1, b1, t1) : 0.0;
                        dl = f64_sub(vn, vo);
                    }
                }
            } else if (x >= 0 && x < p.B && y >= 0 && y < p.B && x != y) {
                b1 = x;
                b2 = y;
                const BlockRow r1 = p.rows[b1], r2 = p.rows[b2];
                t1 = p.assign[b1];
                t2 = p.assign[b2];
                if (t1 >= 0 && t2 >= 0 && t1 != t2) {
                    const double l1 = f64_add(f64_sub(__ldcg(p.pm + t1), r1.mass), r2.mass);
                    const double l2 = f64_add(f64_sub(__ldcg(p.pm + t2), r2.mass), r1.mass);
                    if (!(l1 > s_tab[1][t1]) && !(l2 > s_tab[1][t2])) {
                        int lo1, hi1, lo2, hi2;  // windows after the swap (hybrid.py:400-403)
                        if (p.nbr || p.bwin) {
                            lo1 = wlo;
                            hi1 = whi == INT_MAX ? p.T - 1 : whi;
                            lo2 = wlo2;
                            hi2 = whi2 == INT_MAX ? p.T - 1 : whi2;
                        } else {
                            move_window(p, r1, b2, t1, lo1, hi1);
                            move_window(p, r2, b1, t2, lo2, hi2);
                        }
                        ok = lo1 != -2 && lo1 <= t2 && t2 <= hi1 && lo2 != -2 && lo2 <= t1 && t1 <= hi2;
                    }
                }
                if (ok) {
                    const double v12 = kernel_value(p, r1, b1, t2), v11 = kernel_value(p, r1, b1, t1);
                    const double v21 = kernel_value(p, r2, b2, t1), v22 = kernel_value(p, r2, b2, t2);
                    dl = f64_add(f64_sub(v12, v11), f64_sub(v21, v22));
                }
            }
            p.feas[i] = ok ? 1 : 0;
            p.delta[i] = dl;
            if (ok) {
                const Best cb{dl, i, -1};
                if (better(cb, mine)) mine = cb;
            } else if (STATS) {
                if (p.exp_delta) p.exp_delta[i] = -kInf;
                if (p.cvar) p.cvar[i] = -kInf;
                if (p.scen_delta)
                    for (int s_ = 0; s_ < S; s_++) p.scen_delta[(size_t)i * S + s_] = -__int_as_float(0x7f800000);
            }
        }
        // statistics of this step's feasible moves, the warp on one move at a time
        for (unsigned fm = STATS ? __ballot_sync(FULL, ok) : 0u; fm; fm &= fm - 1) {
            const int src = __ffs(fm) - 1;
            const int mi = base + src;
            const int c1 = __shfl_sync(FULL, b1, src), c2 = __shfl_sync(FULL, b2, src);
            const int u1 = __shfl_sync(FULL, t1, src), u2 = __shfl_sync(FULL, t2, src);
            auto sval = [&](double x_, int t, int s_, double sp, double dc) {
                return f64_sub(f64_mul(f64_mul(f64_mul(x_, s_tab[0][t]), s_sig[s_ * T + t]), sp), dc);
            };
            const double sp1 = __ldg(&p.rows[c1].spatial);
            const double sp2 = c2 >= 0 ? __ldg(&p.rows[c2].spatial) : 0.0;
            const double k11 = (net && u1 >= 0) ? f64_mul(s_tab[0][u1], __ldg(p.cost + (size_t)c1 * T + u1)) : 0.0;
            const double k12 = (net && u2 >= 0) ? f64_mul(s_tab[0][u2], __ldg(p.cost + (size_t)c1 * T + u2)) : 0.0;
            const double k21 = (net && c2 >= 0) ? f64_mul(s_tab[0][u1], __ldg(p.cost + (size_t)c2 * T + u1)) : 0.0;
            const double k22 = (net && c2 >= 0) ? f64_mul(s_tab[0][u2], __ldg(p.cost + (size_t)c2 * T + u2)) : 0.0;
            for (int s0 = 2 * lane; s0 < S; s0 += 64) {  // lane: scenarios s0, s0 + 1 (one 128-bit load per row)
                const double2 w1 = __ldg(reinterpret_cast<const double2 *>(p.vmax + (size_t)c1 * Sp + s0));
                double2 w2 = make_double2(0.0, 0.0);
                if (p.kind == PP_MOVE_SWAP) w2 = __ldg(reinterpret_cast<const double2 *>(p.vmax + (size_t)c2 * Sp + s0));
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int s_ = s0 + h;
                    if (s_ >= S) break;
                    const double x1 = h ? w1.y : w1.x;
                    double ds;
                    if (p.kind == PP_MOVE_REASSIGN) {
                        ds = (u2 >= 0) ? sval(x1, u2, s_, sp1, k12) : 0.0;
                        if (u1 >= 0) ds = f64_sub(ds, sval(x1, u1, s_, sp1, k11));
                    } else {
                        const double x2 = h ? w2.y : w2.x;
                        ds = f64_add(f64_sub(sval(x1, u2, s_, sp1, k12), sval(x1, u1, s_, sp1, k11)),
                                     f64_sub(sval(x2, u1, s_, sp2, k21), sval(x2, u2, s_, sp2, k22)));
                    }
                    vb[s_] = ds;
                    if (p.scen_delta) p.scen_delta[(size_t)mi * S + s_] = (float)ds;
                }
            }
            __syncwarp();
            const double ex = warp_pairwise_mean(vb, p.plan, lv);
            // the k-smallest scratch reuses the slice (after the mean has read it)
            const double cv = warp_cvar(vb, S, p.cvar_k, reinterpret_cast<unsigned long long *>(vb), P2 >> 5);
            if (lane == 0) {
                if (p.exp_delta) p.exp_delta[mi] = ex;
                if (p.cvar) p.cvar[mi] = cv;
            }
            __syncwarp();
        }
    }
    grid_argmax(mine, s_red, p.partial, p.counter, p.global);
}

extern "C" {

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
    mp.nbr = c->nbr.as<int32_t>();  // (null when a block has more than 32 neighbours)
    mp.assign = c->assign_ptr;
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
    bool pdl;
    TRY(refresh_pm(c, st, &pdl));
    // persistent warps, statistics a warp per feasible move: S <= 256, k <= 25
    static const bool force_thread = std::getenv("PP_MOVES_THREAD") != nullptr;  // diagnostics: A/B the kernels
    const bool warp_path = !force_thread && (!stats || (S <= 256 && c->cvar_k <= 32));
    if (warp_path) {
        const int P2 = S <= 32 ? 32 : S <= 64 ? 64 : S <= 128 ? 128 : 256;
        const size_t smem = sizeof(double) * ((stats ? (size_t)S * T : 0) + (size_t)MW_NW * (P2 + kMaxLeaves));
        int sms = 148;
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device) != cudaSuccess || sms < 1) sms = 148;
        const int wgrid = std::max(1, std::min((M + 32 * MW_NW - 1) / (32 * MW_NW), 8 * sms));
        TRY(ensure_grid_scratch(c, wgrid));  // may re-allocate: take the pointers after it
        mp.partial = c->partial.as<pp_best>();
        mp.counter = c->counter.as<unsigned int>();
        // batches with several moves per block: the windows once per block first
        static const bool no_bwin = std::getenv("PP_NO_BLOCK_WINDOWS") != nullptr;  // diagnostics
        if (mp.nbr && !no_bwin && (long long)M >= 2ll * c->B) {
            TRY(c->mv_win.ensure(3 * sizeof(int2) * (size_t)c->B));
            const int bgrid = std::max(1, std::min((c->B + 255) / 256, 8 * sms));
            TRY(launch_eval_n(k_block_windows, bgrid, 256, 0, st, pdl, mp, c->mv_win.as<int2>()));
            mp.bwin = c->mv_win.as<int2>();
            pdl = true;  // the moves kernel behind the windows (which complete after the masses)
        }
        if (stats) {
            TRY(set_smem_attr(k_moves_warp<true>, smem, c->device));
            TRY(launch_eval_n(k_moves_warp<true>, wgrid, MW_THREADS, smem, st, pdl, mp));
        } else {
            TRY(set_smem_attr(k_moves_warp<false>, smem, c->device));
            TRY(launch_eval_n(k_moves_warp<false>, wgrid, MW_THREADS, smem, st, pdl, mp));
        }
    } else switch (kc) {
        case 0: TRY(launch_eval(k_eval_moves<0>, grid, 0, st, pdl, mp)); break;
        case 2: TRY(launch_eval(k_eval_moves<2>, grid, 0, st, pdl, mp)); break;
        case 8: TRY(launch_eval(k_eval_moves<8>, grid, 0, st, pdl, mp)); break;
        default: TRY(launch_eval(k_eval_moves<128>, grid, 0, st, pdl, mp)); break;
    }
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
        TRY(check_schedule_range(c, false));
    }
    return PP_OK;
}

}  // extern "C"
