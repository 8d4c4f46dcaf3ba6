// pp_eval.cu -- evaluate_candidates_parallel (evaluate.py:306-430): the staged fast-path kernel
// and pp_eval_candidates (which dispatches to pp_eval_general.cu otherwise).
#include "pp_internal.cuh"

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
// k_eval_warp: the fast path of pp_eval_candidates (T <= 32, degree <= 32; S <= 256 when
// statistics are requested).
// Every warp owns CPW consecutive candidates end to end; warps never wait for one another
// until the final CTA argmax, so the SM overlaps one warp's load latency with another's
// arithmetic.  Lane t is period t for the capacity / value / argmax of a candidate
// (evaluate.py:361-388); lane k is neighbour slot k for its precedence window.
//   loads     candidate ids -> {BlockRow, own period, unit, mining-cost row (lane t),
//             vmax row (cp.async to the warp's shared slice), 32 neighbour ids (lane k)}
//             -> neighbour periods; window = redux.sync max / min over the lanes
//   wait      griddepcontrol.wait (the period-mass kernel), lane t loads pm[t]
//   moves     capacity (373-378), value (379-384), lowest-t argmax (387-388) per candidate:
//             ballot of the feasible periods, butterfly argmax, trace row written by lane t
//   stats     KC > 0 (CVaR k <= 8): every precedence-feasible pair, one thread per pair pooled
//             across the CTA, before the wait; KC < 0 (k > 8): every capacity-feasible pair,
//             one warp per pair dealt across the CTA's warps, after it (section 4.1 of DESIGN.md):
//             expected delta (numpy pairwise mean) and CVaR10
//   argmax    warp -> CTA -> deterministic grid argmax (last CTA)
// Everything before the wait is independent of the period masses and overlaps the
// period-mass kernel under programmatic dependent launch.
// ------------------------------------------------------------------------------------
constexpr int CPW = 4;  // candidates per warp
constexpr int WV_THREADS = 256;  // k_eval_warp CTA: 8 warps (128 measured the same)
constexpr int WV_MINB = 4;       // resident CTAs per SM (64 registers per thread)

__device__ __forceinline__ int nth_bit(unsigned m, int k) {  // index of the k-th (0-based) set bit
    for (; k > 0; k--) m &= m - 1;
    return __ffs(m) - 1;
}
constexpr int NBR_W = 32;  // neighbour slots per block (padded table, one 128-byte row)
constexpr int NBR_SUCC = 1 << 30;  // successor tag in the neighbour table; -1 = padding

struct WarpLayout {  // per-warp slice of dynamic shared memory (byte offsets)
    int vrow, cost, val, ex, cv, big, total;
};
// dynamic shared memory: [sigma S x T (statistics)] [NW warp slices]
static __host__ __device__ inline int sig_bytes(int S, int T, bool stats) { return stats ? ((8 * S * T + 15) & ~15) : 0; }
static __host__ __device__ inline int align16(int x) { return (x + 15) & ~15; }
// bign: warp-per-move statistics (KC < 0): per-scenario deltas padded to a power of two + leaf sums
static __host__ __device__ inline int big_pow2(int S) {
    int n = 32;
    while (n < S) n <<= 1;
    return n;
}
static __host__ __device__ inline WarpLayout warp_layout(int T, int Sp, bool stats, bool need_vrow, bool net,
                                                         int bign = 0) {
    WarpLayout L;
    int o = 0;
    L.vrow = o;
    o += need_vrow ? align16(8 * CPW * Sp) : 0;
    L.cost = o;
    o += net ? align16(8 * CPW * T) : 0;
    L.val = o;  // per-(candidate, lane) kernel value
    o += 8 * CPW * 32;
    L.ex = o;
    o += stats ? align16(8 * CPW * T) : 0;
    L.cv = o;
    o += stats ? align16(8 * CPW * T) : 0;
    L.big = o;
    o += bign ? align16(8 * (bign + kMaxLeaves)) : 0;
    L.total = o;
    return L;
}


// 128-bit compare-and-swap of a pp_best record {value, block, period} in the selection order of
// evaluate.py:404-409; the initial record {-inf, -1, -1} loses to every selectable move.
__device__ __forceinline__ void best_cas(pp_best *g, const Best &x) {
    unsigned long long *a = reinterpret_cast<unsigned long long *>(g);
    unsigned long long lo = __ldcg(a), hi = __ldcg(a + 1);
    const unsigned long long nlo = (unsigned long long)__double_as_longlong(x.v);
    const unsigned long long nhi = (unsigned long long)(unsigned)x.b | ((unsigned long long)(unsigned)x.t << 32);
    for (;;) {
        const Best cur{__longlong_as_double((long long)lo), (int)(unsigned)(hi & 0xffffffffull), (int)(unsigned)(hi >> 32)};
        if (cur.b >= 0 && !better(x, cur)) return;
        unsigned long long olo, ohi;
        asm volatile(
            "{\n\t.reg .b128 d, c, n;\n\t"
            "mov.b128 c, {%2, %3};\n\t"
            "mov.b128 n, {%4, %5};\n\t"
            "atom.global.cas.b128 d, [%6], c, n;\n\t"
            "mov.b128 {%0, %1}, d;\n\t}"
            : "=l"(olo), "=l"(ohi)
            : "l"(lo), "l"(hi), "l"(nlo), "l"(nhi), "l"(a)
            : "memory");
        if (olo == lo && ohi == hi) return;
        lo = olo;
        hi = ohi;
    }
}

#ifdef PP_EVAL_PROBE
__device__ unsigned long long g_ev_probe[4096][12];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define EV_PROBE(k) do { if (threadIdx.x == 0 && blockIdx.x < 4096) g_ev_probe[blockIdx.x][k] = gtimer(); } while (0)
// per warp: lane 0 of every warp stamps phase k
__device__ unsigned long long g_wp_probe[1024][8][12];
#define WP_PROBE(k) do { if ((threadIdx.x & 31) == 0 && blockIdx.x < 1024) g_wp_probe[blockIdx.x][threadIdx.x >> 5][k] = gtimer(); } while (0)
extern "C" PP_API int pp_debug_warp_probe(unsigned long long *out) {
    return cudaMemcpyFromSymbol(out, g_wp_probe, sizeof(g_wp_probe)) == cudaSuccess ? 0 : 3;
}
#else
#define EV_PROBE(k) do { } while (0)
#define WP_PROBE(k) do { } while (0)
#endif

template <int KC, bool SCEN>
__global__ void __launch_bounds__(WV_THREADS, KC < 0 ? 4 : WV_MINB) k_eval_warp(const EvalParams p) {
    extern __shared__ __align__(16) unsigned char wv_dyn[];
    __shared__ Best s_red[WV_THREADS / 32];
    __shared__ int s_cab[WV_THREADS / 32 * CPW], s_cb[WV_THREADS / 32 * CPW], s_wcnt[WV_THREADS / 32];
    __shared__ double s_csp[WV_THREADS / 32 * CPW], s_cm[WV_THREADS / 32 * CPW], s_cu[WV_THREADS / 32 * CPW];
    __shared__ int s_pair[WV_THREADS / 32 * CPW * 32];
    __shared__ double s_tab[3][32];  // cap, disc, sig_row per period (cp.async at entry)
    __shared__ unsigned s_okm[WV_THREADS / 32 * CPW];  // feasible-period masks (sparse pairs)
    constexpr int NW = WV_THREADS / 32;
    constexpr unsigned FULL = 0xffffffffu;
    const int T = p.T, S = p.S, Sp = p.Sp;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool net = p.flags & PP_NET_MINING_COST;
    const bool literal = p.flags & PP_LITERAL_VALUE;
    constexpr bool STATS_T = KC != 0;  // KC > 0: pooled thread per move, top-KC in registers;
                                       // KC < 0: warp per move, bitonic sort (k > 8 or S > 128)
    const bool stats = STATS_T && (SCEN || p.exp_delta || p.cvar || p.n_pairs);
    // vmax rows staged per warp: the pooled statistics read every precedence-feasible move's row;
    // the big-S statistics read only capacity-feasible moves' rows, straight from L2
    const bool need_vrow = (stats && KC > 0) || (!literal && p.scen >= 0);
    const bool want_unit = !literal && p.scen < 0;
    const bool want_trace = p.trace_val || p.trace_feas;
    // the layout the host sized the launch with (warp_layout, passed in: not recomputed per thread)
    const WarpLayout L{p.wl[0], p.wl[1], p.wl[2], p.wl[3], p.wl[4], p.wl[5], p.wl[6]};
    const int sigb = sig_bytes(S, T, stats && KC > 0);  // big-S statistics read sigma through L1
    double *s_sig = reinterpret_cast<double *>(wv_dyn);
    unsigned char *wslices = wv_dyn + sigb;
    unsigned char *wbase = wslices + (size_t)warp * L.total;
    double *w_vrow = reinterpret_cast<double *>(wbase + L.vrow);
    double *w_cost = reinterpret_cast<double *>(wbase + L.cost);
    double *w_ex = reinterpret_cast<double *>(wbase + L.ex);
    double *w_cv = reinterpret_cast<double *>(wbase + L.cv);
    const int cw = (blockIdx.x * NW + warp) * CPW;
    EV_PROBE(0);
    WP_PROBE(0);

    // ---- loads: ids, then every row of the warp's candidates in one round trip ----
    int bl = -1;
    if (p.cand_host) {  // ids in page-locked host memory (no copy-in): one 128-byte PCIe read per CTA
        __shared__ int s_cid[NW * CPW];
        static_assert(NW * CPW == 32, "one lane per candidate of the CTA");
        if (warp == 0) {
            const int g = blockIdx.x * NW * CPW + lane;
            s_cid[lane] = g < p.C ? p.cand[g] : -1;
        }
        __syncthreads();
        if (lane < CPW && cw + lane < p.C) bl = s_cid[warp * CPW + lane];
    } else if (lane < CPW && cw + lane < p.C) {
        bl = __ldg(p.cand + cw + lane);
    }
    if (lane < CPW && cw + lane < p.C) {
        if (bl < 0 || bl >= p.B) {
            if (p.bad_cand) *p.bad_cand = 1;  // reported by the host-mode call
            bl = -1;
        }
    }
    int b[CPW];
#pragma unroll
    for (int j = 0; j < CPW; j++) b[j] = __shfl_sync(FULL, bl, j);
    if (stats && KC > 0) {  // sigma [S][T] for the pooled pair statistics, staged once per CTA
        const int n = S * T;    // 16-byte copies (the table and the slot are 16-byte aligned)
        for (int e = threadIdx.x; e < (n >> 1); e += WV_THREADS) cp_async16(s_sig + 2 * e, p.sigma + 2 * e);
        if ((n & 1) && threadIdx.x == 0) cp_async8(s_sig + n - 1, p.sigma + n - 1);
    }
    if (threadIdx.x < T) {
        cp_async8(&s_tab[0][threadIdx.x], p.cap + threadIdx.x);
        cp_async8(&s_tab[1][threadIdx.x], p.disc + threadIdx.x);
        cp_async8(&s_tab[2][threadIdx.x], p.sig_row + threadIdx.x);
    }
    // every independent load of the warp's candidates is issued before any result is used (a
    // store of a loaded value would hold the warp until that load returns): neighbour ids, mining
    // costs, vmax rows, the per-candidate scalars; then the neighbours' periods
    int nb[CPW];
    // the rows per candidate (one round each) or as one flat list over the lanes (two rounds at C2
    // instead of four); measured per instantiation: flat is faster at C2 (KC 2: step 19.45 ->
    // 19.2 us) and C3 (KC < 0), slower at C4 (KC 8 then, S = 50: kernel 59.4 -> 63.5 us, more spills)
    constexpr bool FLAT_ROWS = KC == 2 || KC < 0;
#pragma unroll
    for (int j = 0; j < CPW; j++) nb[j] = b[j] >= 0 ? __ldg(p.nbr + (size_t)b[j] * NBR_W + lane) : -1;
    if constexpr (!FLAT_ROWS) {
#pragma unroll
        for (int j = 0; j < CPW; j++)
            if (net && lane < T && b[j] >= 0) cp_async8(w_cost + j * T + lane, p.cost + (size_t)b[j] * T + lane);
        if (need_vrow) {
#pragma unroll
            for (int j = 0; j < CPW; j++)
                if (b[j] >= 0)
                    for (int q = lane; q < (Sp >> 1); q += 32)
                        cp_async16(w_vrow + (size_t)j * Sp + 2 * q, p.vmax + (size_t)b[j] * Sp + 2 * q);
        }
    } else {
        static_assert(CPW == 4, "three thresholds below");
        if (net) {  // element e of the flat list: candidate j = e / T, period e - j T
            const int n = CPW * T;
            for (int e0 = 0; e0 < n; e0 += 32) {
                const int e = e0 + lane;
                const int j = (e >= T) + (e >= 2 * T) + (e >= 3 * T);
                const int bj = __shfl_sync(FULL, bl, j);
                if (e < n && bj >= 0) cp_async8(w_cost + e, p.cost + (size_t)bj * T + (e - j * T));
            }
        }
        if (need_vrow) {  // 16-byte chunk e: candidate j = e / h, chunk e - j h
            const int h = Sp >> 1, n = CPW * h;
            for (int e0 = 0; e0 < n; e0 += 32) {
                const int e = e0 + lane;
                const int j = (e >= h) + (e >= 2 * h) + (e >= 3 * h);
                const int bj = __shfl_sync(FULL, bl, j);
                if (e < n && bj >= 0) cp_async16(w_vrow + 2 * e, p.vmax + (size_t)bj * Sp + 2 * (e - j * h));
            }
        }
    }
    double mass_l = 0.0, spat_l = 0.0, unit_l = 0.0;
    int ab_l = -1;
    if (lane < CPW && bl >= 0) {
        mass_l = __ldg(&p.rows[bl].mass);
        spat_l = __ldg(&p.rows[bl].spatial);
        ab_l = __ldg(p.assign + bl);
        if (want_unit) unit_l = __ldg(p.unit_mean + bl);
    }
    // neighbour periods -> precedence window (evaluate.py:361-372): lo = latest predecessor
    // period (an unmined predecessor forbids every period), hi = earliest mined successor
    int tn[CPW];
#pragma unroll
    for (int j = 0; j < CPW; j++) tn[j] = nb[j] >= 0 ? p.assign[nb[j] & (NBR_SUCC - 1)] : 0;
    if (lane < CPW) {  // per-candidate scalars to shared memory (the pair pool and the moves)
        const int i = warp * CPW + lane;
        s_cm[i] = mass_l;
        s_csp[i] = spat_l;
        s_cu[i] = unit_l;
        s_cab[i] = ab_l;
        s_cb[i] = bl;
    }
    unsigned win[CPW];  // precedence window of candidate j as a period mask (lane t = period t)
#pragma unroll
    for (int j = 0; j < CPW; j++) {
        const bool pred = nb[j] >= 0 && !(nb[j] & NBR_SUCC), succ = nb[j] >= 0 && (nb[j] & NBR_SUCC);
        const int lc = pred ? (tn[j] < 0 ? INT_MAX : tn[j]) : 0;
        const int hc = (succ && tn[j] >= 0) ? tn[j] : INT_MAX;
        const int lo = (int)__reduce_max_sync(FULL, (unsigned)lc);
        const int hi = (int)__reduce_min_sync(FULL, (unsigned)hc);
        win[j] = __ballot_sync(FULL, b[j] >= 0 && lane < T && lane >= lo && lane <= hi);
    }
    if constexpr (KC < 0) {
        if (stats) {  // warm L2 (rows of windowed candidates) and L1 (sigma) for the statistics,
                      // which run after the period masses; this overlaps the period-mass kernel
#pragma unroll
            for (int j = 0; j < CPW; j++)
                if (win[j] && lane * 16 < Sp)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(p.vmax + (size_t)b[j] * Sp + lane * 16));
            for (int e = threadIdx.x * 16; e < S * T; e += WV_THREADS * 16)
                asm volatile("prefetch.global.L1 [%0];" ::"l"(p.sigma_ts + e));
        }
    }
    cp_async_wait_all();
    __syncwarp();
    EV_PROBE(1);
    WP_PROBE(1);

    // ---- statistics of the precedence-feasible (candidate, period) pairs, before the
    //      period masses are known (overlaps the period-mass kernel); capacity only
    //      removes pairs, so the outputs below select from these ----
    if constexpr (KC > 0) {
        if (stats) {
            // CTA-wide pool of the pairs, one thread per pair: a warp holds ~9 pairs at C2, a CTA
            // ~70, so pooling keeps ~3x more of each warp's lanes busy than per-warp lists
            int cum[CPW + 1];
            cum[0] = 0;
#pragma unroll
            for (int j = 0; j < CPW; j++) cum[j + 1] = cum[j] + __popc(win[j]);
            const int np = cum[CPW];
            if (lane == 0) s_wcnt[warp] = np;
            __syncthreads();
            int base = 0, total = 0;
#pragma unroll
            for (int w = 0; w < NW; w++) {
                const int x = s_wcnt[w];
                base += w < warp ? x : 0;
                total += x;
            }
            {
                const unsigned lt = (1u << lane) - 1u;
#pragma unroll
                for (int j = 0; j < CPW; j++)
                    if ((win[j] >> lane) & 1u) {
                        PP_DCHECK(base + cum[j] + __popc(win[j] & lt) < NW * CPW * 32);
                        s_pair[base + cum[j] + __popc(win[j] & lt)] = ((warp * CPW + j) << 8) | lane;
                    }
            }
            __syncthreads();
            EV_PROBE(8);
            WP_PROBE(2);
#ifdef PP_EVAL_PROBE
            const long long c_st0 = clock64();
#endif
            for (int k = threadIdx.x; k < total; k += WV_THREADS) {
                const int e = s_pair[k], i = e >> 8, t = e & 0xff;
                const int wq = i / CPW, jq = i - wq * CPW;
                unsigned char *wb = wslices + (size_t)wq * L.total;
                const int ab = s_cab[i];
                const double sp = s_csp[i];
                const int abc = ab >= 0 ? ab : 0;
                const double d_t = s_tab[1][t], d_ab = s_tab[1][abc];
                const double *wc = reinterpret_cast<const double *>(wb + L.cost) + jq * T;
                const double dc_t = net ? f64_mul(d_t, wc[t]) : 0.0;
                const double dc_ab = net ? f64_mul(d_ab, wc[abc]) : 0.0;
                {  // the move's kernel value (evaluate.py:379-384), used by the selection below
                    double unit;
                    if (literal) unit = f64_mul(s_cm[i], 100.0);
                    else if (p.scen >= 0) unit = reinterpret_cast<const double *>(wb + L.vrow)[(size_t)jq * Sp + p.scen];
                    else unit = s_cu[i];
                    double v = f64_mul(f64_mul(f64_mul(unit, d_t), s_tab[2][t]), sp);
                    if (net) v = f64_sub(v, dc_t);
                    reinterpret_cast<double *>(wb + L.val)[jq * 32 + t] = v;
                }
                float *sd = SCEN ? p.scen_delta + (size_t)(blockIdx.x * NW * CPW + i) * S * T + t : nullptr;
                pair_stats<KC, SCEN>(p, S, T, s_sig, reinterpret_cast<double *>(wb + L.vrow) + (size_t)jq * Sp, t, abc,
                                     d_t, dc_t, d_ab, dc_ab, sp, ab >= 0,
                                     reinterpret_cast<double *>(wb + L.ex) + jq * T + t,
                                     reinterpret_cast<double *>(wb + L.cv) + jq * T + t, sd);
            }
            WP_PROBE(3);
#ifdef PP_EVAL_PROBE
            if ((threadIdx.x & 31) == 0 && blockIdx.x < 1024) g_wp_probe[blockIdx.x][threadIdx.x >> 5][10] = clock64() - c_st0;
#endif
            __syncthreads();
        }
    }
    EV_PROBE(7);
    WP_PROBE(4);


    // ---- moves, pm-independent half: the value of every window period (evaluate.py:379-384),
    //      kept in the lane's registers for the selection after the wait ----
    if (!(KC > 0 && stats)) __syncthreads();  // s_tab (the pooled path passed a CTA barrier already)
    double *w_val = reinterpret_cast<double *>(wbase + L.val);
    double vj[CPW];
#pragma unroll
    for (int j = 0; j < CPW; j++) {
        const int ci = warp * CPW + j;
        const bool in = (win[j] >> lane) & 1u;
        double v = -kInf;
        if (KC > 0 && stats) {
            if (in) v = w_val[j * 32 + lane];  // computed with the statistics of the move
        } else if (in) {
            const double disc_t = s_tab[1][lane];
            double unit;
            if (literal) unit = f64_mul(s_cm[ci], 100.0);
            else if (p.scen >= 0) unit = w_vrow[(size_t)j * Sp + p.scen];
            else unit = s_cu[ci];
            v = f64_mul(f64_mul(f64_mul(unit, disc_t), s_tab[2][lane]), s_csp[ci]);
            if (net) v = f64_sub(v, f64_mul(disc_t, w_cost[j * T + lane]));
        }
        vj[j] = v;
    }
    EV_PROBE(2);
    WP_PROBE(5);

    // ---- moves, pm half: capacity (evaluate.py:373-378) and the selection: the reference's strict
    //      '>' scan over t (387-388) keeps the first maximum, i.e. the maximum of (value, -t); as an
    //      order-preserving 64-bit key (-0.0 folded onto +0.0, which compare equal) that is two
    //      warp maxima (high then low word) and the lowest lane holding it.  -inf / NaN never
    //      selected ----
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // a plain (L1-cached) load: one L2 request per SM instead of one per warp on the same line --
    // all ~4,000 warps pass the wait together (griddepcontrol.wait makes the writes visible; no
    // load of pm precedes it)
    const double pm_t = lane < T ? p.pm[lane] : 0.0;
    EV_PROBE(3);
    WP_PROBE(6);
    Best wbest{-kInf, INT_MAX, INT_MAX};
    unsigned okm[CPW];
    bool okl[CPW];
    unsigned hi[CPW], lo[CPW], mhi[CPW], mlo[CPW];
    // the four candidates' steps interleaved: capacity and keys, then each warp reduction for all four
#pragma unroll
    for (int j = 0; j < CPW; j++) {
        const int ci = warp * CPW + j;
        const double mass = s_cm[ci];
        const int ab = s_cab[ci];
        b[j] = s_cb[ci];
        bool ok = false;
        if ((win[j] >> lane) & 1u) {
            double load = f64_add(pm_t, mass);
            if (ab == lane) load = f64_sub(load, mass);
            ok = !(load > s_tab[0][lane]);
        }
        okl[j] = ok;
        const bool sel = ok && vj[j] > -kInf;
        const unsigned long long kk = sel ? f64_key(vj[j] == 0.0 ? 0.0 : vj[j]) : 0ull;
        hi[j] = (unsigned)(kk >> 32);
        lo[j] = (unsigned)kk;
    }
#pragma unroll
    for (int j = 0; j < CPW; j++) {
        okm[j] = __ballot_sync(FULL, okl[j]);
        mhi[j] = __reduce_max_sync(FULL, hi[j]);
    }
#pragma unroll
    for (int j = 0; j < CPW; j++) mlo[j] = __reduce_max_sync(FULL, (hi[j] == mhi[j] && hi[j]) ? lo[j] : 0u);
    int my_bt = INT_MAX;  // lane j < CPW: candidate j's selected period and value
    double my_bv = -kInf;
#pragma unroll
    for (int j = 0; j < CPW; j++) {
        const unsigned win_t = __ballot_sync(FULL, hi[j] && hi[j] == mhi[j] && lo[j] == mlo[j]);
        const int bt = win_t ? __ffs(win_t) - 1 : INT_MAX;
        const double bv = __shfl_sync(FULL, vj[j], win_t ? bt : 0);
        if (lane == j) {
            my_bt = bt;
            my_bv = bv;
        }
        const int g = cw + j;
        if (want_trace && g < p.C && lane < T) {
            if (p.trace_val) p.trace_val[(size_t)g * T + lane] = okl[j] ? vj[j] : -kInf;
            if (p.trace_feas) p.trace_feas[(size_t)g * T + lane] = okl[j] ? 1 : 0;
        }
    }
    // per-candidate outputs by lane j (one store each, not four rounds of lane 0), and the
    // warp's best move over lanes 0..CPW-1 (bl = lane j's candidate id, -1 past the end)
    if (lane < CPW && bl >= 0) {
        const int g = cw + lane;
        const bool f = my_bt != INT_MAX;
        p.best_t[g] = f ? my_bt : -1;
        p.best_val[g] = f ? my_bv : -kInf;
        p.feas[g] = f ? 1 : 0;
        if (f) wbest = Best{my_bv, bl, my_bt};
    }
#pragma unroll
    for (int off = 1; off < CPW; off <<= 1) {
        const Best o = shfl_best(wbest, off);
        if (better(o, wbest)) wbest = o;
    }
    // ---- KC < 0: statistics of the feasible moves, one warp per move (after the capacity
    //      test: with many scenarios the statistics dominate, so only feasible moves pay).  The
    //      CTA's feasible moves are dealt round-robin to its warps (a warp's own four candidates
    //      hold anywhere from 0 to 60 of them) ----
    if constexpr (KC < 0) {
        if (stats) {
            static_assert(NW * CPW == 32, "one lane per candidate of the CTA");
            {
                unsigned mine = 0u;
#pragma unroll
                for (int j = 0; j < CPW; j++)
                    if (lane == j) mine = okm[j];
                if (lane < CPW) s_okm[warp * CPW + lane] = mine;
            }
            __syncthreads();
            EV_PROBE(8);
            const unsigned om = s_okm[lane];  // lane i: candidate i of the CTA
            int incl = __popc(om);
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += y;
            }
            const int excl = incl - __popc(om);
            const int nmoves = __shfl_sync(FULL, incl, 31);
            const int P2 = big_pow2(S);
            double *vb = reinterpret_cast<double *>(wbase + L.big);
            double *lv = vb + P2;
            const int *P = p.plan;
            const int nleaf = __ldg(P + 1);
            const int kq = p.cvar_k;
            for (int mv = warp; mv < nmoves; mv += NW) {
                const int ci = __ffs(__ballot_sync(FULL, excl <= mv && mv < incl)) - 1;
                const int t = nth_bit(__shfl_sync(FULL, om, ci), mv - __shfl_sync(FULL, excl, ci));
                const int wq = ci / CPW, jq = ci - wq * CPW;
                unsigned char *wb = wslices + (size_t)wq * L.total;
                const double *crow = reinterpret_cast<const double *>(wb + L.cost) + jq * T;
                const double *rowb = p.vmax + (size_t)s_cb[ci] * Sp;
                const int ab = s_cab[ci];
                const double sp = s_csp[ci];
                const bool mined = ab >= 0;
                const int abc = mined ? ab : 0;
                const double d_ab = s_tab[1][abc];
                const double dc_ab = net ? f64_mul(d_ab, crow[abc]) : 0.0;
                const double d_t = s_tab[1][t];
                const double dc_t = net ? f64_mul(d_t, crow[t]) : 0.0;
                const size_t g = (size_t)blockIdx.x * NW * CPW + ci;
                unsigned long long k8[8];  // element lane + 32 r as a sort key; padding last
                // every load of the move's scenario rows first (one round trip, not eight), then the values
                double xr[8], gt[8], ga[8];
#pragma unroll
                for (int r = 0; r < 8; r++) {
                    const int s_ = lane + 32 * r;
                    const bool in = s_ < S;
                    xr[r] = in ? __ldg(rowb + s_) : 0.0;
                    gt[r] = in ? __ldg(p.sigma_ts + t * S + s_) : 0.0;
                    ga[r] = (in && mined) ? __ldg(p.sigma_ts + abc * S + s_) : 0.0;
                }
#pragma unroll
                for (int r = 0; r < 8; r++) {
                    const int s_ = lane + 32 * r;
                    k8[r] = ~0ull;
                    if (s_ < S) {
                        const double x = xr[r];
                        const double vn = f64_sub(f64_mul(f64_mul(f64_mul(x, d_t), gt[r]), sp), dc_t);
                        const double vo = mined ? f64_sub(f64_mul(f64_mul(f64_mul(x, d_ab), ga[r]), sp), dc_ab) : 0.0;
                        const double v = f64_sub(vn, vo);
                        if constexpr (SCEN) p.scen_delta[(g * S + s_) * T + t] = (float)v;
                        vb[s_] = v;
                        k8[r] = f64_key(v);
                    }
                }
                __syncwarp();
                if (mv == 0) EV_PROBE(9);
                // expected delta: numpy pairwise over d[0..S) (the plan's leaves, 8 lanes each)
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
                // CVaR10: the k smallest in ascending order (np.sort, saa.py:157-164) over the
                // deltas just consumed by the mean, then their pairwise mean
                if (mv == 0) EV_PROBE(10);
                const double kv = warp_k_smallest(k8, kq, reinterpret_cast<unsigned long long *>(vb), P2 >> 5);
                if (mv == 0) EV_PROBE(11);
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
                if (lane == 0) {
                    reinterpret_cast<double *>(wb + L.cv)[jq * T + t] = f64_div(f64_add(0.0, rc), (double)kq);
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
                    reinterpret_cast<double *>(wb + L.ex)[jq * T + t] = f64_div(f64_add(0.0, stk[0]), (double)S);
                }
                __syncwarp();
            }
            __syncthreads();  // the owners' dense outputs read these statistics
        }
    }
    EV_PROBE(4);
    WP_PROBE(7);

    // ---- per-(candidate, period) statistics outputs (capacity-feasible pairs only) ----
    if constexpr (STATS_T) {
        if (stats && (SCEN || p.exp_delta || p.cvar)) {  // (sparse pairs only: nothing dense to write)
#pragma unroll
            for (int j = 0; j < CPW; j++) {
                const int g = cw + j;
                if (g >= p.C || lane >= T) continue;
                const bool ok = (okm[j] >> lane) & 1u;
                if (p.exp_delta) p.exp_delta[(size_t)g * T + lane] = ok ? w_ex[j * T + lane] : -kInf;
                if (p.cvar) p.cvar[(size_t)g * T + lane] = ok ? w_cv[j * T + lane] : -kInf;
                if constexpr (SCEN) {
                    if (!ok)  // infeasible: raw deltas are -inf
                        for (int s = 0; s < S; s++)
                            p.scen_delta[((size_t)g * S + s) * T + lane] = -__int_as_float(0x7f800000);
                }
            }
        }
    }
    EV_PROBE(5);
    WP_PROBE(8);

    // ---- CTA epilogue after one barrier: warp 0 merges the warps' best moves into the global
    //      record (one 128-bit compare-and-swap per CTA, the record initialised ahead of the
    //      launch); warp 1 reserves the CTA's sparse pairs with one atomic (not one per warp: the
    //      counter is a single contended address) and lane t writes candidate i's period-t entry ----
    // the copy-out launch (PDL) may be staged once every CTA of the grid has reached this point, so
    // its CTAs never take a slot an evaluation CTA still needs
    asm volatile("griddepcontrol.launch_dependents;");
    if (lane == 0) s_red[warp] = wbest;
    const bool want_pairs = STATS_T && stats && p.n_pairs;
    if (want_pairs) {
        unsigned mine = 0u;  // lane j publishes candidate j's mask (okm is warp-uniform)
#pragma unroll
        for (int j = 0; j < CPW; j++)
            if (lane == j) mine = okm[j];
        if (lane < CPW) s_okm[warp * CPW + lane] = (cw + lane < p.C) ? mine : 0u;
    }
    __syncthreads();
    if (warp == 0) {
        Best x = lane < NW ? s_red[lane] : Best{-kInf, INT_MAX, INT_MAX};
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const Best o = shfl_best(x, off);
            if (better(o, x)) x = o;
        }
        if (lane == 0 && x.b != INT_MAX) best_cas(p.global, x);
    }
    if (want_pairs && warp == (NW > 1 ? 1 : 0)) {
        // lane i: candidate i of the CTA (NW * CPW == 32): its pairs go to a contiguous range after
        // the exclusive scan of the counts; one atomic reserves the CTA's range
        static_assert(NW * CPW == 32, "one lane per candidate of the CTA");
        const unsigned m = s_okm[lane];
        const int cnt = __popc(m);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(FULL, incl, 31);
        int pbase = 0;
        if (lane == 0 && total) pbase = atomicAdd(p.n_pairs, total);
        pbase = __shfl_sync(FULL, pbase, 0);
        const int wq = lane / CPW, jq = lane - wq * CPW;
        const double *wex = reinterpret_cast<const double *>(wslices + (size_t)wq * L.total + L.ex) + jq * T;
        const double *wcv = reinterpret_cast<const double *>(wslices + (size_t)wq * L.total + L.cv) + jq * T;
        int q = pbase + incl - cnt;
        for (unsigned mm = m; mm; mm &= mm - 1, q++) {
            const int t = __ffs(mm) - 1;
            PP_DCHECK(q < p.C * p.T && t < p.T);
            p.pair_cand[q] = blockIdx.x * NW * CPW + lane;
            p.pair_period[q] = t;
            p.pair_exp[q] = wex[t];
            p.pair_cvar[q] = wcv[t];
        }
    }
    EV_PROBE(6);
    WP_PROBE(9);
}

#ifdef PP_EVAL_PROBE
__device__ unsigned long long g_stamp[8];
__global__ void k_stamp(int slot) { g_stamp[slot] = gtimer(); }
extern "C" PP_API int pp_debug_stamp(void *stream, int slot) {
    k_stamp<<<1, 1, 0, (cudaStream_t)stream>>>(slot);
    return cudaGetLastError() == cudaSuccess ? 0 : 3;
}
extern "C" PP_API int pp_debug_stamps(unsigned long long *out) {
    return cudaMemcpyFromSymbol(out, g_stamp, sizeof(g_stamp)) == cudaSuccess ? 0 : 3;
}
extern "C" PP_API int pp_debug_eval_probe(unsigned long long *out) {
    return cudaMemcpyFromSymbol(out, g_ev_probe, sizeof(unsigned long long) * 4096 * 12) == cudaSuccess ? 0 : 3;
}
#endif


// ------------------------------------------------------------------------------------
// k_realism: lns_repair's realism-fallback choice (hybrid.py:256-263) on the device -- among
// the feasible candidates (best period >= 0), the first by geological consistency descending,
// then block ascending: the evaluate.py:404-409 total order with value = spatial[b], so the same
// deterministic grid argmax (per-CTA partials, last CTA reduces) gives it.
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_realism(const int32_t *__restrict__ cand, int C, int B,
                                                 const int32_t *__restrict__ best_t, const BlockRow *__restrict__ rows,
                                                 pp_best *partial, unsigned int *counter, pp_best *out) {
    __shared__ Best s_red[8];
    Best mine{-kInf, INT_MAX, INT_MAX};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < C; i += gridDim.x * blockDim.x) {
        const int b = __ldg(cand + i), t = best_t[i];
        if (b < 0 || b >= B || t < 0) continue;
        const Best o{__ldg(&rows[b].spatial), b, t};
        if (better(o, mine)) mine = o;
    }
    grid_argmax(mine, s_red, partial, counter, out);
}

// ------------------------------------------------------------------------------------
// Host-mode copy-out: when every output array is page-locked (device-mapped under UVA), one
// launch writes all of them straight into host memory with 16-byte stores, reading the sparse
// pair count on the device -- instead of one cudaMemcpyAsync per array (each ~4 us of CPU) and
// a speculative pair copy.
// ------------------------------------------------------------------------------------
struct CopySeg {
    const unsigned char *src;
    unsigned char *dst;
    unsigned long long bytes;  // fixed size, or
    int per_pair;              // > 0: bytes = n_pairs * per_pair
};
constexpr int PP_MAX_SEGS = 16;
struct CopyOut {
    CopySeg seg[PP_MAX_SEGS];
    int nseg;
    const int32_t *n_pairs;
};

__global__ void __launch_bounds__(256) k_copy_out(const CopyOut co) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // launched under PDL behind the evaluation
    const CopySeg &sg = co.seg[blockIdx.y];
    const unsigned long long bytes =
        sg.per_pair > 0 ? (unsigned long long)max(0, __ldcg(co.n_pairs)) * sg.per_pair : sg.bytes;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    const unsigned long long tid = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(sg.src) | reinterpret_cast<uintptr_t>(sg.dst)) & 15u) == 0;
    unsigned long long body = 0;
    if (vec) {
        body = bytes & ~15ull;
        const uint4 *s4 = reinterpret_cast<const uint4 *>(sg.src);
        uint4 *d4 = reinterpret_cast<uint4 *>(sg.dst);
        for (unsigned long long i = tid; i < body / 16; i += stride) d4[i] = __ldcg(s4 + i);
    }
    for (unsigned long long i = body + tid; i < bytes; i += stride) sg.dst[i] = sg.src[i];
}

// device pointer of a page-locked host buffer, or nullptr (pageable / unknown)
extern "C" {

int pp_eval_candidates(pp_ctx *c, const int32_t *cand, int32_t C, int32_t scenario, uint32_t flags,
                       const pp_cand_out *out, int32_t mem, void *stream) {
    HostTrace ht("pp_eval_candidates");
    TRY(check_ready(c, flags, scenario));
    if (C < 0 || (C > 0 && !cand)) return fail(PP_ERR_INVALID_ARGS, "bad candidate array");
    if (!out || !out->best_t || !out->best_val || !out->feasible || !out->global)
        return fail(PP_ERR_INVALID_ARGS, "best_t, best_val, feasible and global outputs are required");
    const bool pairs = out->n_pairs != nullptr;
    if (pairs && (!out->pair_cand || !out->pair_period || !out->pair_exp || !out->pair_cvar))
        return fail(PP_ERR_INVALID_ARGS, "n_pairs needs pair_cand, pair_period, pair_exp and pair_cvar");
    const bool stats = out->exp_delta || out->cvar || out->scen_delta || pairs;
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

    // ---- a repeat of the previous host-mode call (same ids, outputs, state, buffers): replay ----
    const bool warp_path_ = T <= 32 && (!stats || S <= 256) && c->nbr.ptr;
    static const bool no_graph = std::getenv("PP_NO_EVAL_GRAPH") != nullptr;  // diagnostics
    const bool graph_shape = mem == PP_MEM_HOST && warp_path_ && C > 0 && !out->realism && !out->scen_delta && !no_graph;
    pp_ctx::EvalGraphKey gkey;
    auto make_key = [&](pp_ctx::EvalGraphKey &k) {
        memset(&k, 0, sizeof(k));  // (padding bytes compare too)
        k.cand = cand;
        k.C = C;
        k.scenario = scenario;
        k.flags = flags;
        k.pm_dirty = c->pm_dirty;
        k.bad_pending = c->bad_pending;
        k.cvar_k = c->cvar_k;
        k.S = S;
        k.T = T;
        k.B = c->B;
        k.Sp = c->Sp;
        k.out = *out;
        k.assign_ptr = c->assign_ptr;
        for (DevBuf *d : c->all()) k.gensum += d->gen;
        k.pinned_gen = pinned_generation();  // (the page-locked buffers' device mappings are baked in)
    };
    if (graph_shape) make_key(gkey);
    const bool replay = graph_shape && c->ev_exec && memcmp(&gkey, &c->ev_key, sizeof(gkey)) == 0;
    const bool graph_ok = graph_shape && !replay &&
                    mapped_host(cand) && mapped_host(out->best_t) && mapped_host(out->best_val) &&
                    mapped_host(out->feasible) && (!out->trace_val || mapped_host(out->trace_val)) &&
                    (!out->trace_feas || mapped_host(out->trace_feas)) && (!out->exp_delta || mapped_host(out->exp_delta)) &&
                    (!out->cvar || mapped_host(out->cvar)) &&
                    (!pairs || (mapped_host(out->pair_cand) && mapped_host(out->pair_period) &&
                                mapped_host(out->pair_exp) && mapped_host(out->pair_cvar)));
    if (replay) {
        if (cudaGraphLaunch(c->ev_exec, st) != cudaSuccess)
            return fail(PP_ERR_CUDA, "graph launch: %s", cudaGetErrorString(cudaGetLastError()));
        c->pm_dirty = false;  // (the graph holds the period-mass launch when they were stale)
        ht.mark("graph launch");
        CUDA_TRY(stream_wait(st));
        ht.mark("sync");
        int32_t bad_c = 0;
        for (int i = 0; i < c->ev_nb; i++) {
            const pp_ctx::EvalBounce &e = c->ev_bounce[i];
            memcpy(e.user ? e.user : &bad_c, c->h_bounce + e.off, e.bytes);
        }
        TRY(check_schedule_range(c, c->ev_bad_copy));
        if (bad_c) return fail(PP_ERR_INVALID_ARGS, "candidate block out of range [0, %d)", c->B);
        if (pairs) c->last_pairs = (size_t)std::max(0, *out->n_pairs);
        return PP_OK;
    }
    // the second identical call in a row is captured (the first one allocated every buffer)
    const bool capture = graph_ok && c->ev_have_seen && memcmp(&gkey, &c->ev_seen, sizeof(gkey)) == 0;
    if (graph_ok) {
        c->ev_seen = gkey;
        c->ev_have_seen = true;
    }
    if (capture) {
        if (c->ev_exec) cudaGraphExecDestroy(c->ev_exec);
        if (c->ev_graph) cudaGraphDestroy(c->ev_graph);
        c->ev_exec = nullptr;
        c->ev_graph = nullptr;
        memset(&c->ev_key, 0, sizeof(c->ev_key));
        CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
    }
    struct CaptureGuard {  // an error return inside the capture must not leave the stream capturing
        cudaStream_t st;
        bool on;
        ~CaptureGuard() {
            if (!on) return;
            cudaGraph_t g = nullptr;
            cudaStreamEndCapture(st, &g);
            if (g) cudaGraphDestroy(g);
            cudaGetLastError();
        }
    } cguard{st, capture};
    pp_cand_out o = *out;
    const int32_t *dcand = cand;
    bool cand_host = false;  // dcand: the device mapping of page-locked host ids (k_eval_warp only)
    const bool warp_path = T <= 32 && (!stats || S <= 256) && c->nbr.ptr;
    if (mem == PP_MEM_HOST) {
        if (!warp_path) {  // the warp kernel range-checks the ids itself (reported after the sync)
            int32_t lo = 0, hi = 0;  // branch-free min/max (vectorises)
            for (int i = 0; i < C; i++) {
                lo = std::min(lo, cand[i]);
                hi = std::max(hi, cand[i]);
            }
            if (lo < 0 || hi >= c->B) return fail(PP_ERR_INVALID_ARGS, "candidate block out of range [0, %d)", c->B);
            ht.mark("validate");
        } else if (!c->bad_cand.ptr) {
            TRY(c->bad_cand.ensure(sizeof(int32_t)));
        }
        const size_t Cs = (size_t)std::max(C, 1), CT = Cs * T;
        TRY(c->h_cand.ensure(sizeof(int32_t) * Cs));
        TRY(c->h_o1.ensure(sizeof(int32_t) * Cs));
        TRY(c->h_o2.ensure(sizeof(double) * Cs));
        TRY(c->h_o3.ensure(Cs));
        TRY(c->h_glob.ensure(2 * sizeof(pp_best)));
        o.best_t = c->h_o1.as<int32_t>();
        o.best_val = c->h_o2.as<double>();
        o.feasible = c->h_o3.as<uint8_t>();
        o.global = c->h_glob.as<pp_best>();
        if (out->realism) o.realism = c->h_glob.as<pp_best>() + 1;
        if (out->trace_val) { TRY(c->h_o4.ensure(sizeof(double) * CT)); o.trace_val = c->h_o4.as<double>(); }
        if (out->trace_feas) { TRY(c->h_o5.ensure(CT)); o.trace_feas = c->h_o5.as<uint8_t>(); }
        if (out->exp_delta) { TRY(c->h_o6.ensure(sizeof(double) * CT)); o.exp_delta = c->h_o6.as<double>(); }
        if (out->cvar) { TRY(c->h_o7.ensure(sizeof(double) * CT)); o.cvar = c->h_o7.as<double>(); }
        if (out->scen_delta) { TRY(c->h_o8.ensure(sizeof(float) * CT * std::max(S, 1))); o.scen_delta = c->h_o8.as<float>(); }
        if (pairs) {
            TRY(c->h_p.ensure((2 * sizeof(int32_t) + 2 * sizeof(double)) * CT + 16));
            char *q = static_cast<char *>(c->h_p.ptr);
            o.pair_exp = reinterpret_cast<double *>(q);
            o.pair_cvar = reinterpret_cast<double *>(q + sizeof(double) * CT);
            o.pair_cand = reinterpret_cast<int32_t *>(q + 2 * sizeof(double) * CT);
            o.pair_period = reinterpret_cast<int32_t *>(q + 2 * sizeof(double) * CT + sizeof(int32_t) * CT);
            o.n_pairs = reinterpret_cast<int32_t *>(q + (2 * sizeof(double) + 2 * sizeof(int32_t)) * CT);
        }
        // page-locked ids on the warp path: read in place by k_eval_warp (one PCIe read per CTA)
        // instead of a DMA copy-in ahead of the kernels
        static const bool no_zc = std::getenv("PP_NO_ZEROCOPY_CAND") != nullptr;  // diagnostics
        const void *mc = (C > 0 && warp_path && !out->realism && !no_zc) ? mapped_host(cand) : nullptr;
        if (mc) {
            dcand = static_cast<const int32_t *>(mc);
            cand_host = true;
        } else {
            if (C > 0) CUDA_TRY(cudaMemcpyAsync(c->h_cand.ptr, cand, sizeof(int32_t) * C, cudaMemcpyHostToDevice, st));
            dcand = c->h_cand.as<int32_t>();
        }
        ht.mark("h2d");
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
    ep.sigma_ts = (flags & PP_USE_SIGMA) ? c->sigma_ts.as<double>() : c->ones_st.as<double>();
    ep.cand = dcand;
    ep.cand_host = cand_host ? 1 : 0;
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
    ep.pair_cand = o.pair_cand;
    ep.pair_period = o.pair_period;
    ep.pair_exp = o.pair_exp;
    ep.pair_cvar = o.pair_cvar;
    ep.n_pairs = o.n_pairs;
    ep.partial = c->partial.as<pp_best>();
    ep.counter = c->counter.as<unsigned int>();
    ep.global = o.global;

    // fast path: one warp per CPW candidates (k_eval_warp)
    if (warp_path) {
        // the k-smallest list sized to k (each push compares and moves every slot); -1: warp per move
        const int kcw = !stats ? 0 : c->cvar_k <= 2 ? 2 : c->cvar_k <= 8 ? c->cvar_k : -1;
        const bool need_vrow = (stats && kcw > 0) || (!(flags & PP_LITERAL_VALUE) && scenario >= 0);
        const WarpLayout Lw = warp_layout(T, c->Sp, stats, need_vrow, (flags & PP_NET_MINING_COST) != 0,
                                          kcw < 0 ? big_pow2(S) : 0);
        const size_t smem_w = (size_t)Lw.total * (WV_THREADS / 32) + sig_bytes(S, T, stats && kcw > 0);
        const int wl[7] = {Lw.vrow, Lw.cost, Lw.val, Lw.ex, Lw.cv, Lw.big, Lw.total};
        memcpy(ep.wl, wl, sizeof(wl));
        const int per_cta = CPW * (WV_THREADS / 32);
        const int wgrid = std::max(1, (C + per_cta - 1) / per_cta);
        TRY(ensure_grid_scratch(c, wgrid));
        ht.mark("eval setup");
        if (reinterpret_cast<uintptr_t>(o.global) & 15u)
            return fail(PP_ERR_INVALID_ARGS, "global (pp_best) must be 16-byte aligned");
        bool pdl;
        ep.bad_cand = mem == PP_MEM_HOST ? c->bad_cand.as<int32_t>() : nullptr;
        const EvalInit init{o.n_pairs, o.global, ep.bad_cand};
        TRY(refresh_pm(c, st, &pdl, &init));  // initialises n_pairs and the best record ahead of the evaluation
        ht.mark("pm launch");
        const bool scen = o.scen_delta != nullptr;
#define PP_WARP(KC, SC)                                                     \
    {                                                                       \
        TRY(set_smem_attr(k_eval_warp<KC, SC>, smem_w, c->device));         \
        TRY(launch_eval_n(k_eval_warp<KC, SC>, wgrid, WV_THREADS, smem_w, st, pdl, ep));  \
    }
        if (kcw == 0) PP_WARP(0, false)
        else if (kcw == 2) { if (scen) PP_WARP(2, true) else PP_WARP(2, false) }
        else if (kcw == 3) { if (scen) PP_WARP(3, true) else PP_WARP(3, false) }
        else if (kcw == 4) { if (scen) PP_WARP(4, true) else PP_WARP(4, false) }
        else if (kcw == 5) { if (scen) PP_WARP(5, true) else PP_WARP(5, false) }
        else if (kcw == 6) { if (scen) PP_WARP(6, true) else PP_WARP(6, false) }
        else if (kcw == 7) { if (scen) PP_WARP(7, true) else PP_WARP(7, false) }
        else if (kcw == 8) { if (scen) PP_WARP(8, true) else PP_WARP(8, false) }
        else { if (scen) PP_WARP(-1, true) else PP_WARP(-1, false) }
#undef PP_WARP
        goto copy_out;
    }
    {
        bool pdl;
        const EvalInit init{o.n_pairs, nullptr, nullptr};  // the general kernel's last CTA writes the best record
        TRY(refresh_pm(c, st, &pdl, &init));
        TRY(launch_general_candidates(PER, kc, o.scen_delta != nullptr, C, G, S, c->Sp, T, stats, st, pdl, c->device,
                                      ep));
    }
copy_out:
    if (o.realism) {  // second key over the per-candidate results just written (stream-ordered)
        if (reinterpret_cast<uintptr_t>(o.realism) & 15u)
            return fail(PP_ERR_INVALID_ARGS, "realism (pp_best) must be 16-byte aligned");
        const int rgrid = std::max(1, std::min((C + 255) / 256, 148 * 4));
        TRY(ensure_grid_scratch(c, rgrid));
        k_realism<<<rgrid, 256, 0, st>>>(dcand, C, c->B, o.best_t, c->rows.as<BlockRow>(), c->partial.as<pp_best>(),
                                         c->counter.as<unsigned int>() + 1, o.realism);
        CUDA_TRY(cudaGetLastError());
    }
    ht.mark("launch");

    if (mem == PP_MEM_HOST) {
        const size_t Cs = (size_t)C, CT = Cs * T;
        {  // one copy-out launch when every destination is page-locked
            CopyOut co;
            memset(&co, 0, sizeof(co));
            co.n_pairs = o.n_pairs;
            bool ok = true;
            // small fixed-size results in pageable memory (e.g. a ctypes pp_best) go through a
            // page-locked bounce buffer of the context, copied out by the CPU after the sync
            if (!c->h_bounce) {
                CUDA_TRY(cudaHostAlloc(reinterpret_cast<void **>(&c->h_bounce), 256,
                                       cudaHostAllocPortable | cudaHostAllocMapped));
            }
            struct Bounce {
                void *user;
                size_t off, bytes;
            } bounce[4];
            int nb = 0;
            size_t boff = 0;
            auto add = [&](const void *src, void *dst, size_t bytes, int per_pair) {
                if (!dst || !ok) return;
                void *d = mapped_host(dst);
                if (!d && per_pair == 0 && bytes <= 64 && nb < 4) {
                    bounce[nb++] = Bounce{dst, boff, bytes};
                    d = c->h_bounce + boff;
                    boff += 64;
                }
                if (!d || co.nseg == PP_MAX_SEGS) {
                    ok = false;
                    return;
                }
                co.seg[co.nseg++] = CopySeg{static_cast<const unsigned char *>(src), static_cast<unsigned char *>(d),
                                            (unsigned long long)bytes, per_pair};
            };
            add(o.global, out->global, sizeof(pp_best), 0);
            if (o.realism) add(o.realism, out->realism, sizeof(pp_best), 0);
            if (C > 0) {
                add(o.best_t, out->best_t, sizeof(int32_t) * Cs, 0);
                add(o.best_val, out->best_val, sizeof(double) * Cs, 0);
                add(o.feasible, out->feasible, Cs, 0);
                add(o.trace_val, out->trace_val, sizeof(double) * CT, 0);
                add(o.trace_feas, out->trace_feas, CT, 0);
                add(o.exp_delta, out->exp_delta, sizeof(double) * CT, 0);
                add(o.cvar, out->cvar, sizeof(double) * CT, 0);
                add(o.scen_delta, out->scen_delta, sizeof(float) * CT * S, 0);
            }
            int32_t bad_c = 0;
            if (warp_path) add(c->bad_cand.ptr, &bad_c, sizeof(int32_t), 0);
            const bool bad_copy = c->bad_pending && !c->pm_dirty;
            if (bad_copy) add(c->pm_bad.ptr, c->h_bad, sizeof(int32_t) * 16, 0);
            if (pairs) {
                add(o.n_pairs, out->n_pairs, sizeof(int32_t), 0);
                add(o.pair_cand, out->pair_cand, 0, sizeof(int32_t));
                add(o.pair_period, out->pair_period, 0, sizeof(int32_t));
                add(o.pair_exp, out->pair_exp, 0, sizeof(double));
                add(o.pair_cvar, out->pair_cvar, 0, sizeof(double));
            }
            ht.mark("map check");
            if (ok) {
                // PDL: the launch is staged while the evaluation's CTAs finish (they trigger at
                // their epilogue); griddepcontrol.wait above still orders every read after them
                TRY(launch_eval_n(k_copy_out, dim3(64, co.nseg), 256, 0, st, true, co));
                ht.mark("d2h enqueue");
                if (capture) {  // the launches of this call become the cached graph, run now
                    cudaGraph_t g = nullptr;
                    cguard.on = false;
                    CUDA_TRY(cudaStreamEndCapture(st, &g));
                    cudaGraphExec_t ex = nullptr;
                    if (cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) {
                        cudaGraphDestroy(g);
                        return fail(PP_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(cudaGetLastError()));
                    }
                    c->ev_graph = g;
                    c->ev_exec = ex;
                    make_key(c->ev_key);
                    c->ev_key.pm_dirty = gkey.pm_dirty;  // (the state the graph was captured from)
                    c->ev_key.bad_pending = gkey.bad_pending;
                    c->ev_nb = nb;
                    for (int i = 0; i < nb; i++)
                        c->ev_bounce[i] = pp_ctx::EvalBounce{bounce[i].user == &bad_c ? nullptr : bounce[i].user,
                                                             bounce[i].off, bounce[i].bytes};
                    c->ev_bad_copy = bad_copy;
                    CUDA_TRY(cudaGraphLaunch(ex, st));
                }
                CUDA_TRY(stream_wait(st));
                ht.mark("sync");
                for (int i = 0; i < nb; i++) memcpy(bounce[i].user, c->h_bounce + bounce[i].off, bounce[i].bytes);
                TRY(check_schedule_range(c, bad_copy));
                if (bad_c) return fail(PP_ERR_INVALID_ARGS, "candidate block out of range [0, %d)", c->B);
                if (pairs) c->last_pairs = (size_t)std::max(0, *out->n_pairs);
                return PP_OK;
            }
        }
        if (capture) {  // (no single copy-out after all: run the captured launches once, uncached)
            cudaGraph_t g = nullptr;
            cguard.on = false;
            CUDA_TRY(cudaStreamEndCapture(st, &g));
            cudaGraphExec_t ex = nullptr;
            const cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
            if (e == cudaSuccess) {
                CUDA_TRY(cudaGraphLaunch(ex, st));
                CUDA_TRY(stream_wait(st));
            }
            if (ex) cudaGraphExecDestroy(ex);
            cudaGraphDestroy(g);
            if (e != cudaSuccess) return fail(PP_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(e));
        }
        CUDA_TRY(cudaMemcpyAsync(out->global, o.global, sizeof(pp_best), cudaMemcpyDeviceToHost, st));
        if (o.realism) CUDA_TRY(cudaMemcpyAsync(out->realism, o.realism, sizeof(pp_best), cudaMemcpyDeviceToHost, st));
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
        // sparse pairs: the count and a speculative prefix (sized from the previous call) in
        // the same round trip; the rest, if any, after the count is known
        size_t spec = 0;
        auto copy_pairs = [&](size_t lo, size_t hi) -> int {
            if (hi <= lo) return PP_OK;
            const size_t n = hi - lo;
            CUDA_TRY(cudaMemcpyAsync(out->pair_cand + lo, o.pair_cand + lo, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaMemcpyAsync(out->pair_period + lo, o.pair_period + lo, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaMemcpyAsync(out->pair_exp + lo, o.pair_exp + lo, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaMemcpyAsync(out->pair_cvar + lo, o.pair_cvar + lo, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
            return PP_OK;
        };
        if (pairs) {
            CUDA_TRY(cudaMemcpyAsync(out->n_pairs, o.n_pairs, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
            spec = std::min((size_t)C * T, c->last_pairs + c->last_pairs / 4 + 1024);
            TRY(copy_pairs(0, spec));
        }
        ht.mark("d2h enqueue");
        CUDA_TRY(stream_wait(st));
        ht.mark("sync");
        TRY(check_schedule_range(c, false));
        if (warp_path) {
            int32_t bad_c = 0;
            CUDA_TRY(cudaMemcpy(&bad_c, c->bad_cand.ptr, sizeof(int32_t), cudaMemcpyDeviceToHost));
            if (bad_c) return fail(PP_ERR_INVALID_ARGS, "candidate block out of range [0, %d)", c->B);
        }
        if (pairs) {
            const size_t n = (size_t)std::max(0, *out->n_pairs);
            c->last_pairs = n;
            if (n > spec) {
                TRY(copy_pairs(spec, n));
                CUDA_TRY(stream_wait(st));
            }
        }
    }
    return PP_OK;
}

}  // extern "C"
