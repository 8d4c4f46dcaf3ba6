// pp_npv.cu -- relaxed NPV of P schedules on the device: ScheduleEvaluator.npv_relaxed and
// per_scenario_npv (evaluate.py:222-258) on the single-mode fast path of the stage-2 problem
// (evaluate.py:166-183), bit-exact.  Population fitness of the GA loop (hybrid.py:595-606).
#include "pp_internal.cuh"
#include <cub/block/block_radix_sort.cuh>
#include <unordered_map>
#include <vector>

// ------------------------------------------------------------------------------------
// k_stage2: one CTA per (scenario s, period t, schedule p); periods of more than S2_NMAX mined
// blocks go to k_stage2_big (global-memory runs + merge), so every period size runs on the device.
//   1. the blocks mined in t, in block order (two vectorised passes: count, place);
//   2. the s == 0 CTA also sums their mining costs in numpy's pairwise order (for _npv);
//   3. density = v[s][b] / m[b]; stable descending block radix sort (cub), which is the order of
//      np.argsort(-density, kind="stable");
//   4. the greedy fill is a sequential f64 recurrence (hours_left, total), done by one thread
//      over arrays prepared in parallel (d, m and m / rate in sorted order), four blocks per
//      speculative step.
// ------------------------------------------------------------------------------------
#ifdef PP_EVAL_PROBE
__device__ unsigned long long g_npv_probe[8];
__device__ __forceinline__ unsigned long long np_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define NPVP(k) do { if (threadIdx.x == 0 && blockIdx.x == 1 && blockIdx.y == 0 && blockIdx.z == 0) g_npv_probe[k] = np_gtimer(); } while (0)
extern "C" PP_API int pp_debug_npv_probe(unsigned long long *out) {
    return cudaMemcpyFromSymbol(out, g_npv_probe, sizeof(g_npv_probe)) == cudaSuccess ? 0 : 3;
}
// kernel spans of one pp_npv_moves call: [id][0] earliest CTA start, [id][1] latest warp end
__device__ unsigned long long g_kspan[8][2];
#define KSPAN_BEGIN(id) do { if (threadIdx.x == 0) atomicMin(&g_kspan[id][0], np_gtimer()); } while (0)
#define KSPAN_END(id) do { if ((threadIdx.x & 31) == 0) atomicMax(&g_kspan[id][1], np_gtimer()); } while (0)
// per-call log of the spans (probe builds): npv_moves_impl appends one row per host-mode call
static std::vector<unsigned long long> g_kspan_log;
static void kspan_reset() {
    unsigned long long h[8][2];
    for (int i = 0; i < 8; i++) {
        h[i][0] = ~0ull;
        h[i][1] = 0ull;
    }
    cudaMemcpyToSymbol(g_kspan, h, sizeof(h));
}
static void kspan_append() {
    unsigned long long h[16];
    if (cudaMemcpyFromSymbol(h, g_kspan, sizeof(h)) == cudaSuccess) g_kspan_log.insert(g_kspan_log.end(), h, h + 16);
}
extern "C" PP_API int pp_debug_kspan_log(unsigned long long *out, int64_t max_rows, int64_t *rows) {
    const int64_t n = (int64_t)g_kspan_log.size() / 16;
    *rows = n;
    if (out) std::memcpy(out, g_kspan_log.data(), sizeof(unsigned long long) * 16 * (size_t)std::min(n, max_rows));
    g_kspan_log.clear();
    return 0;
}
extern "C" PP_API int pp_debug_kspan(unsigned long long *out, int reset) {
    if (reset) {
        unsigned long long h[8][2];
        for (int i = 0; i < 8; i++) {
            h[i][0] = ~0ull;
            h[i][1] = 0ull;
        }
        return cudaMemcpyToSymbol(g_kspan, h, sizeof(h)) == cudaSuccess ? 0 : 3;
    }
    return cudaMemcpyFromSymbol(out, g_kspan, sizeof(g_kspan)) == cudaSuccess ? 0 : 3;
}
#else
#define NPVP(k) do { } while (0)
#define KSPAN_BEGIN(id) do { } while (0)
#define KSPAN_END(id) do { } while (0)
#endif

constexpr int S2_THREADS = 1024;
constexpr int S2_IPT = 6;                        // items per thread of the block radix sort
constexpr int S2_NMAX = S2_THREADS * S2_IPT;     // mined blocks per period handled on chip
using S2Sort = cub::BlockRadixSort<double, S2_THREADS, S2_IPT, int>;
using S2Sort1 = cub::BlockRadixSort<double, S2_THREADS, 1, int>;  // periods of <= 1,024 blocks

// dynamic shared memory: [sort temp | later: density d (sorted)] [ids] [m (sorted)] [m / rate (sorted)]
struct S2Layout {
    __host__ __device__ static constexpr size_t a_bytes() {
        return sizeof(typename S2Sort::TempStorage) > 8 * (size_t)S2_NMAX ? sizeof(typename S2Sort::TempStorage)
                                                                              : 8 * (size_t)S2_NMAX;
    }
    __host__ __device__ static constexpr size_t ids_off() { return (a_bytes() + 15) & ~(size_t)15; }
    __host__ __device__ static constexpr size_t m_off() { return ids_off() + 4 * (size_t)S2_NMAX; }
    __host__ __device__ static constexpr size_t q_off() { return m_off() + 8 * (size_t)S2_NMAX; }
    __host__ __device__ static constexpr size_t bytes() { return q_off() + 8 * (size_t)S2_NMAX; }
};


// The blocks of schedule `a` (block ob moved to period ot when ob >= 0) mined in period t, in
// block order: warp w owns [w*chunk, (w+1)*chunk), 128 blocks per step (int4 per lane when
// aligned).  Returns n on every thread; writes ids[0..n) only when n <= nmax.  1024 threads.
__device__ int s2_compact(const int32_t *__restrict__ a, int B, int t, int ob, int ot, int32_t *ids, int nmax) {
    __shared__ int s_wc[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int chunk = ((B + 31) / 32 + 127) & ~127;
    const int lo = warp * chunk, hi = min(B, lo + chunk);
    const bool vec = (B & 3) == 0;
    auto load4 = [&](int b0, int v[4]) {
        const int b = b0 + 4 * lane;
        if (vec && b + 3 < hi) {
            const int4 x = __ldg(reinterpret_cast<const int4 *>(a + b));
            v[0] = x.x;
            v[1] = x.y;
            v[2] = x.z;
            v[3] = x.w;
        } else {
#pragma unroll
            for (int u = 0; u < 4; u++) v[u] = (b + u < hi) ? __ldg(a + b + u) : -2;
        }
        if (ob >= b && ob < b + 4) v[ob - b] = ot;  // the variant's moved block
    };
    int cnt = 0;
    for (int b0 = lo; b0 < hi; b0 += 128) {
        int v[4];
        load4(b0, v);
        cnt += (v[0] == t) + (v[1] == t) + (v[2] == t) + (v[3] == t);
    }
    cnt = __reduce_add_sync(0xffffffffu, (unsigned)cnt);
    if (lane == 0) s_wc[warp] = cnt;
    __syncthreads();
    int base = 0, n = 0;
    for (int w = 0; w < 32; w++) {
        base += w < warp ? s_wc[w] : 0;
        n += s_wc[w];
    }
    __syncthreads();  // s_wc is reused by the next call
    if (n > nmax) return n;
    for (int b0 = lo; b0 < hi; b0 += 128) {
        int v[4];
        load4(b0, v);
        const int c = (v[0] == t) + (v[1] == t) + (v[2] == t) + (v[3] == t);
        int incl = c;  // lanes own consecutive groups of 4 blocks: exclusive scan of the counts
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        int q = base + incl - c;
#pragma unroll
        for (int u = 0; u < 4; u++)
            if (v[u] == t) ids[q++] = b0 + 4 * lane + u;
        base += __shfl_sync(0xffffffffu, incl, 31);
    }
    return n;
}

// The greedy fill of evaluate.py:174-182 over n blocks in density order (d(k) > 0 for k < kpos,
// m(k) the mass, q(k) = m(k) / rate): a sequential f64 recurrence (hours_left, total).  Warp 0
// takes 32 blocks per step speculatively as whole blocks: every lane runs the two chains
// hours_left -= m / rate and total += d * m over the step's 32 blocks (values broadcast through
// shared memory, the same adds in the same order) and lane j keeps the values before block j;
// then each lane tests its block for a stop (k >= kpos, hours_left <= 0) or a partial take
// (hours_left * rate < m).  At the first flagged block the exact scalar loop takes over from
// that block's hours_left and total.  Call from warp 0 only; the result is on lane 0.
// With rec_h / rec_t (may be null) the state before every processed position k -- (hours_left,
// total) -- is recorded for k = 0..K, K the position where the loop stopped (K = n when it ran
// through), and K goes to *rec_k: the prefix an incremental variant restarts from (k_s2_chain).
// Progress flags of the one-block base update (k_s2_apply_one) that the variants' kernels of the
// same call read while it still runs (programmatic dependent launch: all its CTAs are resident
// before theirs start, so the waits cannot deadlock).  A flag is (call epoch << 32) | x:
// x = valid + 2 once the splice is in place and the recorded states H/TT[k] are final for
// k < valid; x = S2_DONE when the period's structure, stop K and stage-2 value are final.
constexpr unsigned S2_DONE = 0xffffffffu;
__device__ __forceinline__ unsigned long long s2_flag_load(const unsigned long long *f) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
    return v;
}
__device__ __forceinline__ void s2_flag_publish(unsigned long long *f, unsigned long long v) {
    __threadfence();  // the caller's (and, through the preceding barrier, its group's) writes first
    atomicExch(f, v);
}
__device__ __forceinline__ unsigned long long s2_flag_wait(const unsigned long long *f, unsigned long long need) {
    unsigned long long v;
    long long spins = 0;
    while ((v = s2_flag_load(f)) < need) {  // bounded: a lost update traps instead of hanging the GPU
        __nanosleep(100);
        if (++spins > (1ll << 26)) __trap();
    }
    return v;
}

// The 32 steps of one batch of the greedy recurrence (evaluate.py:174-182, whole takes): every lane
// runs the same two add chains over the batch's terms (q = m / rate, dm = d * m, staged in the
// warp's shared slots) and keeps the state before its own element.  The terms are read eight at a
// time into registers ahead of their adds (tools/walk_bench.cu: 41 -> 23 cycles per element with
// the inputs loaded one batch ahead, against 52 for the plain broadcast-read loop).
__device__ __forceinline__ void s2_batch_steps(const double *__restrict__ sq, const double *__restrict__ sdm, int lane,
                                               double &h, double &tt, double &h_mine, double &t_mine) {
#pragma unroll
    for (int g = 0; g < 4; g++) {
        double qa[8], da[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
            qa[u] = sq[g * 8 + u];
            da[u] = sdm[g * 8 + u];
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
            if (lane == g * 8 + u) {
                h_mine = h;
                t_mine = tt;
            }
            h = f64_sub(h, qa[u]);
            tt = f64_add(tt, da[u]);
        }
    }
}

template <class DF, class MF, class QF>
__device__ double s2_greedy_warp(int n, int kpos, double hours0, double rate, DF dof, MF mof, QF qof,
                                 double *rec_h = nullptr, double *rec_t = nullptr, int32_t *rec_k = nullptr,
                                 int k_begin = 0, double total0 = 0.0, unsigned long long *prog = nullptr,
                                 unsigned long long eh = 0) {
    // k_begin / total0: resume at position k_begin with state (hours0, total0) -- the recorded
    // state there (an incremental base update, k_s2_apply_one)
    __shared__ double s_q32[32], s_dm32[32];
    const int lane = threadIdx.x & 31;
    double hl = hours0, total = total0;
    int k = n;
    // each lane's element of the next batch is loaded one batch ahead (qof(k) is m / rate at every
    // call site: the term is formed from the loaded mass)
    double m_nx = 0.0, d_nx = 0.0;
    if (k_begin + lane < n) {
        m_nx = mof(k_begin + lane);
        d_nx = dof(k_begin + lane);
    }
    for (int k0 = k_begin; k0 < n; k0 += 32) {
        const int kk = k0 + lane;
        const bool in = kk < n;
        const double m = in ? m_nx : 0.0;
        s_q32[lane] = in ? f64_div(m, rate) : 0.0;
        s_dm32[lane] = in ? f64_mul(d_nx, m) : 0.0;
        if (kk + 32 < n) {
            m_nx = mof(kk + 32);
            d_nx = dof(kk + 32);
        }
        __syncwarp();
        double h = hl, tt = total, h_mine = 0.0, t_mine = 0.0;
        s2_batch_steps(s_q32, s_dm32, lane, h, tt, h_mine, t_mine);
        __syncwarp();
        const bool stop = !in || kk >= kpos || !(h_mine > 0) || f64_mul(h_mine, rate) < m;
        const unsigned sm = __ballot_sync(0xffffffffu, stop);
        if (rec_h && in && (!sm || lane <= __ffs(sm) - 1)) {
            rec_h[kk] = h_mine;
            rec_t[kk] = t_mine;
        }
        if (prog && !sm && (((k0 - k_begin) >> 5) & 7) == 7) {  // every 8 batches: states < k0 + 32 final
            __threadfence();
            __syncwarp();
            if (lane == 0) atomicExch(prog, eh | (unsigned long long)(k0 + 32 + 2));
        }
        if (sm) {
            const int jf = __ffs(sm) - 1;
            k = k0 + jf;
            hl = __shfl_sync(0xffffffffu, h_mine, jf);
            total = __shfl_sync(0xffffffffu, t_mine, jf);
            break;
        }
        hl = h;
        total = tt;
    }
    if (lane == 0) {
        for (; k < n; k++) {
            if (rec_h) {
                rec_h[k] = hl;
                rec_t[k] = total;
            }
            if (k >= kpos || hl <= 0) break;
            const double d = dof(k);
            const double mk = mof(k);
            const double hr = f64_mul(hl, rate);
            if (hr < mk) {  // take = min(m, hours_left * rate) = hours_left * rate
                total = f64_add(total, f64_mul(d, hr));
                hl = f64_sub(hl, f64_div(hr, rate));
            } else {
                total = f64_add(total, f64_mul(d, mk));
                hl = f64_sub(hl, qof(k));
            }
        }
        if (rec_h) {
            if (k >= n) {
                rec_h[n] = hl;
                rec_t[n] = total;
            }
            *rec_k = k < n ? k : n;
        }
    }
    return total;
}

// Per-(scenario, period) structure of one base schedule, kept on the device between pp_npv_moves
// calls so a one-block variant is valued incrementally (k_s2_chain) instead of re-sorting:
//   D/M/BID [S][T][L]  the period's blocks with density > 0 in greedy order (density desc, block
//                      asc), their masses and ids; npos[S][T] of them
//   H/TT    [S][T][L]  (hours_left, total) before position k, k = 0..K[S][T] (K = where the loop
//                      stopped; npos when it ran through)
//   pos     [S][B]     position of block b in its period's list, -1 if its density is <= 0
//   IDS     [T][L]     the period's mined blocks in block order; nper[T] of them
//   CS      [T][L]     their mining costs cost[b][t] in that order (the variants' cost sums)
// L = B + 1.  All pointers null = not recorded.
struct S2Struct {
    double *D, *M, *H, *TT, *CS;
    int32_t *BID, *npos, *K, *pos, *IDS, *nper;
    int L;
};

// Work item of the large-period path: (scenario, grid y, grid z) of a k_stage2 CTA whose period
// has more than S2_NMAX mined blocks.
struct S2Item {
    int s, y, z, n;
};

__global__ void __launch_bounds__(S2_THREADS, 1)
    k_stage2(const int32_t *__restrict__ assign, int B, int T, int S, int Sp, const double *__restrict__ mass,
             const double *__restrict__ cost, const double *__restrict__ vmax, const double *__restrict__ hours,
             double rate, double *__restrict__ raw, double *__restrict__ costsum, int32_t *__restrict__ nmined,
             S2Item *__restrict__ big_items, int32_t *__restrict__ big_count, const int32_t *__restrict__ ovr_b,
             const int32_t *__restrict__ ovr_t, const int32_t *__restrict__ slot_t, const int32_t *__restrict__ tsel,
             const S2Struct rec) {
    extern __shared__ __align__(16) unsigned char s2_dyn[];
    typename S2Sort::TempStorage &sort_tmp = *reinterpret_cast<typename S2Sort::TempStorage *>(s2_dyn);
    double *dsort = reinterpret_cast<double *>(s2_dyn);  // after the sort
    int32_t *ids = reinterpret_cast<int32_t *>(s2_dyn + S2Layout::ids_off());
    double *ms = reinterpret_cast<double *>(s2_dyn + S2Layout::m_off());
    double *qs = reinterpret_cast<double *>(s2_dyn + S2Layout::q_off());
    __shared__ int s_ls[160], s_ll[160];
    __shared__ double s_scr[160];
    // whole schedules: grid (S, T, P), blockIdx.y = period.  One-block variants of a single base
    // schedule (ovr_b != nullptr): grid (S, 2, M), variant m = base with block ovr_b[m] in period
    // ovr_t[m], blockIdx.y = slot of the two periods it changes (slot_t[m][slot], -1 = none)
    const int s = blockIdx.x, p = blockIdx.z;
    const int t = ovr_b ? slot_t[2 * p + blockIdx.y] : (tsel ? tsel[blockIdx.y] : (int)blockIdx.y);
    const int tid = threadIdx.x;
    if (t < 0) return;
    NPVP(0);
    const bool record = rec.D != nullptr;  // whole single schedule (ovr_b == nullptr, P == 1)
    const size_t rst = ((size_t)s * T + t) * rec.L;
    const int32_t *a = ovr_b ? assign : assign + (size_t)p * B;
    const int ob = ovr_b ? ovr_b[p] : -1, ot = ovr_b ? ovr_t[p] : -1;
    // 1. blocks mined in t, block order
    const int n = s2_compact(a, B, t, ob, ot, ids, S2_NMAX);
    const size_t pt = ovr_b ? (size_t)2 * p + blockIdx.y : ((size_t)p * T + t);
    if (n > S2_NMAX) {  // larger than the on-chip buffers: handed to k_stage2_big
        if (tid == 0) big_items[atomicAdd(big_count, 1)] = S2Item{s, (int)blockIdx.y, p, n};
        return;
    }
    __syncthreads();
    NPVP(1);
    // 2. mining-cost sum of the period (numpy pairwise, block order), once per (p, t)
    if (s == 0) {
        for (int k = tid; k < n; k += S2_THREADS) {
            ms[k] = __ldg(cost + (size_t)ids[k] * T + t);
            if (record) {
                rec.IDS[(size_t)t * rec.L + k] = ids[k];
                rec.CS[(size_t)t * rec.L + k] = ms[k];
            }
        }
        __syncthreads();
        const double cs = s2_pairwise(ms, n, s_ls, s_ll, s_scr);
        if (tid == 0) {
            costsum[pt] = cs;
            nmined[pt] = n;
            if (record) rec.nper[t] = n;
        }
        __syncthreads();
    }
    if (n == 0) {
        if (tid == 0) {
            raw[pt * S + s] = 0.0;
            if (record) {
                rec.npos[(size_t)s * T + t] = 0;
                rec.K[(size_t)s * T + t] = 0;
                rec.H[rst] = __ldg(hours + t);
                rec.TT[rst] = 0.0;
            }
        }
        return;
    }
    // 3. densities, stable descending radix sort (= np.argsort(-density, kind="stable"); the order
    //    among densities <= 0 is irrelevant: the greedy stops at the first one)
    if (n <= S2_THREADS) {  // one key per thread: a sixth of the radix passes' work
        double d1[1];
        int i1[1];
        d1[0] = tid < n ? f64_div(__ldg(vmax + (size_t)ids[tid] * Sp + s), __ldg(mass + ids[tid])) : -kInf;
        i1[0] = tid;
        S2Sort1(*reinterpret_cast<typename S2Sort1::TempStorage *>(s2_dyn)).SortDescending(d1, i1);
        __syncthreads();  // the sort's temp storage becomes the sorted densities
        if (tid < n) {
            const int bb = ids[i1[0]];
            const double m = __ldg(mass + bb);
            dsort[tid] = d1[0];
            ms[tid] = m;
            qs[tid] = f64_div(m, rate);
            if (record) {
                rec.D[rst + tid] = d1[0];
                rec.M[rst + tid] = m;
                rec.BID[rst + tid] = bb;
                rec.pos[(size_t)s * B + bb] = d1[0] > 0 ? tid : -1;
            }
        }
    } else {
        double dk[S2_IPT];
        int ik[S2_IPT];
#pragma unroll
        for (int u = 0; u < S2_IPT; u++) {
            const int k = tid * S2_IPT + u;  // blocked arrangement: thread order = position order
            if (k < n) {
                const int b = ids[k];
                dk[u] = f64_div(__ldg(vmax + (size_t)b * Sp + s), __ldg(mass + b));
            } else {
                dk[u] = -kInf;
            }
            ik[u] = k;
        }
        S2Sort(sort_tmp).SortDescending(dk, ik);
        __syncthreads();  // the sort's temp storage becomes the sorted densities
#pragma unroll
        for (int u = 0; u < S2_IPT; u++) {
            const int k = tid * S2_IPT + u;
            if (k < n) {
                const int bb = ids[ik[u]];
                const double m = __ldg(mass + bb);
                dsort[k] = dk[u];
                ms[k] = m;
                qs[k] = f64_div(m, rate);
                if (record) {
                    rec.D[rst + k] = dk[u];
                    rec.M[rst + k] = m;
                    rec.BID[rst + k] = bb;
                    rec.pos[(size_t)s * B + bb] = dk[u] > 0 ? k : -1;
                }
            }
        }
    }
    __syncthreads();
    NPVP(3);
    // 4. the greedy fill (evaluate.py:174-182)
    __shared__ int s_kpos;
    if (tid == 0) s_kpos = n;
    __syncthreads();
    for (int k = tid; k < n; k += S2_THREADS)
        if (dsort[k] <= 0) atomicMin(&s_kpos, k);  // first d <= 0 (the scalar loop's stop)
    __syncthreads();
    if (tid < 32) {
        const int kpos = s_kpos;
        const double total = s2_greedy_warp(
            kpos, kpos, __ldg(hours + t), rate, [&](int k) { return dsort[k]; }, [&](int k) { return ms[k]; },
            [&](int k) { return qs[k]; }, record ? rec.H + rst : nullptr, record ? rec.TT + rst : nullptr,
            record ? rec.K + (size_t)s * T + t : nullptr);
        if (tid == 0) {
            raw[pt * S + s] = total;
            if (record) rec.npos[(size_t)s * T + t] = kpos;
        }
    }
    NPVP(4);
}

// strict total order of the large-period sort: density descending, then block ascending -- the
// order of np.argsort(-density, kind="stable") over blocks listed in block order
__device__ __forceinline__ bool s2_before(double da, int ba, double db, int bb) {
    return da > db || (da == db && ba < bb);
}

// Per-CTA global scratch of the large-period path (n <= B): ids | keys A | keys B | blocks A | blocks B
__host__ __device__ inline size_t s2_big_stride(int B) { return (size_t)B * 28 + 64; }

// k_stage2_big: the (s, t, schedule) problems whose period mines more than S2_NMAX blocks, one
// persistent CTA per SM looping over the work list k_stage2 filled.  Same steps and arithmetic as
// k_stage2 with the arrays in L2-resident global scratch:
//   1. compaction of the period's blocks into ids[] (block order);
//   2. s == 0: mining-cost sum, numpy pairwise order, over ids[];
//   3. (density, block) of every block with density > 0 (the greedy stops at the first d <= 0, so
//      the others never matter), in block order;
//   4. sort: runs of S2_NMAX sorted on chip by the block radix sort (stable: ties keep block
//      order), then pairwise merge-path rounds over the strict (density desc, block asc) order;
//   5. the greedy fill over the sorted prefix (s2_greedy_warp).
__global__ void __launch_bounds__(S2_THREADS, 1)
    k_stage2_big(const int32_t *__restrict__ assign, int B, int T, int S, int Sp, const double *__restrict__ mass,
                 const double *__restrict__ cost, const double *__restrict__ vmax, const double *__restrict__ hours,
                 double rate, double *__restrict__ raw, double *__restrict__ costsum, int32_t *__restrict__ nmined,
                 const S2Item *__restrict__ items, const int32_t *__restrict__ count, unsigned char *__restrict__ scratch,
                 const int32_t *__restrict__ ovr_b, const int32_t *__restrict__ ovr_t,
                 const int32_t *__restrict__ slot_t, const int32_t *__restrict__ tsel, const S2Struct rec) {
    extern __shared__ __align__(16) unsigned char s2_dyn[];
    typename S2Sort::TempStorage &sort_tmp = *reinterpret_cast<typename S2Sort::TempStorage *>(s2_dyn);
    __shared__ int s_np;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned char *base = scratch + (size_t)blockIdx.x * s2_big_stride(B);
    int32_t *ids = reinterpret_cast<int32_t *>(base);
    double *ka = reinterpret_cast<double *>(base + (((size_t)B * 4 + 15) & ~(size_t)15));
    double *kb = ka + B;
    int32_t *ba = reinterpret_cast<int32_t *>(kb + B);
    int32_t *bb = ba + B;
    const int nitems = *count;
    for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
        const S2Item it = items[w];
        const int s = it.s, p = it.z;
        const int t = ovr_b ? slot_t[2 * p + it.y] : (tsel ? tsel[it.y] : it.y);
        const bool record = rec.D != nullptr;
        const size_t rst = ((size_t)s * T + t) * rec.L;
        const int32_t *a = ovr_b ? assign : assign + (size_t)p * B;
        const int ob = ovr_b ? ovr_b[p] : -1, ot = ovr_b ? ovr_t[p] : -1;
        const size_t pt = ovr_b ? (size_t)2 * p + it.y : ((size_t)p * T + t);
        __syncthreads();  // the previous item's readers of the scratch are done
        // 1.
        const int n = s2_compact(a, B, t, ob, ot, ids, B);
        __syncthreads();
        // 2.
        if (record)  // every block of the period leaves its scenario-s position unset ...
            for (int k = tid; k < n; k += S2_THREADS) rec.pos[(size_t)s * B + ids[k]] = -1;
        if (s == 0) {
            for (int k = tid; k < n; k += S2_THREADS) {
                kb[k] = __ldg(cost + (size_t)ids[k] * T + t);
                if (record) {
                    rec.IDS[(size_t)t * rec.L + k] = ids[k];
                    rec.CS[(size_t)t * rec.L + k] = kb[k];
                }
            }
            __syncthreads();
            // leaves: at most n/64 + 2 of them, in ba / bb; leaf values in ka
            const double cs = s2_pairwise(kb, n, ba, bb, ka);
            if (tid == 0) {
                costsum[pt] = cs;
                nmined[pt] = n;
                if (record) rec.nper[t] = n;
            }
            __syncthreads();
        }
        // 3. positive densities in block order: per 1024-tile, a ballot scan
        if (tid == 0) s_np = 0;
        __syncthreads();
        for (int k0 = 0; k0 < n; k0 += S2_THREADS) {
            const int k = k0 + tid;
            double d = 0.0;
            int b = -1;
            if (k < n) {
                b = ids[k];
                d = f64_div(__ldg(vmax + (size_t)b * Sp + s), __ldg(mass + b));
            }
            const bool keep = k < n && d > 0;
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            __shared__ int s_wcnt[32];
            if (lane == 0) s_wcnt[warp] = __popc(bal);
            __syncthreads();
            int off = s_np;
            for (int x = 0; x < warp; x++) off += s_wcnt[x];
            if (keep) {
                const int q = off + __popc(bal & ((1u << lane) - 1u));
                ka[q] = d;
                ba[q] = b;
            }
            __syncthreads();
            if (tid == 0) {
                int tot = 0;
                for (int x = 0; x < 32; x++) tot += s_wcnt[x];
                s_np += tot;
            }
            __syncthreads();
        }
        const int np_ = s_np;
        // 4a. runs of S2_NMAX sorted on chip (blocked arrangement in block order: stable)
        for (int r0 = 0; r0 < np_; r0 += S2_NMAX) {
            const int rn = min(S2_NMAX, np_ - r0);
            double dk[S2_IPT];
            int ik[S2_IPT];
#pragma unroll
            for (int u = 0; u < S2_IPT; u++) {
                const int k = tid * S2_IPT + u;
                dk[u] = k < rn ? ka[r0 + k] : -kInf;
                ik[u] = k < rn ? ba[r0 + k] : INT_MAX;
            }
            __syncthreads();
            S2Sort(sort_tmp).SortDescending(dk, ik);
#pragma unroll
            for (int u = 0; u < S2_IPT; u++) {
                const int k = tid * S2_IPT + u;
                if (k < rn) {
                    ka[r0 + k] = dk[u];
                    ba[r0 + k] = ik[u];
                }
            }
            __syncthreads();
        }
        // 4b. merge rounds, ping-pong between (ka, ba) and (kb, bb)
        double *srck = ka, *dstk = kb;
        int32_t *srcb = ba, *dstb = bb;
        for (int wdt = S2_NMAX; wdt < np_; wdt *= 2) {
            for (int m0 = 0; m0 < np_; m0 += 2 * wdt) {
                const int mid = min(m0 + wdt, np_), end = min(m0 + 2 * wdt, np_);
                const int la = mid - m0, lb = end - mid, L = la + lb;
                const double *Ak = srck + m0, *Bk = srck + mid;
                const int32_t *Ab = srcb + m0, *Bb = srcb + mid;
                const int per = (L + S2_THREADS - 1) / S2_THREADS;
                const int d0 = min(tid * per, L), d1 = min(d0 + per, L);
                if (d0 < d1) {
                    int lo = max(0, d0 - lb), hi = min(d0, la);  // merge path: A elements among the first d0
                    while (lo < hi) {
                        const int md = (lo + hi) >> 1;
                        if (s2_before(Ak[md], Ab[md], Bk[d0 - 1 - md], Bb[d0 - 1 - md]))
                            lo = md + 1;
                        else
                            hi = md;
                    }
                    int ia = lo, ib = d0 - lo;
                    PP_DCHECK(ia >= 0 && ia <= la && ib >= 0 && ib <= lb && m0 + d1 <= np_ && np_ <= B);
                    for (int k = d0; k < d1; k++) {
                        const bool takeA = ib >= lb || (ia < la && s2_before(Ak[ia], Ab[ia], Bk[ib], Bb[ib]));
                        if (takeA) {
                            dstk[m0 + k] = Ak[ia];
                            dstb[m0 + k] = Ab[ia];
                            ia++;
                        } else {
                            dstk[m0 + k] = Bk[ib];
                            dstb[m0 + k] = Bb[ib];
                            ib++;
                        }
                    }
                }
            }
            __syncthreads();
            double *tk = srck;
            srck = dstk;
            dstk = tk;
            int32_t *tb = srcb;
            srcb = dstb;
            dstb = tb;
        }
        if (record) {  // ... and the positives get their place in the greedy order (after the -1s above)
            __syncthreads();
            for (int k = tid; k < np_; k += S2_THREADS) {
                const int bb = srcb[k];
                rec.D[rst + k] = srck[k];
                rec.M[rst + k] = __ldg(mass + bb);
                rec.BID[rst + k] = bb;
                rec.pos[(size_t)s * B + bb] = k;
            }
        }
        // 5. the greedy fill over the positive prefix
        if (tid < 32) {
            const double *dk_ = srck;
            const int32_t *bk_ = srcb;
            const double total = s2_greedy_warp(
                np_, np_, __ldg(hours + t), rate, [&](int k) { return dk_[k]; },
                [&](int k) { return __ldg(mass + bk_[k]); }, [&](int k) { return f64_div(__ldg(mass + bk_[k]), rate); },
                record ? rec.H + rst : nullptr, record ? rec.TT + rst : nullptr,
                record ? rec.K + (size_t)s * T + t : nullptr);
            if (tid == 0) {
                raw[pt * S + s] = total;
                if (record) rec.npos[(size_t)s * T + t] = np_;
            }
        }
    }
}

// Launches the stage-2 problems of grid (S, gy, gz): k_stage2 for every period that fits on chip,
// then k_stage2_big for the rest (only when some period can exceed S2_NMAX, i.e. B > S2_NMAX).
static int run_stage2(pp_ctx *c, cudaStream_t st, const int32_t *da, int gy, int gz, double *raw, double *costsum,
                      int32_t *nmined, const int32_t *ovr_b, const int32_t *ovr_t, const int32_t *slot_t,
                      const int32_t *tsel = nullptr, const S2Struct *rec = nullptr, bool may_be_big = true) {
    const S2Struct none{};
    const S2Struct &rc = rec ? *rec : none;
    const int B = c->B, T = c->T, S = c->S;
    const bool big = B > S2_NMAX && may_be_big;
    TRY(c->s2_items.ensure(sizeof(S2Item) * (size_t)S * gy * gz + 16));
    int32_t *count = reinterpret_cast<int32_t *>(c->s2_items.as<unsigned char>() + sizeof(S2Item) * (size_t)S * gy * gz);
    S2Item *items = c->s2_items.as<S2Item>();
    if (big) CUDA_TRY(cudaMemsetAsync(count, 0, sizeof(int32_t), st));
    TRY(ensure_max_smem(k_stage2, S2Layout::bytes(), c->device));
    k_stage2<<<dim3(S, gy, gz), S2_THREADS, S2Layout::bytes(), st>>>(
        da, B, T, S, c->Sp, c->mass.as<double>(), c->cost.as<double>(), c->vmax.as<double>(), c->hours.as<double>(),
        c->rate, raw, costsum, nmined, items, count, ovr_b, ovr_t, slot_t, tsel, rc);
    CUDA_TRY(cudaGetLastError());
    if (!big) return PP_OK;
    int sms = 148;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device) != cudaSuccess || sms < 1) sms = 148;
    // one CTA per SM, scratch budget 1 GiB
    const size_t stride = s2_big_stride(B);
    const int grid = (int)std::max<size_t>(1, std::min<size_t>((size_t)sms, ((size_t)1 << 30) / stride));
    TRY(c->s2_scratch.ensure(stride * grid));
    TRY(ensure_max_smem(k_stage2_big, S2Layout::bytes(), c->device));
    k_stage2_big<<<grid, S2_THREADS, S2Layout::bytes(), st>>>(
        da, B, T, S, c->Sp, c->mass.as<double>(), c->cost.as<double>(), c->vmax.as<double>(), c->hours.as<double>(),
        c->rate, raw, costsum, nmined, items, count, c->s2_scratch.as<unsigned char>(), ovr_b, ovr_t, slot_t, tsel,
        rc);
    CUDA_TRY(cudaGetLastError());
    return PP_OK;
}


// ------------------------------------------------------------------------------------
// Incremental one-block variants (pp_npv_moves).  A variant moves block b from period t_old to
// t_new; only those two periods' stage-2 problems change.  With the base schedule's greedy
// order and its recorded prefix states (S2Struct) each re-solve is exact without a sort:
//   leave t_old: b sits at position j of the (s, t_old) order (pos[s][b]; absent if its density
//                is <= 0, then nothing changes); restart the recurrence from the state before j
//                and continue with positions j+1, j+2, ...
//   enter t_new: its position j is the binary search of (density, b) in the (s, t_new) order;
//                restart from the state before j with b, then positions j, j+1, ...
// A position beyond the base's stop K leaves the result unchanged.  The recurrence is the
// scalar loop of evaluate.py:174-182 verbatim, so the values equal a full re-solve bit for bit.
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_s2_chain(const S2Struct rec, int B, int T, int S, int Sp, int M,
                                                  const int32_t *__restrict__ blocks, const int32_t *__restrict__ slot_t,
                                                  const int32_t *__restrict__ run, const double *__restrict__ vmax,
                                                  const double *__restrict__ mass, double rate,
                                                  const double *__restrict__ braw, double *__restrict__ mraw,
                                                  const unsigned long long *__restrict__ prog, unsigned long long eh,
                                                  int pend0, int pend1) {
    // pend0 / pend1: the periods k_s2_apply_one is updating concurrently (-1: none); a variant in
    // one of them waits for the splice, then for the recorded state at its place (or the end)
    // one warp per (slot, scenario): lanes load 32 consecutive elements of the modified order at a
    // time (coalesced, one batch ahead), every lane runs the speculative whole-take recurrence over
    // them (the adds of the scalar loop, in its order), and the first element where the scalar loop
    // would stop or take partially hands over to the exact scalar tail -- as s2_greedy_warp.  (A
    // thread per chain measured 2.8x slower: each chain walks its own list, so the loads of a thread
    // are serialised by latency; the warp's coalesced batches are not.)
    constexpr unsigned FULL = 0xffffffffu;
    asm volatile("griddepcontrol.launch_dependents;");  // the accumulation may start (it waits for us)
    KSPAN_BEGIN(2);
    const int lane = threadIdx.x & 31;
    const long long unit = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (unit >= 2ll * M * S) return;
    const int s = (int)(unit % S), si = (int)(unit / S);
    const int t = slot_t[si];
    if (t < 0 || run[si] < 0) return;
    const int b = blocks[si >> 1];
    const size_t st_ = (size_t)s * T + t, base = st_ * rec.L;
    const int y = t == pend0 ? 0 : (t == pend1 ? 1 : -1);
    const unsigned long long *pf = y >= 0 ? prog + (size_t)y * S + s : nullptr;
    if (pf) s2_flag_wait(pf, eh | 2ull);  // the spliced order, npos and positions
    const int np = __ldcg(rec.npos + st_);
    int K = __ldcg(rec.K + st_);
    PP_DCHECK(np >= 0 && np < rec.L);
    const double *D = rec.D + base, *Mm = rec.M + base;
    const bool ins = si & 1;
    double dnew = 0.0, mnew = 0.0;
    int j;
    if (!ins) {
        j = __ldcg(rec.pos + (size_t)s * B + b);
        PP_DCHECK(j < 0 || (j < np && rec.BID[base + j] == b));  // pos[] points at b's place
    } else {
        mnew = __ldg(mass + b);
        dnew = f64_div(__ldg(vmax + (size_t)b * Sp + s), mnew);
        j = -1;
        if (dnew > 0) {  // first position that does not precede (dnew, b) in the greedy order
            const int32_t *BI = rec.BID + base;
            int lo = 0, hi = np;
            while (lo < hi) {
                const int md = (lo + hi) >> 1;
                const double dm = __ldcg(D + md);
                if (dm > dnew || (dm == dnew && __ldcg(BI + md) < b))
                    lo = md + 1;
                else
                    hi = md;
            }
            j = lo;
        }
    }
    if (pf) {  // the state at j recorded (the update's walk passed j), or the update done; a variant
               // that leaves the order unchanged (j < 0) reads the updated base value: done
        const unsigned long long v = s2_flag_wait(pf, j >= 0 ? (eh | (unsigned long long)(j + 3)) : (eh | S2_DONE));
        K = (unsigned)v == S2_DONE ? __ldcg(rec.K + st_) : INT_MAX;  // not done: j is before the stop
    }
    PP_DCHECK(K >= 0 && (K == INT_MAX || K <= np));
    if (j < 0 || j > K) {  // the variant's order agrees with the base's up to its stop
        if (lane == 0) mraw[(size_t)si * S + s] = __ldcg(braw + (size_t)t * S + s);
        KSPAN_END(2);
        return;
    }
    // the modified order: element e = the inserted block (e = 0) then positions j, j+1, ... , or
    // positions j+1, j+2, ... after a removal
    const int E = ins ? np - j + 1 : np - j - 1;
    auto elem = [&](int e, double &d, double &m) {
        if (ins && e == 0) {
            d = dnew;
            m = mnew;
        } else {
            const int k = ins ? j + e - 1 : j + 1 + e;
            PP_DCHECK(k >= 0 && k < np);
            d = __ldcg(D + k);
            m = __ldcg(Mm + k);
        }
    };
    double hl = __ldcg(rec.H + base + j), tot = __ldcg(rec.TT + base + j);
    int e = E;
    __shared__ double s_qd[8][64];
    double *wq_ = s_qd[threadIdx.x >> 5], *wdm = wq_ + 32;
    double dnx = 0.0, mnx = 0.0;  // the next batch's element, loaded one batch ahead
    if (lane < E) elem(lane, dnx, mnx);
    for (int e0 = 0; e0 < E; e0 += 32) {
        const int ee = e0 + lane;
        const bool in = ee < E;
        const double d = dnx, m = mnx;
        if (ee + 32 < E) elem(ee + 32, dnx, mnx);
        // the batch's terms through shared memory (broadcast reads, off the add chains)
        wq_[lane] = in ? f64_div(m, rate) : 0.0;
        wdm[lane] = in ? f64_mul(d, m) : 0.0;
        __syncwarp();
        double h = hl, tt = tot, h_mine = 0.0, t_mine = 0.0;
        s2_batch_steps(wq_, wdm, lane, h, tt, h_mine, t_mine);
        __syncwarp();
        const bool stop = !in || !(h_mine > 0) || f64_mul(h_mine, rate) < m;
        const unsigned sm = __ballot_sync(FULL, stop);
        if (sm) {
            const int jf = __ffs(sm) - 1;
            e = e0 + jf;
            hl = __shfl_sync(FULL, h_mine, jf);
            tot = __shfl_sync(FULL, t_mine, jf);
            break;
        }
        hl = h;
        tot = tt;
    }
    if (lane == 0) {
        for (; e < E; e++) {  // the scalar loop of evaluate.py:174-182
            if (hl <= 0) break;
            double d, m;
            elem(e, d, m);
            const double hr = f64_mul(hl, rate);
            if (hr < m) {  // take = hours_left * rate
                tot = f64_add(tot, f64_mul(d, hr));
                hl = f64_sub(hl, f64_div(hr, rate));
            } else {
                tot = f64_add(tot, f64_mul(d, m));
                hl = f64_sub(hl, f64_div(m, rate));
            }
        }
        mraw[(size_t)si * S + s] = tot;
    }
    KSPAN_END(2);
}

// The variant period's mining-cost sum (numpy pairwise over its blocks in block order, the base
// list with b removed / inserted) and block count, one CTA per re-solved slot (persistent).
__global__ void __launch_bounds__(256) k_s2_varcost(const S2Struct rec, int T, int M, const int32_t *__restrict__ blocks,
                                                    const int32_t *__restrict__ slot_t, const int32_t *__restrict__ run,
                                                    const double *__restrict__ cost, double *__restrict__ mcost,
                                                    int32_t *__restrict__ mn, int cap,
                                                    const unsigned long long *__restrict__ cflag, unsigned long long eh,
                                                    int pend0, int pend1, unsigned long long *__restrict__ vc_done) {
    asm volatile("griddepcontrol.launch_dependents;");  // the chains may start (they wait on their own flags)
    KSPAN_BEGIN(1);
    // the pairwise plan's leaves (<= n/64 + 2) live in shared memory: cap of each array
    extern __shared__ __align__(16) unsigned char vc_dyn[];
    double *lv = reinterpret_cast<double *>(vc_dyn);
    int *ls = reinterpret_cast<int *>(lv + cap);
    int *ll = ls + cap;
    for (int si = blockIdx.x; si < 2 * M; si += gridDim.x) {
        const int t = slot_t[si];
        if (t < 0 || run[si] < 0) continue;
        const int b = blocks[si >> 1];
        const int y = t == pend0 ? 0 : (t == pend1 ? 1 : -1);
        if (y >= 0) {  // the concurrent base update splices this period's list first
            if (threadIdx.x == 0) s2_flag_wait(cflag + y, eh | 1ull);
            __syncthreads();
        }
        const int32_t *ids = rec.IDS + (size_t)t * rec.L;
        const double *csl = rec.CS + (size_t)t * rec.L;
        const double cb = __ldg(cost + (size_t)b * T + t);
        const int n0 = __ldcg(rec.nper + t);
        PP_DCHECK(n0 >= 0 && n0 < rec.L && (n0 + 1) / 64 + 2 <= cap);
        int lo = 0, hi = n0;  // block-order position of b
        while (lo < hi) {
            const int md = (lo + hi) >> 1;
            if (__ldcg(ids + md) < b) lo = md + 1;
            else hi = md;
        }
        const int r = lo;
        const bool ins = si & 1;
        PP_DCHECK(ins || (r < n0 && ids[r] == b));  // a removed block is in its period's list
        const int n = ins ? n0 + 1 : n0 - 1;
        const double cs = s2_pairwise_f(
            [&](int k) {
                return ins ? (k < r ? __ldcg(csl + k) : (k == r ? cb : __ldcg(csl + k - 1))) : __ldcg(csl + (k < r ? k : k + 1));
            },
            n, ls, ll, lv);
        if (threadIdx.x == 0) {
            mcost[si] = cs;
            mn[si] = n;
        }
        __syncthreads();
    }
    KSPAN_END(1);
    if (vc_done && threadIdx.x == 0) {  // this CTA's cost sums are written (the accumulation counts them)
        __threadfence();
        atomicAdd(vc_done, 1ull);
    }
}

// _npv / per_scenario_npv accumulation in the reference's order (t outer, s inner)
__global__ void k_npv_final(int T, int S, const double *__restrict__ raw, const double *__restrict__ costsum,
                            const int32_t *__restrict__ nmined, const double *__restrict__ disc,
                            const double *__restrict__ sigma, double *__restrict__ npv, double *__restrict__ per_scen) {
    const int p = blockIdx.x;
    if (threadIdx.x != 0) return;
    double total = 0.0;
    double *ps = per_scen ? per_scen + (size_t)p * S : nullptr;
    if (ps)
        for (int s = 0; s < S; s++) ps[s] = 0.0;
    for (int t = 0; t < T; t++) {
        const size_t pt = (size_t)p * T + t;
        const double d = disc[t];
        double cv = 0.0;
        if (nmined[pt] > 0) {
            const double cs = costsum[pt];
            total = f64_sub(total, f64_mul(d, cs));
            cv = f64_mul(d, cs);
        }
        for (int s = 0; s < S; s++) {
            const double sg = sigma ? sigma[(size_t)s * T + t] : 1.0;
            const double r = raw[pt * S + s];
            const double term = f64_mul(f64_mul(d, sg), r);
            total = f64_add(total, f64_div(term, (double)S));
            if (ps) ps[s] = f64_add(ps[s], f64_sub(term, cv));
        }
    }
    npv[p] = total;
}

// npv of variant m: the reference's accumulation over (t, s), the two changed periods from the
// variant's stage-2 results, every other period from the base schedule's.  One warp per variant:
// lane s forms the scenario terms (d * sigma * raw) / S in parallel (the divisions dominate) into
// shared memory, lane 0 adds them in the reference's (t, s) order.
__global__ void k_npv_moves_final(int T, int S, int M, const double *__restrict__ braw, const double *__restrict__ bcost,
                                  const int32_t *__restrict__ bn, const double *__restrict__ mraw,
                                  const double *__restrict__ mcost, const int32_t *__restrict__ mn,
                                  const int32_t *__restrict__ slot_t, const int32_t *__restrict__ slot_src,
                                  const double *__restrict__ disc,
                                  const double *__restrict__ sigma, double *__restrict__ npv,
                                  const unsigned long long *__restrict__ pflags, unsigned long long eh,
                                  unsigned long long vc_need) {
    if (eh) {  // as k_npv_moves_final_staged
        asm volatile("griddepcontrol.wait;" ::: "memory");
        for (int i = threadIdx.x; i < 2 * S + 2; i += blockDim.x)
            s2_flag_wait(pflags + i, i < 2 * S ? (eh | S2_DONE) : (eh | 1ull));
        if (threadIdx.x == 0) s2_flag_wait(pflags + 2 * S + 2, vc_need);
        __syncthreads();
    }
    const int lane = threadIdx.x & 31;
    const int m = (int)(((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (m >= M) return;
    const int t0 = slot_t[2 * m], t1 = slot_t[2 * m + 1];
    __shared__ double s_q[8][32];
    double *wq = s_q[(threadIdx.x >> 5) & 7];
    double total = 0.0;
    for (int t = 0; t < T; t++) {
        const double *raw;
        double cs;
        int n;
        if (t == t0 || t == t1) {
            const int k = slot_src[2 * m + (t == t0 ? 0 : 1)];  // deduplicated re-solve
            raw = mraw + (size_t)k * S;
            cs = __ldcg(mcost + k);
            n = __ldcg(mn + k);
        } else {
            raw = braw + (size_t)t * S;
            cs = __ldcg(bcost + t);
            n = __ldcg(bn + t);
        }
        const double d = disc[t];
        if (n > 0) total = f64_sub(total, f64_mul(d, cs));
        for (int s0 = 0; s0 < S; s0 += 32) {
            const int s = s0 + lane;
            if (s < S) {
                const double sg = sigma ? sigma[(size_t)s * T + t] : 1.0;
                wq[lane] = f64_div(f64_mul(f64_mul(d, sg), __ldcg(raw + s)), (double)S);
            }
            __syncwarp();
            const int cnt = min(32, S - s0);
            if (lane == 0)  // the adds in the reference's order; the terms are broadcast reads
                for (int u = 0; u < cnt; u++) total = f64_add(total, wq[u]);
            __syncwarp();
        }
    }
    if (lane == 0) npv[m] = total;
}

// The same accumulation with every term of the variant formed up front: the warp's lanes form
// all T*S terms (their loads and divisions independent of one another, so in flight together)
// into the warp's shared slice, then lane 0 adds them in the reference's (t, s) order -- one
// dependent add chain instead of T rounds of load latency.  For T*S <= NPVF_MAX.
constexpr int NPVF_MAX = 480;
constexpr int NPVF_WARPS = 4;
__global__ void __launch_bounds__(32 * NPVF_WARPS)
    k_npv_moves_final_staged(int T, int S, int M, const double *__restrict__ braw, const double *__restrict__ bcost,
                             const int32_t *__restrict__ bn, const double *__restrict__ mraw,
                             const double *__restrict__ mcost, const int32_t *__restrict__ mn,
                             const int32_t *__restrict__ slot_t, const int32_t *__restrict__ slot_src,
                             const double *__restrict__ disc, const double *__restrict__ sigma,
                             double *__restrict__ npv, const unsigned long long *__restrict__ pflags,
                             unsigned long long eh, unsigned long long vc_need) {
    // eh != 0: launched as a programmatic dependent of the chains, while the one-block base update
    // and the cost sums may still be finishing: the chains' results after griddepcontrol.wait,
    // the base values after every period's flag says done, the cost sums after all their CTAs
    KSPAN_BEGIN(3);
    if (eh) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        for (int i = threadIdx.x; i < 2 * S + 2; i += blockDim.x)
            s2_flag_wait(pflags + i, i < 2 * S ? (eh | S2_DONE) : (eh | 1ull));
        if (threadIdx.x == 0) s2_flag_wait(pflags + 2 * S + 2, vc_need);
        __syncthreads();
    }
    __shared__ double s_term[NPVF_WARPS][NPVF_MAX];
    __shared__ double s_cost[NPVF_WARPS][32];  // d * cs per period, or +inf: no mined block (skip)
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int m = (int)blockIdx.x * NPVF_WARPS + w;
    if (m >= M) return;
    const int t0 = slot_t[2 * m], t1 = slot_t[2 * m + 1];
    const int k0 = slot_src[2 * m], k1 = slot_src[2 * m + 1];
    double *tw = s_term[w];
    for (int i = lane; i < T * S; i += 32) {
        const int t = i / S, s = i - t * S;
        const double *raw = t == t0 ? mraw + (size_t)k0 * S : t == t1 ? mraw + (size_t)k1 * S : braw + (size_t)t * S;
        const double d = disc[t];
        const double sg = sigma ? sigma[(size_t)s * T + t] : 1.0;
        tw[i] = f64_div(f64_mul(f64_mul(d, sg), __ldcg(raw + s)), (double)S);
    }
    if (lane < T) {
        const int t = lane;
        const double cs = t == t0 ? __ldcg(mcost + k0) : t == t1 ? __ldcg(mcost + k1) : __ldcg(bcost + t);
        const int n = t == t0 ? __ldcg(mn + k0) : t == t1 ? __ldcg(mn + k1) : __ldcg(bn + t);
        s_cost[w][t] = n > 0 ? f64_mul(disc[t], cs) : kInf;
    }
    __syncwarp();
    if (lane == 0) {
        double total = 0.0;
        for (int t = 0; t < T; t++) {
            const double dc = s_cost[w][t];
            if (dc != kInf) total = f64_sub(total, dc);
            for (int s = 0; s < S; s++) total = f64_add(total, tw[t * S + s]);
        }
        npv[m] = total;
        KSPAN_END(3);
    }
}

extern "C" {

int pp_set_plant(pp_ctx *c, const double *plant_hours, double rate) {
    if (!c || !c->have_instance) return fail(PP_ERR_STATE, "pp_set_instance first");
    if (!plant_hours) return fail(PP_ERR_INVALID_ARGS, "plant_hours is NULL");
    if (!(rate > 0)) return fail(PP_ERR_INVALID_ARGS, "the stage-2 fast path needs a positive rate");
    TRY(use_device(c));
    TRY(c->hours.ensure(sizeof(double) * c->T));
    CUDA_TRY(dev_upload(c, c->hours.ptr, plant_hours, sizeof(double) * c->T));
    c->rate = rate;
    c->have_plant = true;
    c->npv_gen++;
    return PP_OK;
}

int pp_npv_relaxed(pp_ctx *c, const int32_t *assign, int32_t P, uint32_t flags, double *npv_out, double *per_scen_out,
                   int32_t mem, void *stream) {
    if (!c || !c->have_instance || !c->have_scen || !c->have_plant)
        return fail(PP_ERR_STATE, "pp_set_instance, pp_set_scenarios and pp_set_plant first");
    if (P < 0 || (P > 0 && (!assign || !npv_out))) return fail(PP_ERR_INVALID_ARGS, "bad arguments");
    if ((flags & PP_USE_SIGMA) && !c->have_sigma) return fail(PP_ERR_STATE, "PP_USE_SIGMA without an uploaded sigma");
    if (P == 0) return PP_OK;
    TRY(use_device(c));
    cudaStream_t st = pick(c, stream);
    const int B = c->B, T = c->T, S = c->S;
    const int32_t *da = assign;
    double *dn = npv_out, *dps = per_scen_out;
    if (mem == PP_MEM_HOST) {
        TRY(c->h_assign.ensure(sizeof(int32_t) * (size_t)P * B));
        TRY(c->h_d1.ensure(sizeof(double) * P));
        CUDA_TRY(cudaMemcpyAsync(c->h_assign.ptr, assign, sizeof(int32_t) * (size_t)P * B, cudaMemcpyHostToDevice, st));
        da = c->h_assign.as<int32_t>();
        dn = c->h_d1.as<double>();
        if (per_scen_out) {
            TRY(c->h_pm.ensure(sizeof(double) * (size_t)P * S));
            dps = c->h_pm.as<double>();
        }
    }
    TRY(c->npv_raw.ensure(sizeof(double) * (size_t)P * T * S));
    c->npv_gen++;  // overwrites pp_npv_moves' cached base results
    TRY(c->npv_cost.ensure(sizeof(double) * (size_t)P * T));
    TRY(c->npv_n.ensure(sizeof(int32_t) * (size_t)P * T));
    TRY(run_stage2(c, st, da, T, P, c->npv_raw.as<double>(), c->npv_cost.as<double>(), c->npv_n.as<int32_t>(),
                   nullptr, nullptr, nullptr));
    k_npv_final<<<P, 32, 0, st>>>(T, S, c->npv_raw.as<double>(), c->npv_cost.as<double>(), c->npv_n.as<int32_t>(),
                                  c->disc.as<double>(), (flags & PP_USE_SIGMA) ? c->sigma.as<double>() : nullptr, dn,
                                  dps);
    CUDA_TRY(cudaGetLastError());
    if (mem == PP_MEM_HOST) {
        CUDA_TRY(cudaMemcpyAsync(npv_out, dn, sizeof(double) * P, cudaMemcpyDeviceToHost, st));
        if (per_scen_out)
            CUDA_TRY(cudaMemcpyAsync(per_scen_out, dps, sizeof(double) * (size_t)P * S, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(stream_wait(st));
    }
    return PP_OK;
}

int pp_stage2(pp_ctx *c, const int32_t *assign, int32_t P, double *raw_out, double *cost_out, int32_t mem,
              void *stream) {
    if (!c || !c->have_instance || !c->have_scen || !c->have_plant)
        return fail(PP_ERR_STATE, "pp_set_instance, pp_set_scenarios and pp_set_plant first");
    if (P < 0 || (P > 0 && (!assign || !raw_out))) return fail(PP_ERR_INVALID_ARGS, "bad arguments");
    if (P == 0) return PP_OK;
    TRY(use_device(c));
    cudaStream_t st = pick(c, stream);
    const int B = c->B, T = c->T, S = c->S;
    const int32_t *da = assign;
    if (mem == PP_MEM_HOST) {
        TRY(c->h_assign.ensure(sizeof(int32_t) * (size_t)P * B));
        CUDA_TRY(cudaMemcpyAsync(c->h_assign.ptr, assign, sizeof(int32_t) * (size_t)P * B, cudaMemcpyHostToDevice, st));
        da = c->h_assign.as<int32_t>();
    }
    TRY(c->npv_raw.ensure(sizeof(double) * (size_t)P * T * S));
    c->npv_gen++;  // overwrites pp_npv_moves' cached base results
    TRY(c->npv_cost.ensure(sizeof(double) * (size_t)P * T));
    TRY(c->npv_n.ensure(sizeof(int32_t) * (size_t)P * T));
    TRY(run_stage2(c, st, da, T, P, c->npv_raw.as<double>(), c->npv_cost.as<double>(), c->npv_n.as<int32_t>(),
                   nullptr, nullptr, nullptr));
    // periods with no mined block have no costsum written: zero them in the copy (cost 0.0)
    const cudaMemcpyKind k = mem == PP_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    CUDA_TRY(cudaMemcpyAsync(raw_out, c->npv_raw.ptr, sizeof(double) * (size_t)P * T * S, k, st));
    if (cost_out) {
        if (mem == PP_MEM_HOST) {
            std::vector<double> cs((size_t)P * T);
            std::vector<int32_t> nm((size_t)P * T);
            CUDA_TRY(cudaMemcpyAsync(cs.data(), c->npv_cost.ptr, sizeof(double) * cs.size(), k, st));
            CUDA_TRY(cudaMemcpyAsync(nm.data(), c->npv_n.ptr, sizeof(int32_t) * nm.size(), k, st));
            CUDA_TRY(stream_wait(st));
            for (size_t i = 0; i < cs.size(); i++) cost_out[i] = nm[i] > 0 ? cs[i] : 0.0;
            return PP_OK;
        }
        CUDA_TRY(cudaMemcpyAsync(cost_out, c->npv_cost.ptr, sizeof(double) * (size_t)P * T, k, st));
    }
    if (mem == PP_MEM_HOST) CUDA_TRY(stream_wait(st));
    return PP_OK;
}

__global__ void k_scatter_assign(int32_t *__restrict__ assign, const int32_t *__restrict__ blk,
                                 const int32_t *__restrict__ per, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) assign[blk[i]] = per[i];  // distinct blocks (a diff)
}


// ------------------------------------------------------------------------------------
// Incremental base update when the base schedule changed by ONE block b: t_old -> t_new (the
// polish pattern: every accepted move ends a call).  Instead of re-solving the two periods from
// scratch (compaction, sort, greedy), the recorded structure is spliced: grid (S, 2), y = 0 takes b
// out of (s, t_old), y = 1 puts it into (s, t_new) at its binary-searched place; the arrays after
// the place shift by one in 1024-element chunks (ascending for a removal, descending for an
// insertion, so no chunk overwrites what a later one reads), the positions of the shifted blocks
// are renumbered, and the greedy resumes from the recorded state at the place (the prefix before it
// is unchanged) with recording.  One extra CTA per period (blockIdx.x == S) splices the
// block-ordered id and cost lists the same way and recomputes the period's mining-cost sum (numpy
// pairwise) beside the greedy CTAs.  Identical to a rebuild.  The call's variant kernels run
// concurrently as programmatic dependents and wait only on the progress flags they need.
// ------------------------------------------------------------------------------------
__device__ void s2_apply_cost(const S2Struct &rec, int T, int b, int t, bool ins, const double *__restrict__ cost,
                              double *__restrict__ costsum, int32_t *__restrict__ nmined,
                              unsigned long long *__restrict__ cflag, unsigned long long eh) {
    __shared__ int s_j, s_ls[256], s_ll[256];
    __shared__ double s_lv[256];
    const int tid = threadIdx.x;
    int32_t *ids = rec.IDS + (size_t)t * rec.L;
    double *csl = rec.CS + (size_t)t * rec.L;
    const int n0 = rec.nper[t];
    if (tid == 0) {
        int lo = 0, hi = n0;
        while (lo < hi) {
            const int md = (lo + hi) >> 1;
            if (ids[md] < b) lo = md + 1;
            else hi = md;
        }
        s_j = lo;
    }
    __syncthreads();
    const int r = s_j;
    PP_DCHECK(n0 >= 0 && n0 + 1 < 16000 && (ins || (r < n0 && ids[r] == b)));
    if (!ins) {
        for (int k0 = r; k0 < n0 - 1; k0 += S2_THREADS) {
            const int k = k0 + tid;
            int bb = 0;
            double cc = 0.0;
            if (k < n0 - 1) {
                bb = ids[k + 1];
                cc = csl[k + 1];
            }
            __syncthreads();
            if (k < n0 - 1) {
                ids[k] = bb;
                csl[k] = cc;
            }
            __syncthreads();
        }
    } else {
        for (int k1 = n0; k1 > r; k1 -= S2_THREADS) {
            const int k = k1 - 1 - tid;
            int bb = 0;
            double cc = 0.0;
            if (k >= r) {
                bb = ids[k];
                cc = csl[k];
            }
            __syncthreads();
            if (k >= r) {
                ids[k + 1] = bb;
                csl[k + 1] = cc;
            }
            __syncthreads();
        }
        if (tid == 0) {
            ids[r] = b;
            csl[r] = __ldg(cost + (size_t)b * T + t);
        }
    }
    __syncthreads();
    const int n1 = ins ? n0 + 1 : n0 - 1;
    const double cs = s2_pairwise(csl, n1, s_ls, s_ll, s_lv);  // n1 < 16000: <= 252 leaves
    if (tid == 0) {
        rec.nper[t] = n1;
        costsum[t] = cs;
        nmined[t] = n1;
        s2_flag_publish(cflag + blockIdx.y, eh | 1ull);  // the block-ordered list is spliced
    }
}

__global__ void __launch_bounds__(S2_THREADS, 1)
    k_s2_apply_one(const S2Struct rec, int B, int T, int S, int Sp, int b, int t_old, int t_new,
                   const double *__restrict__ mass, const double *__restrict__ cost, const double *__restrict__ vmax,
                   const double *__restrict__ hours, double rate, double *__restrict__ raw,
                   double *__restrict__ costsum, int32_t *__restrict__ nmined, unsigned long long *__restrict__ prog,
                   unsigned long long *__restrict__ cflag, unsigned long long eh, int32_t *__restrict__ dbase) {
    // prog[y][s] / cflag[y] (y = blockIdx.y): progress of this update for the variants' kernels of
    // the same call, which run concurrently (programmatic dependents, launched once every CTA here
    // has started)
    asm volatile("griddepcontrol.launch_dependents;");
    KSPAN_BEGIN(0);
    __shared__ int s_j;
    const int s = blockIdx.x;
    const bool ins = blockIdx.y == 1;
    const int t = ins ? t_new : t_old;
    if (s == 0 && blockIdx.y == 0 && threadIdx.x == 0) dbase[b] = t_new;  // the device copy of the base
    if (s == S) {  // the cost CTA
        if (t < 0) {
            if (threadIdx.x == 0) s2_flag_publish(cflag + blockIdx.y, eh | 1ull);
        } else {
            s2_apply_cost(rec, T, b, t, ins, cost, costsum, nmined, cflag, eh);
        }
        return;
    }
    unsigned long long *pf = prog + (size_t)blockIdx.y * S + s;
    if (t < 0) {  // no such period (the block was / becomes unmined): nothing to update
        if (threadIdx.x == 0) s2_flag_publish(pf, eh | S2_DONE);
        return;
    }
    const int tid = threadIdx.x;
    const size_t st_ = (size_t)s * T + t, base = st_ * rec.L;
    double *D = rec.D + base, *M_ = rec.M + base, *H = rec.H + base, *TT = rec.TT + base;
    int32_t *BI = rec.BID + base;
    const int np = rec.npos[st_];
    PP_DCHECK(np >= 0 && np + 1 < rec.L);
    const double mb = __ldg(mass + b);
    const double db = f64_div(__ldg(vmax + (size_t)b * Sp + s), mb);
    // 1. the place of b in the greedy order
    if (tid == 0) {
        int j;
        if (!ins) {
            j = rec.pos[(size_t)s * B + b];  // -1: not in the list (density <= 0)
        } else if (!(db > 0)) {
            j = -1;
            rec.pos[(size_t)s * B + b] = -1;
        } else {
            int lo = 0, hi = np;
            while (lo < hi) {
                const int md = (lo + hi) >> 1;
                if (D[md] > db || (D[md] == db && BI[md] < b)) lo = md + 1;
                else hi = md;
            }
            j = lo;
        }
        PP_DCHECK(ins || j < 0 || (j < np && BI[j] == b));
        s_j = j;
    }
    __syncthreads();
    const int j = s_j;
    const int K = rec.K[st_];
    PP_DCHECK(K >= 0 && K <= np);
    if (j >= 0) {
        // 2. splice the order (D, M, BID) and renumber the shifted blocks' positions
        if (!ins) {
            for (int k0 = j; k0 < np - 1; k0 += S2_THREADS) {
                const int k = k0 + tid;
                double dd = 0.0, mm = 0.0;
                int bb = 0;
                if (k < np - 1) {
                    dd = D[k + 1];
                    mm = M_[k + 1];
                    bb = BI[k + 1];
                }
                __syncthreads();
                if (k < np - 1) {
                    D[k] = dd;
                    M_[k] = mm;
                    BI[k] = bb;
                    rec.pos[(size_t)s * B + bb] = k;
                }
                __syncthreads();
            }
        } else {
            for (int k1 = np; k1 > j; k1 -= S2_THREADS) {
                const int k = k1 - 1 - tid;  // old position, moves to k + 1
                double dd = 0.0, mm = 0.0;
                int bb = 0;
                if (k >= j) {
                    dd = D[k];
                    mm = M_[k];
                    bb = BI[k];
                }
                __syncthreads();
                if (k >= j) {
                    D[k + 1] = dd;
                    M_[k + 1] = mm;
                    BI[k + 1] = bb;
                    rec.pos[(size_t)s * B + bb] = k + 1;
                }
                __syncthreads();
            }
            if (tid == 0) {
                D[j] = db;
                M_[j] = mb;
                BI[j] = b;
                rec.pos[(size_t)s * B + b] = j;
            }
        }
        const int npn = ins ? np + 1 : np - 1;
        if (tid == 0) rec.npos[st_] = npn;
        __syncthreads();
        if (tid == 0) s2_flag_publish(pf, eh | (unsigned long long)(j + 3));  // spliced; states <= j final
        // 3. the greedy from the place on, from the recorded state there (unchanged prefix); a place
        //    beyond the stop changes nothing the greedy reaches
        if (j <= K && tid < 32) {
            const double total = s2_greedy_warp(
                npn, npn, H[j], rate, [&](int k) { return D[k]; }, [&](int k) { return M_[k]; },
                [&](int k) { return f64_div(M_[k], rate); }, H, TT, rec.K + st_, j, TT[j], pf, eh);
            if (tid == 0) raw[(size_t)t * S + s] = total;
        }
    }
    if (tid < 32) {  // the period's structure, stop and value are final
        __syncwarp();
        if (tid == 0) s2_flag_publish(pf, eh | S2_DONE);
        KSPAN_END(0);
    }
}

// carve the base structure (S2Struct) out of c->s2_rec for the current (S, T, B)
static int s2_struct(pp_ctx *c, S2Struct *r) {
    const size_t S = c->S, T = c->T, B = c->B, L = B + 1;
    const size_t nd = S * T * L;
    const size_t bytes = 4 * nd * sizeof(double) + T * L * sizeof(double) + nd * sizeof(int32_t) + 2 * S * T * sizeof(int32_t) +
                         S * B * sizeof(int32_t) + T * L * sizeof(int32_t) + T * sizeof(int32_t) + 256;
    TRY(c->s2_rec.ensure(bytes));
    unsigned char *p = c->s2_rec.as<unsigned char>();
    auto take = [&](size_t n) {
        unsigned char *q = p;
        p += (n + 15) & ~(size_t)15;
        return q;
    };
    r->D = reinterpret_cast<double *>(take(nd * 8));
    r->M = reinterpret_cast<double *>(take(nd * 8));
    r->H = reinterpret_cast<double *>(take(nd * 8));
    r->TT = reinterpret_cast<double *>(take(nd * 8));
    r->CS = reinterpret_cast<double *>(take(T * L * 8));
    r->BID = reinterpret_cast<int32_t *>(take(nd * 4));
    r->npos = reinterpret_cast<int32_t *>(take(S * T * 4));
    r->K = reinterpret_cast<int32_t *>(take(S * T * 4));
    r->pos = reinterpret_cast<int32_t *>(take(S * B * 4));
    r->IDS = reinterpret_cast<int32_t *>(take(T * L * 4));
    r->nper = reinterpret_cast<int32_t *>(take(T * 4));
    r->L = (int)L;
    return PP_OK;
}

}  // extern "C"

// hint (may be null): the only blocks that can differ from the cached base (pp_polish_sweep knows
// them: the block it accepted since its previous evaluation), instead of the memcmp diff
static int npv_moves_impl(pp_ctx *c, const int32_t *assign, const int32_t *blocks, const int32_t *periods, int32_t M,
                          uint32_t flags, double *npv_out, int32_t mem, void *stream,
                          const std::vector<int32_t> *hint = nullptr) {
    if (!c || !c->have_instance || !c->have_scen || !c->have_plant)
        return fail(PP_ERR_STATE, "pp_set_instance, pp_set_scenarios and pp_set_plant first");
    if (!assign || M < 0 || (M > 0 && (!blocks || !periods || !npv_out))) return fail(PP_ERR_INVALID_ARGS, "bad arguments");
    if ((flags & PP_USE_SIGMA) && !c->have_sigma) return fail(PP_ERR_STATE, "PP_USE_SIGMA without an uploaded sigma");
    if (M == 0) return PP_OK;
    HostTrace ht_("pp_npv_moves");
    TRY(use_device(c));
    cudaStream_t st = pick(c, stream);
    const int B = c->B, T = c->T, S = c->S;
    // which periods each variant changes (host arrays needed: the base assignment of the block)
    std::vector<int32_t> hb(M), ht(M), hdev;
    const bool host = mem == PP_MEM_HOST;
    const int32_t *ha = assign;
    if (host) {
        std::copy(blocks, blocks + M, hb.begin());
        std::copy(periods, periods + M, ht.begin());
    } else {
        hdev.resize(B);
        CUDA_TRY(cudaMemcpyAsync(hb.data(), blocks, sizeof(int32_t) * M, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(ht.data(), periods, sizeof(int32_t) * M, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(hdev.data(), assign, sizeof(int32_t) * B, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(stream_wait(st));
        ha = hdev.data();
    }
    // slot[2m] = the period the move leaves, slot[2m+1] = the period it enters (-1 = none).
    // The re-solve of the left period (block removed) depends only on the block, so the moves of
    // one block share it: run[] = the periods actually re-solved (-1 for a duplicate), src[] = the
    // slot whose results a move reads.
    std::vector<int32_t> slot((size_t)2 * M), run((size_t)2 * M), src((size_t)2 * M);
    std::unordered_map<int32_t, int32_t> left_of;
    for (int m = 0; m < M; m++) {
        if (hb[m] < 0 || hb[m] >= B || ht[m] < -1 || ht[m] >= T) return fail(PP_ERR_INVALID_ARGS, "move %d out of range", m);
        const int told = ha[hb[m]], tnew = ht[m];
        slot[2 * m] = (told >= 0 && told < T && told != tnew) ? told : -1;
        slot[2 * m + 1] = (tnew >= 0 && tnew != told) ? tnew : -1;
        run[2 * m] = slot[2 * m];
        run[2 * m + 1] = slot[2 * m + 1];
        src[2 * m] = 2 * m;
        src[2 * m + 1] = 2 * m + 1;
        if (slot[2 * m] >= 0) {
            auto it = left_of.emplace(hb[m], 2 * m);
            if (!it.second) {
                src[2 * m] = it.first->second;
                run[2 * m] = -1;
            }
        }
    }
    // the base schedule's structure: reused when the tables (npv_gen), the result buffers (their
    // allocation generation: a re-allocation may return the same address) and the structure are
    // intact; then only the periods whose block sets changed since the cached base are re-solved
    int Mcap = 1024;
    while (Mcap < M) Mcap <<= 1;
    TRY(c->npv_raw.ensure(sizeof(double) * ((size_t)T * S + (size_t)2 * Mcap * S)));
    TRY(c->npv_cost.ensure(sizeof(double) * ((size_t)T + 2 * (size_t)Mcap)));
    TRY(c->npv_n.ensure(sizeof(int32_t) * ((size_t)T + 2 * (size_t)Mcap)));
    const uint64_t recgen = c->s2_rec.gen;
    S2Struct rec;
    TRY(s2_struct(c, &rec));
    const bool intact = c->npvm_gen == c->npv_gen && c->npvm_bufgen[0] == c->npv_raw.gen &&
                        c->npvm_bufgen[1] == c->npv_cost.gen && c->npvm_bufgen[2] == c->npv_n.gen &&
                        c->s2_rec.gen == recgen && c->npvm_base.size() == (size_t)B;
    // the blocks that changed since the cached base (their old and new periods are the ones to
    // re-solve): equal 64-block runs are skipped with memcmp, so a base that drifted by a few blocks
    // costs a few microseconds; period sizes (whether the large-period kernel can be needed) are kept
    // in step with the diff, and the range check covers every entry the device has not seen
    std::vector<int32_t> dirty, chg_b, chg_t;
    std::vector<int32_t> &cnt = c->npvm_cnt;
    bool full = !intact;
    if (!full && hint) {
        std::vector<char> mark(T, 0);
        const int32_t *old = c->npvm_base.data();
        for (const int32_t b : *hint) {
            const int32_t o = old[b], n = ha[b];
            if (o == n) continue;
            if (n < -1 || n >= T) return fail(PP_ERR_INVALID_ARGS, "assign[%d] = %d out of range", b, n);
            if (o >= 0) mark[o] = 1;
            if (n >= 0) mark[n] = 1;
            chg_b.push_back(b);
            chg_t.push_back(n);
        }
        for (int t = 0; t < T; t++)
            if (mark[t]) dirty.push_back(t);
    } else if (!full) {
        std::vector<char> mark(T, 0);
        const int32_t *old = c->npvm_base.data();
        for (int b0 = 0; b0 < B; b0 += 64) {
            const int nb = std::min(64, B - b0);
            if (std::memcmp(old + b0, ha + b0, sizeof(int32_t) * nb) == 0) continue;
            for (int b = b0; b < b0 + nb; b++) {
                const int32_t o = old[b], n = ha[b];
                if (o == n) continue;
                if (n < -1 || n >= T) return fail(PP_ERR_INVALID_ARGS, "assign[%d] = %d out of range", b, n);
                if (o >= 0) mark[o] = 1;
                if (n >= 0) mark[n] = 1;
                chg_b.push_back(b);
                chg_t.push_back(n);
            }
            if (chg_b.size() * 8 > (size_t)B) break;  // a new schedule rather than a drift
        }
        for (int t = 0; t < T; t++)
            if (mark[t]) dirty.push_back(t);
        full = (int)dirty.size() * 2 > T || chg_b.size() * 8 > (size_t)B;
    }
    if (full) {
        cnt.assign(T, 0);
        int32_t lo = 0, hi = -1;  // branch-free range check (vectorises), then the period sizes
        for (int b = 0; b < B; b++) {
            lo = std::min(lo, ha[b]);
            hi = std::max(hi, ha[b]);
        }
        if (lo < -1 || hi >= T) return fail(PP_ERR_INVALID_ARGS, "assign holds a period outside [-1, %d)", T);
        for (int b = 0; b < B; b++)
            if (ha[b] >= 0) cnt[ha[b]]++;
        chg_b.clear();
        chg_t.clear();
        dirty.clear();
    } else {
        const int32_t *old = c->npvm_base.data();
        for (size_t k = 0; k < chg_b.size(); k++) {
            if (old[chg_b[k]] >= 0) cnt[old[chg_b[k]]]--;
            if (chg_t[k] >= 0) cnt[chg_t[k]]++;
        }
    }
    ht_.mark("diff");
    const bool may_be_big = *std::max_element(cnt.begin(), cnt.end()) > S2_NMAX;
    // the device keeps its own copy of the base assignment: a full upload when the structure is
    // rebuilt, else only the changed entries (scattered by k_scatter_assign)
    TRY(c->s2_assign.ensure(sizeof(int32_t) * (size_t)B));
    int32_t *dbase = c->s2_assign.as<int32_t>();
    const size_t nchg = full ? 0 : chg_b.size();
    // one packed upload (blocks | periods | slots | runs | sources | re-solved periods | changed
    // blocks | their periods) and one result copy: each separate small copy costs a PCIe round trip
    const size_t nin = 8 * (size_t)M + T + 2 * nchg;
    TRY(c->h_assign.ensure(sizeof(int32_t) * std::max<size_t>(nin, 1)));
    int32_t *db = c->h_assign.as<int32_t>(), *dt = db + M, *ds = dt + M, *dr = ds + 2 * M,
            *dsrc = dr + 2 * M, *dtsel = dsrc + 2 * M, *dcb = dtsel + T, *dct = dcb + nchg;
    TRY(c->h_d1.ensure(sizeof(double) * ((size_t)M + 1)));
    const size_t out_bytes = sizeof(double) * (size_t)M;
    unsigned char *stage = nullptr;
    TRY(host_stage(c, std::max(sizeof(int32_t) * std::max(nin, (size_t)B), out_bytes), &stage));
    std::vector<int32_t> pkv(host ? 0 : std::max(nin, (size_t)B));  // device mode returns before the
    int32_t *pk = host ? reinterpret_cast<int32_t *>(stage) : pkv.data();  // copy completes: pageable
    if (full) {
        if (host) {
            CUDA_TRY(cudaMemcpyAsync(dbase, assign, sizeof(int32_t) * B, cudaMemcpyHostToDevice, st));
        } else {
            CUDA_TRY(cudaMemcpyAsync(dbase, assign, sizeof(int32_t) * B, cudaMemcpyDeviceToDevice, st));
        }
    }
    std::copy(hb.begin(), hb.end(), pk);
    std::copy(ht.begin(), ht.end(), pk + M);
    std::copy(slot.begin(), slot.end(), pk + 2 * M);
    std::copy(run.begin(), run.end(), pk + 4 * M);
    std::copy(src.begin(), src.end(), pk + 6 * M);
    std::copy(dirty.begin(), dirty.end(), pk + 8 * M);
    if (nchg) {
        std::copy(chg_b.begin(), chg_b.end(), pk + 8 * M + T);
        std::copy(chg_t.begin(), chg_t.end(), pk + 8 * M + T + nchg);
    }
    CUDA_TRY(cudaMemcpyAsync(db, pk, sizeof(int32_t) * nin, cudaMemcpyHostToDevice, st));
    // one moved block: the update kernel splices it (and writes its entry of the device base)
    const bool splice = !full && chg_b.size() == 1 && c->npvm_cnt[dirty[0]] < 16000 &&
                        (dirty.size() < 2 || c->npvm_cnt[dirty[1]] < 16000);
    if (nchg && !splice) {
        k_scatter_assign<<<(unsigned)((nchg + 255) / 256), 256, 0, st>>>(dbase, dcb, dct, (int)nchg);
        CUDA_TRY(cudaGetLastError());
    }
    const int32_t *da = dbase;
    ht_.mark("upload");
#ifdef PP_EVAL_PROBE
    if (host) kspan_reset();
#endif
    // a one-block base update (k_s2_apply_one) runs concurrently with this call's variant kernels,
    // which wait on its progress flags for the two periods it updates (pend0 / pend1)
    int pend0 = -1, pend1 = -1;
    unsigned long long pend_eh = 0;
    double *braw = c->npv_raw.as<double>(), *mraw = braw + (size_t)T * S;
    double *bcost = c->npv_cost.as<double>(), *mcost = bcost + T;
    int32_t *bn = c->npv_n.as<int32_t>(), *mn = bn + T;
    if (full) {
        TRY(run_stage2(c, st, da, T, 1, braw, bcost, bn, nullptr, nullptr, nullptr, nullptr, &rec, may_be_big));
    } else if (splice) {  // one block moved: splice
        const int bb = chg_b[0], to = c->npvm_base[bb], tn = chg_t[0];
        TRY(c->npvm_flags.ensure(sizeof(unsigned long long) * (2 * (size_t)S + 3)));
        if (c->npvm_flags.gen != c->npvm_flags_gen) {  // fresh buffer: epoch 0 everywhere, no CTA counted
            CUDA_TRY(cudaMemsetAsync(c->npvm_flags.ptr, 0, sizeof(unsigned long long) * (2 * (size_t)S + 3), st));
            c->npvm_flags_gen = c->npvm_flags.gen;
            c->npvm_epoch = 0;
            c->npvm_vc = 0;
        }
        pend_eh = (unsigned long long)(++c->npvm_epoch) << 32;
        pend0 = to;
        pend1 = tn;
        k_s2_apply_one<<<dim3(S + 1, 2), S2_THREADS, 0, st>>>(
            rec, B, T, S, c->Sp, bb, to, tn, c->mass.as<double>(), c->cost.as<double>(), c->vmax.as<double>(),
            c->hours.as<double>(), c->rate, braw, bcost, bn, c->npvm_flags.as<unsigned long long>(),
            c->npvm_flags.as<unsigned long long>() + 2 * S, pend_eh, dbase);
        CUDA_TRY(cudaGetLastError());
    } else if (!dirty.empty())
        TRY(run_stage2(c, st, da, (int)dirty.size(), 1, braw, bcost, bn, nullptr, nullptr, nullptr, dtsel, &rec,
                       may_be_big));
    {
        // the cost sums (k_s2_varcost) and the stage-2 chains (k_s2_chain) read disjoint parts of the
        // base structure.  After a one-block update both are programmatic dependents of it on the
        // stream (varcost first, the chains once every varcost CTA has started), overlapping it
        // through its flags; otherwise the cost sums run on the side stream beside the chains
        const int cap = B / 64 + 16;
        const size_t smem = (size_t)16 * cap;
        TRY(ensure_side_stream(c));
        const int grid = std::max(1, std::min(2 * M, 4 * c->n_sms));
        TRY(set_smem_attr(k_s2_varcost, smem, c->device));
        const unsigned long long *pflags = c->npvm_flags.as<unsigned long long>();
        const long long nthr = 2ll * M * S * 32;  // a warp per (slot, scenario)
        const int cgrid = (int)((nthr + 255) / 256);
        if (pend_eh) {
            c->npvm_vc += (unsigned long long)grid;  // the accumulation waits for this many finished CTAs
            TRY(launch_eval_n(k_s2_varcost, grid, 256, smem, st, true, rec, T, M, (const int32_t *)db, (const int32_t *)ds,
                              (const int32_t *)dr, (const double *)c->cost.as<double>(), mcost, mn, cap,
                              pflags + 2 * S, pend_eh, pend0, pend1, c->npvm_flags.as<unsigned long long>() + 2 * S + 2));
            TRY(launch_eval_n(k_s2_chain, cgrid, 256, 0, st, true, rec, B, T, S, c->Sp, M, (const int32_t *)db,
                              (const int32_t *)ds, (const int32_t *)dr, (const double *)c->vmax.as<double>(),
                              (const double *)c->mass.as<double>(), c->rate, (const double *)braw, mraw, pflags,
                              pend_eh, pend0, pend1));
        } else {
            CUDA_TRY(cudaEventRecord(c->ev_fork, st));
            CUDA_TRY(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
            k_s2_varcost<<<grid, 256, smem, c->side>>>(rec, T, M, db, ds, dr, c->cost.as<double>(), mcost, mn, cap,
                                                       pflags, 0ull, -1, -1, nullptr);
            CUDA_TRY(cudaGetLastError());
            CUDA_TRY(cudaEventRecord(c->ev_join, c->side));
            k_s2_chain<<<cgrid, 256, 0, st>>>(rec, B, T, S, c->Sp, M, db, ds, dr, c->vmax.as<double>(),
                                              c->mass.as<double>(), c->rate, braw, mraw, pflags, 0ull, -1, -1);
            CUDA_TRY(cudaGetLastError());
            CUDA_TRY(cudaStreamWaitEvent(st, c->ev_join, 0));
        }
    }
    ht_.mark("launch");
    double *dn = host ? c->h_d1.as<double>() : npv_out;
    {
        const double *sg = (flags & PP_USE_SIGMA) ? c->sigma.as<double>() : nullptr;
        const unsigned long long *pf = c->npvm_flags.as<unsigned long long>();
        const bool pdl = pend_eh != 0;  // a programmatic dependent of the chains (see the kernels)
        if (T * S <= NPVF_MAX && T <= 32)
            TRY(launch_eval_n(k_npv_moves_final_staged, (M + NPVF_WARPS - 1) / NPVF_WARPS, 32 * NPVF_WARPS, 0, st, pdl,
                              T, S, M, (const double *)braw, (const double *)bcost, (const int32_t *)bn,
                              (const double *)mraw, (const double *)mcost, (const int32_t *)mn, (const int32_t *)ds,
                              (const int32_t *)dsrc, (const double *)c->disc.as<double>(), sg, dn, pf, pend_eh,
                              c->npvm_vc));
        else
            TRY(launch_eval_n(k_npv_moves_final, (M + 7) / 8, 256, 0, st, pdl, T, S, M, (const double *)braw,
                              (const double *)bcost, (const int32_t *)bn, (const double *)mraw, (const double *)mcost,
                              (const int32_t *)mn, (const int32_t *)ds, (const int32_t *)dsrc,
                              (const double *)c->disc.as<double>(), sg, dn, pf, pend_eh, c->npvm_vc));
    }
    // the structure now describes `ha` (complete once the stream reaches this point)
    c->npvm_gen = c->npv_gen;
    c->npvm_bufgen[0] = c->npv_raw.gen;
    c->npvm_bufgen[1] = c->npv_cost.gen;
    c->npvm_bufgen[2] = c->npv_n.gen;
    if (full) {
        c->npvm_base.assign(ha, ha + B);
    } else {
        for (size_t k = 0; k < chg_b.size(); k++) c->npvm_base[chg_b[k]] = chg_t[k];
    }
    if (host) {
        CUDA_TRY(cudaMemcpyAsync(stage, dn, out_bytes, cudaMemcpyDeviceToHost, st));
        ht_.mark("final+d2h");
        CUDA_TRY(stream_wait(st));
        ht_.mark("sync");
#ifdef PP_EVAL_PROBE
        kspan_append();
#endif
        std::memcpy(npv_out, stage, sizeof(double) * M);
    }
    return PP_OK;
}


extern "C" {

int pp_npv_moves(pp_ctx *c, const int32_t *assign, const int32_t *blocks, const int32_t *periods, int32_t M,
                 uint32_t flags, double *npv_out, int32_t mem, void *stream) {
    return npv_moves_impl(c, assign, blocks, periods, M, flags, npv_out, mem, stream);
}

// The single-block sweep of polish_schedule (hybrid.py:357-385) as a native driver over speculative
// chunks of blocks: the options of blocks [b0, b1) -- unmine first when no successor is mined, then
// every period of the precedence window (hybrid.py:348-355) other than the current one whose
// capacity admits the block (load[t] + m <= cap[t]) -- valued against the current schedule in one
// incremental pp_npv_moves evaluation; the blocks are then decided in order with the reference's
// rule (the best option strictly above cur + 1e-9), and the first acceptance ends the chunk, so
// every decision is the sequential one.  The chunk halves after an early acceptance and doubles
// otherwise (1 .. chunk_max blocks).
int pp_polish_sweep(pp_ctx *c, int32_t *assign, double *load, double *cur_val, uint32_t flags, int32_t chunk0,
                    int32_t chunk_max, int32_t *improved_out, int64_t *calls_out) {
    if (!c || !c->have_instance || !c->have_scen || !c->have_plant)
        return fail(PP_ERR_STATE, "pp_set_instance, pp_set_scenarios and pp_set_plant first");
    if (!assign || !load || !cur_val || !improved_out) return fail(PP_ERR_INVALID_ARGS, "bad arguments");
    const int B = c->B, T = c->T;
    const int UN = -1;
    const std::vector<int> &st = c->h_start, &np = c->h_npred, &adj = c->h_adj;
    const std::vector<double> &mass = c->h_mass, &cap = c->h_cap;
    int k = std::max(1, chunk0);
    const int kmax = std::max(1, chunk_max);
    std::vector<int32_t> ob, ot;   // the chunk's options (block, period)
    std::vector<int32_t> first;    // per chunk block: index of its first option, then one past the last
    std::vector<double> vals;
    std::vector<int32_t> moved;  // blocks accepted since the previous evaluation (its diff)
    int improved = 0;
    int64_t calls = 0;
    double cv = *cur_val;
    int b0 = 0;
    while (b0 < B) {
        const int b1 = std::min(B, b0 + k);
        ob.clear();
        ot.clear();
        first.assign((size_t)(b1 - b0) + 1, 0);
        for (int b = b0; b < b1; b++) {
            first[b - b0] = (int)ob.size();
            const int orig = assign[b];
            bool pred_un = false;
            int t_lo = 0;
            for (int q = st[b]; q < st[b] + np[b]; q++) {
                const int tp = assign[adj[q]];
                if (tp == UN) {
                    pred_un = true;
                    break;
                }
                t_lo = std::max(t_lo, tp);
            }
            bool succ_mined = false;
            int t_hi = T - 1;
            for (int q = st[b] + np[b]; q < st[b + 1]; q++) {
                const int tc = assign[adj[q]];
                if (tc != UN) {
                    t_hi = succ_mined ? std::min(t_hi, tc) : tc;
                    succ_mined = true;
                }
            }
            if (!succ_mined && orig != UN) {
                ob.push_back(b);
                ot.push_back(UN);
            }
            if (!pred_un)
                for (int t = t_lo; t <= t_hi; t++)
                    if (t != orig && load[t] + mass[b] <= cap[t]) {
                        ob.push_back(b);
                        ot.push_back(t);
                    }
        }
        first[b1 - b0] = (int)ob.size();
        int nxt = b1;
        if (!ob.empty()) {
            vals.resize(ob.size());
            TRY(npv_moves_impl(c, assign, ob.data(), ot.data(), (int32_t)ob.size(), flags, vals.data(), PP_MEM_HOST,
                               nullptr, calls ? &moved : nullptr));
            moved.clear();
            calls++;
            for (int b = b0; b < b1; b++) {
                const int lo = first[b - b0], hi = first[b - b0 + 1];
                if (lo == hi) continue;
                const int orig = assign[b];
                int best_t = orig;
                double best_val = cv;
                for (int q = lo; q < hi; q++)
                    if (vals[q] > best_val + 1e-9) {
                        best_t = ot[q];
                        best_val = vals[q];
                    }
                if (best_t != orig) {
                    moved.push_back(b);  // the next evaluation's base differs from this one's in b only
                    assign[b] = best_t;
                    improved = 1;
                    cv = best_val;
                    if (orig != UN) load[orig] -= mass[b];
                    if (best_t != UN) load[best_t] += mass[b];
                    nxt = b + 1;
                    break;
                }
            }
        }
        k = nxt < b1 ? std::max(1, k / 2) : std::min(kmax, k * 2);
        b0 = nxt;
    }
    *cur_val = cv;
    *improved_out = improved;
    if (calls_out) *calls_out = calls;
    return PP_OK;
}

}  // extern "C"
