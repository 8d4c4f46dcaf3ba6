// pp_lns.cu -- lns_repair's insertion loop (hybrid.py:238-266) as one device-resident CUDA graph.
//
// The reference loop, per round: rank the unassigned pool by scheduled-neighbour similarity
// (_scheduled_neighbor_similarity, hybrid.py:142-156) and take the first candidate_width blocks in
// (similarity desc, block asc) order; evaluate them (evaluate_candidates_parallel); stop when no
// move exists (stalled) or, with only_positive, when the best improvement is <= 0; otherwise apply
// the best move -- or, when the best block's geological consistency is below the realism
// threshold, the feasible candidate first in (consistency desc, block asc) order -- and drop the
// block from the pool.  Every round depends on the previous one's schedule, so the rounds are
// sequential; here they run as a conditional WHILE node of a CUDA graph whose body is
//   k_lns_rank (one CTA: similarities, candidate_width rounds of CTA argmax)
//   -> k_pm_cluster -> k_eval_warp -> k_realism   (the pp_eval_candidates device path, captured)
//   -> k_lns_apply (decision, schedule and pool update, loop condition)
// so a whole repair is one graph launch and one synchronisation instead of a host round trip per
// round.  Results are identical to the host-driven loop (tests/test_lns_gpu.py).
#include "pp_internal.cuh"

namespace {

constexpr int LNS_THREADS = 1024;
constexpr int LNS_WMAX = 64;   // candidate_width supported by the graph path
constexpr int LNS_MAXDEG = 7;  // rook lists of <= 7: numpy's mean is then a sequential sum

struct LnsCtl {
    int32_t pool_n, iters, stalled, stop;
    int32_t max_iters, only_positive, pad0, pad1;
    double threshold;
};

__device__ __forceinline__ bool key_before(unsigned long long ka, int ba, unsigned long long kb, int bb) {
    return ka > kb || (ka == kb && ba < bb);  // similarity descending, block ascending
}

__global__ void k_lns_begin(const LnsCtl *__restrict__ ctl, cudaGraphConditionalHandle h) {
    cudaGraphSetConditional(h, (ctl->pool_n > 0 && ctl->max_iters > 0) ? 1u : 0u);
}

// The first W pool blocks in (similarity desc, block asc) order into cand[0..W) (-1 padding).
// similarity (hybrid.py:142-156): -mean |mean_grade[b] - mean_grade[j]| over the rook neighbours j
// already scheduled, in rook order (np.mean of <= 7 values: a sequential sum over the list, then
// one division); -inf without one.  Sorted on -similarity, so -0.0 and +0.0 tie.
__global__ void __launch_bounds__(LNS_THREADS) k_lns_rank(const LnsCtl *__restrict__ ctl, const int32_t *__restrict__ pool,
                                                          const int32_t *__restrict__ assign, const double *__restrict__ mg,
                                                          const int32_t *__restrict__ rptr, const int32_t *__restrict__ ridx,
                                                          unsigned long long *__restrict__ keys, int32_t *__restrict__ cand,
                                                          int W) {
    __shared__ unsigned long long s_k[LNS_THREADS / 32];
    __shared__ int s_b[LNS_THREADS / 32];
    __shared__ unsigned long long s_pk;
    __shared__ int s_pb, s_done;
    constexpr unsigned FULL = 0xffffffffu;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = ctl->pool_n;
    for (int i = tid; i < n; i += LNS_THREADS) {
        const int b = pool[i];
        const double gb = mg[b];
        double acc = 0.0;
        int cnt = 0;
        for (int q = rptr[b]; q < rptr[b + 1]; q++) {
            const int j = ridx[q];
            if (assign[j] != -1) {
                const double v = fabs(f64_sub(gb, mg[j]));
                acc = cnt ? f64_add(acc, v) : v;
                cnt++;
            }
        }
        const double sim = cnt ? -f64_div(acc, (double)cnt) : -kInf;
        keys[i] = f64_key(sim == 0.0 ? 0.0 : sim);
    }
    if (tid == 0) s_done = 0;
    __syncthreads();
    unsigned long long pk = 0ull;
    int pb = -1;
    for (int r = 0; r < W; r++) {
        if (s_done) {  // the pool is exhausted: pad
            if (tid == 0) cand[r] = -1;
            continue;
        }
        unsigned long long bk = 0ull;
        int bb = INT_MAX;
        for (int i = tid; i < n; i += LNS_THREADS) {
            const unsigned long long k = keys[i];
            const int b = pool[i];
            const bool elig = r == 0 || key_before(pk, pb, k, b);  // strictly after the previous pick
            if (elig && (bb == INT_MAX || key_before(k, b, bk, bb))) {
                bk = k;
                bb = b;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long ok = __shfl_xor_sync(FULL, bk, o);
            const int ob = __shfl_xor_sync(FULL, bb, o);
            if (ob != INT_MAX && (bb == INT_MAX || key_before(ok, ob, bk, bb))) {
                bk = ok;
                bb = ob;
            }
        }
        if (lane == 0) {
            s_k[warp] = bk;
            s_b[warp] = bb;
        }
        __syncthreads();
        if (warp == 0) {
            bk = s_k[lane];
            bb = s_b[lane];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long ok = __shfl_xor_sync(FULL, bk, o);
                const int ob = __shfl_xor_sync(FULL, bb, o);
                if (ob != INT_MAX && (bb == INT_MAX || key_before(ok, ob, bk, bb))) {
                    bk = ok;
                    bb = ob;
                }
            }
            if (lane == 0) {
                cand[r] = bb == INT_MAX ? -1 : bb;
                s_pk = bk;
                s_pb = bb;
                if (bb == INT_MAX) s_done = 1;
            }
        }
        __syncthreads();
        pk = s_pk;
        pb = s_pb;
    }
}

// The round's decision (hybrid.py:252-266) and the loop condition.
__global__ void k_lns_apply(LnsCtl *__restrict__ ctl, const pp_best *__restrict__ rec, const BlockRow *__restrict__ rows,
                            int32_t *__restrict__ assign, int32_t *__restrict__ pool, int32_t *__restrict__ pos,
                            cudaGraphConditionalHandle h) {
    if (threadIdx.x != 0) return;
    const pp_best best = rec[0];
    bool go = false;
    if (best.block < 0) {
        ctl->stalled = 1;
        ctl->stop = 1;
    } else if (ctl->only_positive && !(best.value > 0.0)) {
        ctl->stop = 1;
    } else {
        pp_best ch = best;
        if (rows[best.block].spatial < ctl->threshold) ch = rec[1];  // the realism fallback's choice
        PP_DCHECK(ch.block >= 0 && pos[ch.block] >= 0);
        assign[ch.block] = ch.period;
        const int i = pos[ch.block], last = pool[--ctl->pool_n];  // unordered pool: swap-remove
        pool[i] = last;
        pos[last] = i;
        pos[ch.block] = -1;
        ctl->iters++;
        go = ctl->pool_n > 0 && ctl->iters < ctl->max_iters;
    }
    cudaGraphSetConditional(h, go ? 1u : 0u);
}

// The graph: k_lns_begin (the initial condition) -> WHILE { the round }, the round captured
// into the loop body (c->lns_graph / c->lns_exec)
static int lns_build_graph(pp_ctx *c, cudaStream_t st, int W, uint32_t flags, LnsCtl *dctl, int32_t *dpool,
                           int32_t *dpos, int32_t *dcand, pp_best *rec, const pp_cand_out &o) {
    cudaGraph_t g = nullptr;
    auto bail = [&](int r) {
        if (g) cudaGraphDestroy(g);
        return r;
    };
    CUDA_TRY(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle hc;
    if (cudaGraphConditionalHandleCreate(&hc, g, 0, cudaGraphCondAssignDefault) != cudaSuccess)
        return bail(fail(PP_ERR_CUDA, "cudaGraphConditionalHandleCreate: %s", cudaGetErrorString(cudaGetLastError())));
    cudaGraphNode_t begin;
    {
        cudaKernelNodeParams kp = {};
        void *args[] = {&dctl, &hc};
        kp.func = reinterpret_cast<void *>(k_lns_begin);
        kp.gridDim = dim3(1);
        kp.blockDim = dim3(1);
        kp.kernelParams = args;
        if (cudaGraphAddKernelNode(&begin, g, nullptr, 0, &kp) != cudaSuccess)
            return bail(fail(PP_ERR_CUDA, "graph: k_lns_begin node: %s", cudaGetErrorString(cudaGetLastError())));
    }
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = hc;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t loop;
    if (cudaGraphAddNode(&loop, g, &begin, 1, &cp) != cudaSuccess)
        return bail(fail(PP_ERR_CUDA, "graph: WHILE node: %s", cudaGetErrorString(cudaGetLastError())));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    // the round, captured into the loop body
    if (cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
        return bail(fail(PP_ERR_CUDA, "capture: %s", cudaGetErrorString(cudaGetLastError())));
    // the ranking (one CTA) runs beside the period masses (one cluster): both read only the round's
    // schedule; the evaluation joins them
    int rc = PP_OK;
    rc = ensure_side_stream(c);
    if (rc == PP_OK && (cudaEventRecord(c->ev_fork, st) != cudaSuccess || cudaStreamWaitEvent(c->side, c->ev_fork, 0) != cudaSuccess))
        rc = fail(PP_ERR_CUDA, "lns: fork");
    if (rc == PP_OK) {
        k_lns_rank<<<1, LNS_THREADS, 0, c->side>>>(dctl, dpool, c->assign_ptr, c->lns_mg.as<double>(),
                                                   c->lns_rptr.as<int32_t>(), c->lns_ridx.as<int32_t>(),
                                                   c->lns_keys.as<unsigned long long>(), dcand, W);
        if (cudaGetLastError() != cudaSuccess || cudaEventRecord(c->ev_join, c->side) != cudaSuccess)
            rc = fail(PP_ERR_CUDA, "lns: k_lns_rank");
    }
    if (rc == PP_OK) {
        bool launched;
        c->pm_dirty = true;  // every round recomputes the period masses of the round's schedule
        rc = refresh_pm(c, st, &launched, nullptr);
    }
    if (rc == PP_OK && cudaStreamWaitEvent(st, c->ev_join, 0) != cudaSuccess) rc = fail(PP_ERR_CUDA, "lns: join");
    if (rc == PP_OK) rc = pp_eval_candidates(c, dcand, W, PP_SCENARIO_EXPECTED, flags, &o, PP_MEM_DEVICE, st);
    if (rc == PP_OK) {
        k_lns_apply<<<1, 32, 0, st>>>(dctl, rec, c->rows.as<BlockRow>(), c->assign.as<int32_t>(), dpool, dpos, hc);
        if (cudaGetLastError() != cudaSuccess) rc = fail(PP_ERR_CUDA, "k_lns_apply launch");
    }
    cudaGraph_t cap = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(st, &cap);
    if (rc != PP_OK) return bail(rc);
    if (ec != cudaSuccess) return bail(fail(PP_ERR_CUDA, "end capture: %s", cudaGetErrorString(ec)));
    cudaGraphExec_t ex = nullptr;
    if (cudaGraphInstantiate(&ex, g, 0) != cudaSuccess)
        return bail(fail(PP_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(cudaGetLastError())));
    c->lns_graph = g;
    c->lns_exec = ex;
    return PP_OK;
}

}  // namespace

extern "C" {

int pp_set_rook(pp_ctx *c, const int32_t *rook_ptr, const int32_t *rook_idx) {
    if (!c || !c->have_instance) return fail(PP_ERR_STATE, "pp_set_instance first");
    if (!rook_ptr) return fail(PP_ERR_INVALID_ARGS, "rook_ptr is NULL");
    const int B = c->B;
    if (rook_ptr[0] != 0) return fail(PP_ERR_INVALID_ARGS, "rook_ptr[0] must be 0");
    for (int b = 0; b < B; b++) {
        const int d = rook_ptr[b + 1] - rook_ptr[b];
        if (d < 0 || d > LNS_MAXDEG)
            return fail(PP_ERR_SHAPE, "block %d has %d rook neighbours (the device ranking takes <= %d)", b, d,
                        LNS_MAXDEG);
    }
    const int E = rook_ptr[B];
    if (E > 0 && !rook_idx) return fail(PP_ERR_INVALID_ARGS, "rook_idx is NULL");
    for (int q = 0; q < E; q++)
        if (rook_idx[q] < 0 || rook_idx[q] >= B) return fail(PP_ERR_INVALID_ARGS, "rook neighbour %d out of range", rook_idx[q]);
    TRY(use_device(c));
    TRY(c->lns_rptr.ensure(sizeof(int32_t) * (size_t)(B + 1)));
    TRY(c->lns_ridx.ensure(sizeof(int32_t) * (size_t)std::max(E, 1)));
    TRY(c->lns_rpi.ensure(sizeof(int32_t) * (size_t)std::max(E, 1)));
    CUDA_TRY(cudaMemcpy(c->lns_rptr.ptr, rook_ptr, sizeof(int32_t) * (size_t)(B + 1), cudaMemcpyHostToDevice));
    if (E > 0) {
        std::vector<int32_t> pi((size_t)E);  // the pair's first block (rook_weights' i_idx)
        for (int b = 0; b < B; b++)
            for (int q = rook_ptr[b]; q < rook_ptr[b + 1]; q++) pi[q] = b;
        CUDA_TRY(cudaMemcpy(c->lns_ridx.ptr, rook_idx, sizeof(int32_t) * (size_t)E, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(c->lns_rpi.ptr, pi.data(), sizeof(int32_t) * (size_t)E, cudaMemcpyHostToDevice));
    }
    c->rook_pairs = E;
    c->have_rook = true;
    return PP_OK;
}

int pp_lns_insert(pp_ctx *c, int32_t *assign, uint8_t *pool, const double *mean_grade, int32_t max_iters,
                  int32_t candidate_width, double realism_threshold, int32_t only_positive, uint32_t flags,
                  int32_t *iters_out, int32_t *stalled_out) {
    if (!c || !c->have_instance || !c->have_spatial || !c->have_rook)
        return fail(PP_ERR_STATE, "pp_set_instance, pp_set_geology and pp_set_rook first");
    if (!assign || !pool || !mean_grade || !iters_out || !stalled_out) return fail(PP_ERR_INVALID_ARGS, "bad arguments");
    if (candidate_width < 1 || candidate_width > LNS_WMAX)
        return fail(PP_ERR_SHAPE, "candidate_width %d outside [1, %d]", candidate_width, LNS_WMAX);
    if (max_iters < 0) return fail(PP_ERR_INVALID_ARGS, "max_iters < 0");
    flags &= (PP_NET_MINING_COST | PP_USE_SIGMA);
    HostTrace ht("pp_lns_insert");
    TRY(use_device(c));
    cudaStream_t st = c->stream;
    const int B = c->B, W = candidate_width;
    for (int b = 0; b < B; b++)
        if (assign[b] < -1 || assign[b] >= c->T) return fail(PP_ERR_INVALID_ARGS, "schedule has period indices out of range");
    TRY(pp_set_schedule(c, assign, PP_MEM_HOST, st));
    TRY(check_ready(c, flags, -1));
    // the pool as an unordered list (the ranking's order is total, so list order does not matter)
    std::vector<int32_t> list, pos((size_t)B, -1);
    list.reserve(1024);
    for (int b = 0; b < B; b++)
        if (pool[b]) {
            pos[b] = (int32_t)list.size();
            list.push_back(b);
        }
    LnsCtl h{};
    h.pool_n = (int32_t)list.size();
    h.max_iters = max_iters;
    h.only_positive = only_positive ? 1 : 0;
    h.threshold = realism_threshold;
    TRY(c->lns_ctl.ensure(sizeof(LnsCtl)));
    TRY(c->lns_pool.ensure(sizeof(int32_t) * (size_t)std::max<size_t>(list.size(), 1)));
    TRY(c->lns_pos.ensure(sizeof(int32_t) * (size_t)B));
    TRY(c->lns_mg.ensure(sizeof(double) * (size_t)B));
    TRY(c->lns_keys.ensure(sizeof(unsigned long long) * (size_t)std::max<size_t>(list.size(), 1)));
    // per round: cand[W] | best_t[W] | best_val[W] | feasible[W] | two 16-byte pp_best records
    TRY(c->lns_out.ensure(64 + 2 * sizeof(pp_best) + (size_t)W * (4 + 4 + 8 + 1) + 64));
    unsigned char *ob = c->lns_out.as<unsigned char>();
    pp_best *rec = reinterpret_cast<pp_best *>(ob);  // 256-byte aligned allocation: 16-byte aligned
    int32_t *dcand = reinterpret_cast<int32_t *>(ob + 64);
    int32_t *bt = dcand + W;
    double *bv = reinterpret_cast<double *>(ob + 64 + (((size_t)8 * W + 7) & ~(size_t)7));
    uint8_t *fe = reinterpret_cast<uint8_t *>(bv + W);
    LnsCtl *dctl = c->lns_ctl.as<LnsCtl>();
    int32_t *dpool = c->lns_pool.as<int32_t>(), *dpos = c->lns_pos.as<int32_t>();
    if (!list.empty()) CUDA_TRY(cudaMemcpyAsync(dpool, list.data(), sizeof(int32_t) * list.size(), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(dpos, pos.data(), sizeof(int32_t) * (size_t)B, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(c->lns_mg.ptr, mean_grade, sizeof(double) * (size_t)B, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemcpyAsync(dctl, &h, sizeof(LnsCtl), cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaMemsetAsync(dcand, 0xff, sizeof(int32_t) * (size_t)W, st));

    pp_cand_out o;
    memset(&o, 0, sizeof(o));
    o.best_t = bt;
    o.best_val = bv;
    o.feasible = fe;
    o.global = rec;
    o.realism = rec + 1;
    // the executable graph is kept in the context and reused while its shape (width, flags) and
    // every device buffer it references (no re-allocation since: the sum of the buffers'
    // allocation generations) are unchanged; a call then costs the uploads, one launch, the copies
    uint64_t gensum = 0;
    for (DevBuf *d : c->all()) gensum += d->gen;
    const uint64_t key[3] = {(uint64_t)W, (uint64_t)flags, gensum};
    if (!c->lns_exec || memcmp(key, c->lns_key, sizeof(key)) != 0) {
        if (c->lns_exec) cudaGraphExecDestroy(c->lns_exec);
        if (c->lns_graph) cudaGraphDestroy(c->lns_graph);
        c->lns_exec = nullptr;
        c->lns_graph = nullptr;
        // one uncaptured evaluation first: every scratch buffer and kernel attribute the round needs
        // is in place before capture (no allocation or attribute call may happen inside it)
        TRY(pp_eval_candidates(c, dcand, W, PP_SCENARIO_EXPECTED, flags, &o, PP_MEM_DEVICE, st));
        gensum = 0;  // (that evaluation may have grown a buffer)
        for (DevBuf *d : c->all()) gensum += d->gen;
        const uint64_t key2[3] = {(uint64_t)W, (uint64_t)flags, gensum};
        TRY(lns_build_graph(c, st, W, flags, dctl, dpool, dpos, dcand, rec, o));
        memcpy(c->lns_key, key2, sizeof(key2));
        ht.mark("build");
    }
    if (cudaGraphLaunch(c->lns_exec, st) != cudaSuccess) {
        c->pm_dirty = true;
        return fail(PP_ERR_CUDA, "graph launch: %s", cudaGetErrorString(cudaGetLastError()));
    }
    c->pm_dirty = true;  // the schedule changes on the device
    CUDA_TRY(cudaMemcpyAsync(assign, c->assign.ptr, sizeof(int32_t) * (size_t)B, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(pos.data(), dpos, sizeof(int32_t) * (size_t)B, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(&h, dctl, sizeof(LnsCtl), cudaMemcpyDeviceToHost, st));
    const cudaError_t es = cudaStreamSynchronize(st);
    if (es != cudaSuccess) return fail(PP_ERR_CUDA, "lns graph: %s", cudaGetErrorString(es));
    ht.mark("run+d2h");
    for (int b = 0; b < B; b++) pool[b] = pos[b] >= 0 ? 1 : 0;
    *iters_out = h.iters;
    *stalled_out = h.stalled;
    return PP_OK;
}

}  // extern "C"
