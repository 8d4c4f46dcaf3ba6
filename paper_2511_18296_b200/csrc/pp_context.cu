// pp_context.cu -- error channel, device context and library entry points of the C ABI.
//
// Translation units of libpitplan_b200.so (C ABI: include/pitplan_b200.h):
//   pp_context.cu   error channel, device context, shared host helpers
//   pp_schedule.cu  period masses (numpy pairwise tree, bit-exact), check_feasible,
//                   topological-wave repair, table preparation (geology, scenario tables,
//                   linear ENPV), accepted-move application, ordered argmax reduce
//   pp_eval.cu      evaluate_candidates_parallel: staged fast path + general kernel
//   pp_moves.cu     explicit reassign / unmine / swap moves
//
// All float arithmetic on the value path uses explicit round-to-nearest intrinsics and the
// library is compiled with -fmad=false: no multiply-add is ever contracted, so every double
// matches the reference's numpy/Python scalar evaluation bit for bit.

#include "pp_internal.cuh"
#include <atomic>
#include <mutex>
#include <vector>

// ------------------------------------------------------------------------------------
// error plumbing
// ------------------------------------------------------------------------------------
static thread_local std::string g_last_error;

int fail(int code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}


// Registry of the page-locked buffers pp_host_alloc handed out (host range -> device mapping), so
// the host-mode copy-out resolves its destinations without a driver query per array and call.
namespace {
struct PinnedRange {
    uintptr_t lo, hi, dev;
};
std::mutex g_pinned_mu;
std::vector<PinnedRange> g_pinned;
std::atomic<uint64_t> g_pinned_gen{0};  // bumped on every (un)registration: cached mappings compare it
}  // namespace

uint64_t pinned_generation() { return g_pinned_gen.load(std::memory_order_relaxed); }

void pinned_register(void *host, size_t bytes, void *dev) {
    g_pinned_gen.fetch_add(1, std::memory_order_relaxed);
    std::lock_guard<std::mutex> lock(g_pinned_mu);
    g_pinned.push_back({reinterpret_cast<uintptr_t>(host), reinterpret_cast<uintptr_t>(host) + bytes,
                        reinterpret_cast<uintptr_t>(dev)});
}

void pinned_unregister(void *host) {
    g_pinned_gen.fetch_add(1, std::memory_order_relaxed);
    std::lock_guard<std::mutex> lock(g_pinned_mu);
    const uintptr_t h = reinterpret_cast<uintptr_t>(host);
    for (size_t i = 0; i < g_pinned.size(); i++)
        if (g_pinned[i].lo == h) {
            g_pinned.erase(g_pinned.begin() + (long)i);
            return;
        }
}

void *pinned_lookup(const void *host) {
    std::lock_guard<std::mutex> lock(g_pinned_mu);
    const uintptr_t h = reinterpret_cast<uintptr_t>(host);
    for (const PinnedRange &r : g_pinned)
        if (h >= r.lo && h < r.hi) return reinterpret_cast<void *>(r.dev + (h - r.lo));
    return nullptr;
}

#ifdef PP_CHECKED
// guard-zone registry of the live device buffers (checked builds only)
namespace {
std::mutex g_guard_mu;
std::vector<DevBuf *> g_guard_bufs;
long long g_guard_bad = 0;  // corrupted guards found so far (at free / re-allocation / explicit checks)
}  // namespace

void guard_register(DevBuf *b) {
    std::lock_guard<std::mutex> lock(g_guard_mu);
    g_guard_bufs.push_back(b);
}

void guard_unregister(DevBuf *b) {
    std::lock_guard<std::mutex> lock(g_guard_mu);
    for (size_t i = 0; i < g_guard_bufs.size(); i++)
        if (g_guard_bufs[i] == b) {
            g_guard_bufs.erase(g_guard_bufs.begin() + (long)i);
            return;
        }
}

bool guard_intact(const DevBuf *b) {
    if (!b->base) return true;
    std::vector<unsigned char> h(2 * PP_GUARD);
    if (cudaDeviceSynchronize() != cudaSuccess ||
        cudaMemcpy(h.data(), b->base, PP_GUARD, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(h.data() + PP_GUARD, static_cast<const unsigned char *>(b->ptr) + b->bytes, PP_GUARD,
                   cudaMemcpyDeviceToHost) != cudaSuccess)
        return true;  // a sticky CUDA error is reported by the call that hit it
    size_t first = SIZE_MAX, nbad = 0;
    for (size_t i = 0; i < h.size(); i++)
        if (h[i] != 0xA5) {
            nbad++;
            if (first == SIZE_MAX) first = i;
        }
    if (!nbad) return true;
    std::lock_guard<std::mutex> lock(g_guard_mu);
    g_guard_bad++;
    fprintf(stderr, "[pp checked] guard of a %zu-byte buffer overwritten: %zu bytes, first at %s%zd\n", b->bytes, nbad,
            first < PP_GUARD ? "payload-" : "payload end+", first < PP_GUARD ? (ssize_t)(PP_GUARD - first) : (ssize_t)(first - PP_GUARD));
    return false;
}
#endif

void *mapped_host(const void *p) {
    if (!p) return nullptr;
    if (void *d = pinned_lookup(p)) return d;  // one of pp_host_alloc's buffers: no driver query
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return (a.type == cudaMemoryTypeHost && a.devicePointer) ? a.devicePointer : nullptr;
}

int ensure_side_stream(pp_ctx *c) {
    if (c->side) return PP_OK;
    CUDA_TRY(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device) == cudaSuccess && sms > 0) c->n_sms = sms;
    return PP_OK;
}

int ensure_grid_scratch(pp_ctx *c, int grid) {
    TRY(c->partial.ensure(sizeof(pp_best) * (size_t)std::max(grid, 1)));
    if (c->counter.bytes == 0) {
        TRY(c->counter.ensure(sizeof(unsigned int) * 4));
        CUDA_TRY(dev_zero(c, c->counter.ptr, c->counter.bytes));
    }
    return PP_OK;
}


// (kernel, device) -> largest dynamic shared memory opted in so far; returns 1 (and records it)
// when cudaFuncSetAttribute is still needed for `bytes`
int smem_attr_needed(const void *kern, int device, size_t bytes) {
    struct Entry {
        const void *kern;
        int device;
        size_t bytes;
    };
    static std::mutex mu;
    static std::vector<Entry> seen;
    std::lock_guard<std::mutex> lock(mu);
    for (Entry &e : seen)
        if (e.kern == kern && e.device == device) {
            if (e.bytes >= bytes) return 0;
            e.bytes = bytes;
            return 1;
        }
    seen.push_back(Entry{kern, device, bytes});
    return 1;
}

int pick_kc(int k) {
    if (k <= 2) return 2;
    if (k <= 8) return 8;
    if (k <= 128) return 128;
    return -1;
}

int check_ready(pp_ctx *c, uint32_t flags, int scenario) {
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

int pp_abi_version(void) { return PP_ABI_VERSION; }

#ifdef PP_CHECKED
// negative control of the checked build (not in the header): one byte written just past the end
// of the context's period-mass buffer, as an out-of-bounds kernel store would
PP_API int pp_debug_corrupt_guard(pp_ctx *c) {
    if (!c || !c->pm.ptr) return fail(PP_ERR_STATE, "no period-mass buffer yet");
    CUDA_TRY(cudaMemset(static_cast<unsigned char *>(c->pm.ptr) + c->pm.bytes, 0, 1));
    return PP_OK;
}
#endif

int pp_debug_check_guards(int64_t *n_bad) {
#ifdef PP_CHECKED
    if (!n_bad) return fail(PP_ERR_INVALID_ARGS, "n_bad is NULL");
    std::vector<DevBuf *> bufs;
    {
        std::lock_guard<std::mutex> lock(g_guard_mu);
        bufs = g_guard_bufs;
    }
    for (DevBuf *b : bufs) guard_intact(b);
    std::lock_guard<std::mutex> lock(g_guard_mu);
    *n_bad = g_guard_bad;
    return PP_OK;
#else
    (void)n_bad;
    return fail(PP_ERR_STATE, "not a checked build (build_checked(): libpitplan_b200_checked.so)");
#endif
}

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
    if (c->h_bad) cudaFreeHost(c->h_bad);
    if (c->h_bounce) cudaFreeHost(c->h_bounce);
    if (c->h_stage) cudaFreeHost(c->h_stage);
    if (c->lns_exec) cudaGraphExecDestroy(c->lns_exec);
    if (c->lns_graph) cudaGraphDestroy(c->lns_graph);
    if (c->ev_exec) cudaGraphExecDestroy(c->ev_exec);
    if (c->ev_graph) cudaGraphDestroy(c->ev_graph);
    if (c->side) {
        cudaStreamSynchronize(c->side);
        cudaStreamDestroy(c->side);
    }
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
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
    const size_t n = std::max<size_t>(bytes, 1);
    CUDA_TRY(cudaHostAlloc(ptr, n, cudaHostAllocPortable | cudaHostAllocMapped));
    void *dev = nullptr;
    CUDA_TRY(cudaHostGetDevicePointer(&dev, *ptr, 0));
    pinned_register(*ptr, n, dev);
    return PP_OK;
}

int pp_host_free(void *ptr) {
    if (ptr) {
        pinned_unregister(ptr);
        CUDA_TRY(cudaFreeHost(ptr));
    }
    return PP_OK;
}

}  // extern "C"
