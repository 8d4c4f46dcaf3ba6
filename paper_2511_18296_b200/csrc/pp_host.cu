// pp_host.cu -- host-native pieces of the GA generation (no device work).
//
// pp_host_mutate: HybridSearch._mutate (hybrid.py:692-714), the per-block reassignment that
// keeps precedence validity, as a native loop driven by the caller's numpy Generator stream.
// The reference draws from a numpy Generator over PCG64 (rng.py:23-32): rng.random() consumes
// one 64-bit output ((x >> 11) * 2^-53); rng.integers(lo, hi) (int64, hi - lo <= 2^32) draws
// 32-bit words through the bit generator's shared uint32 buffer (the low half of a fresh
// 64-bit output, the high half kept for the next 32-bit draw) and maps them with Lemire's
// bounded multiply and its rejection test; a range of one value draws nothing.  The caller
// passes a block of raw 64-bit outputs (PCG64.random_raw) and the buffer state, and gets back
// how many outputs were consumed and the buffer state after them, so it can set the
// Generator exactly where the reference's loop would have left it.
#include "pp_internal.cuh"

namespace {

struct RawStream {
    const uint64_t *raw;
    int64_t n, pos;
    int32_t has;     // a buffered upper 32-bit half is pending
    uint32_t half;   // that half
    bool exhausted = false;
    uint64_t u64() {
        if (pos >= n) {
            exhausted = true;
            return 0;
        }
        return raw[pos++];
    }
    uint32_t u32() {
        if (has) {
            has = 0;
            return half;
        }
        const uint64_t v = u64();
        has = 1;
        half = (uint32_t)(v >> 32);
        return (uint32_t)(v & 0xffffffffull);
    }
    double random() { return (double)(u64() >> 11) * (1.0 / 9007199254740992.0); }
    // Generator.integers(lo, hi), hi > lo, hi - lo <= 2^32
    int64_t integers(int64_t lo, int64_t hi) {
        const uint64_t rng = (uint64_t)(hi - lo - 1);
        if (rng == 0) return lo;
        if (rng == 0xffffffffull) return lo + (int64_t)u32();
        const uint32_t rng_excl = (uint32_t)rng + 1u;
        uint64_t m = (uint64_t)u32() * rng_excl;
        uint32_t left = (uint32_t)(m & 0xffffffffull);
        if (left < rng_excl) {
            const uint32_t thr = (uint32_t)((0xffffffffull - rng) % rng_excl);
            while (left < thr) {
                m = (uint64_t)u32() * rng_excl;
                left = (uint32_t)(m & 0xffffffffull);
                if (exhausted) break;
            }
        }
        return lo + (int64_t)(m >> 32);
    }
};

}  // namespace

extern "C" {

int pp_host_mutate(int64_t *assign, int32_t n_blocks, const int64_t *blocks, int64_t n_sel, const int32_t *pred_ptr,
                   const int32_t *pred_idx, const int32_t *succ_ptr, const int32_t *succ_idx, int32_t n_periods,
                   double rate, const uint64_t *raw, int64_t n_raw, int32_t *has_u32, uint32_t *uinteger,
                   int64_t *consumed) {
    if (!assign || (n_sel > 0 && !blocks) || !pred_ptr || !succ_ptr || !has_u32 || !uinteger || !consumed ||
        n_blocks < 0 || n_periods < 1 || (n_raw > 0 && !raw))
        return fail(PP_ERR_INVALID_ARGS, "pp_host_mutate: bad arguments");
    RawStream rs{raw, n_raw, 0, *has_u32, *uinteger};
    const int64_t UN = -1;
    std::vector<int64_t> undo_b;  // restore the caller's array if the stream runs out
    std::vector<int64_t> undo_t;
    for (int64_t i = 0; i < n_sel; i++) {
        const int64_t b = blocks[i];
        if (b < 0 || b >= n_blocks) return fail(PP_ERR_INVALID_ARGS, "pp_host_mutate: block %lld out of range", (long long)b);
        if (rs.random() >= rate) {
            if (rs.exhausted) break;
            continue;
        }
        const int32_t p0 = pred_ptr[b], p1 = pred_ptr[b + 1], s0 = succ_ptr[b], s1 = succ_ptr[b + 1];
        const int64_t old = assign[b];
        if (old == UN) {
            bool any_un = false;
            int64_t t_min = 0;
            bool first = true;
            for (int32_t k = p0; k < p1; k++) {
                const int64_t tp = assign[pred_idx[k]];
                if (tp == UN) {
                    any_un = true;
                    break;
                }
                t_min = first ? tp : std::max(t_min, tp);
                first = false;
            }
            if (any_un) continue;
            const int64_t v = rs.integers(t_min, n_periods);
            undo_b.push_back(b);
            undo_t.push_back(old);
            assign[b] = v;
        } else {
            bool any_mined_succ = false;
            int64_t t_max = n_periods - 1;
            bool firsts = true;
            for (int32_t k = s0; k < s1; k++) {
                const int64_t tc = assign[succ_idx[k]];
                if (tc == UN) continue;
                any_mined_succ = true;
                t_max = firsts ? tc : std::min(t_max, tc);
                firsts = false;
            }
            if (!any_mined_succ && rs.random() < 0.25) {
                undo_b.push_back(b);
                undo_t.push_back(old);
                assign[b] = UN;
                continue;
            }
            int64_t t_min = 0;  // max over the predecessors' periods as stored (UNMINED = -1 included)
            bool firstp = true;
            for (int32_t k = p0; k < p1; k++) {
                const int64_t tp = assign[pred_idx[k]];
                t_min = firstp ? tp : std::max(t_min, tp);
                firstp = false;
            }
            if (t_min <= t_max) {
                const int64_t v = rs.integers(t_min, t_max + 1);
                undo_b.push_back(b);
                undo_t.push_back(old);
                assign[b] = v;
            }
        }
        if (rs.exhausted) break;
    }
    if (rs.exhausted) {  // not enough raw outputs: undo, the caller retries with a longer block
        for (size_t k = undo_b.size(); k-- > 0;) assign[undo_b[k]] = undo_t[k];
        return fail(PP_ERR_SHAPE, "pp_host_mutate: raw stream exhausted");
    }
    *consumed = rs.pos;
    *has_u32 = rs.has;
    *uinteger = rs.half;
    return PP_OK;
}

}  // extern "C"
