/*
 * pitplan_b200.h -- C ABI of the B200-native move-evaluation engine.
 *
 * The reference (`pitplan`, pure Python) has no FFI: its plug-in point for this
 * path is the Python function
 *     pitplan.evaluate.evaluate_candidates_parallel   (pkg/src/pitplan/evaluate.py:306-318)
 * plus the feasibility / repair helpers it and its callers use:
 *     pitplan.evaluate.check_feasible                 (evaluate.py:82-105)
 *     pitplan.hybrid._precedence_repair_pass          (hybrid.py:493-510)
 *     pitplan.hybrid.lns_repair (unmine fixpoint)     (hybrid.py:199-211)
 * The Python shim `paper_2511_18296_b200.evaluate` keeps those signatures and
 * binds this library with ctypes (INTEGRATION.md shows the binding).
 *
 * Conventions
 *   - every entry point returns an int status: 0 ok, PP_ERR_* otherwise; the
 *     message of the last failure on the calling thread is pp_last_error().
 *   - no C++ exception, abort or silent CPU fallback crosses this boundary.
 *   - `mem` selects the address space of the caller's array arguments:
 *       PP_MEM_HOST   host pointers (pageable or pp_host_alloc'd); the call copies
 *                     in, runs, copies out and returns after the stream drains.
 *       PP_MEM_DEVICE device pointers (e.g. torch tensor data_ptr()); the call only
 *                     enqueues work on `stream` (NULL = the context's own stream).
 *     Instance / scenario uploads (pp_set_instance ...) always take host pointers.
 *   - UNMINED = -1 is the "not scheduled" period, as blockmodel.py:18.
 *   - all floating point is IEEE binary64 with the reference's operation order; the
 *     kernels are compiled without FMA contraction so results are bit-identical to
 *     the reference CPU evaluator.
 *   - a context is not thread-safe; use one context per host thread.
 */
#ifndef PITPLAN_B200_H
#define PITPLAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PP_ABI_VERSION 3

/* status codes (mapped to pitplan.errors classes by the Python shim) */
#define PP_OK 0
#define PP_ERR_INVALID_ARGS 1   /* -> InvalidArgs   (errors.py:16)  */
#define PP_ERR_SHAPE 2          /* -> ShapeMismatch (errors.py:24)  */
#define PP_ERR_CUDA 3           /* -> DeviceError                   */
#define PP_ERR_VALIDATION 4     /* -> ValidationError (errors.py:12) e.g. a cycle */
#define PP_ERR_STATE 5          /* call order: instance/scenarios/schedule missing */

#define PP_MEM_HOST 0
#define PP_MEM_DEVICE 1
#define PP_MEM_DEVICE_BORROW 2  /* pp_set_schedule only: read the caller's device buffer in place */

/* evaluation flags (evaluate_candidates_parallel keyword arguments, evaluate.py:306-318) */
#define PP_NET_MINING_COST 1u   /* net_mining_cost=True: value -= disc[t] * cost[b][t] */
#define PP_LITERAL_VALUE 2u     /* literal_kernel_value=True: unit = mass * 100 */
#define PP_USE_SIGMA 4u         /* sigma is not None: sig_row from the uploaded sigma[S][T] */

#define PP_SCENARIO_EXPECTED (-1) /* s=None: scenario-mean unit values and sigma row */

#define PP_MOVE_REASSIGN 0      /* move (b, t_new): t_new in [-1, T) */
#define PP_MOVE_SWAP 1          /* move (b1, b2): exchange their periods */

#define PP_REPAIR_PUSH_FORWARD 0 /* _precedence_repair_pass (hybrid.py:493-510) */
#define PP_REPAIR_UNMINE 1       /* lns_repair unmine fixpoint (hybrid.py:199-211) */

#if defined(__GNUC__)
#define PP_API __attribute__((visibility("default")))
#else
#define PP_API
#endif

typedef struct pp_ctx pp_ctx;

/* Selected move.  For candidate evaluation: value = improvement, block / period of the
 * move, block = -1 when no candidate is feasible (best is None, evaluate.py:411-421).
 * For explicit moves: value = delta, block = move index (-1 if none), period = -1. */
typedef struct pp_best {
    double value;
    int32_t block;
    int32_t period;
} pp_best;

/* Outputs of pp_eval_candidates; NULL members are not computed / written.
 * best_t, best_val, feasible and global are required. */
typedef struct pp_cand_out {
    int32_t *best_t;     /* [C] best period or -1                    (CandidateMove.period)      */
    double *best_val;    /* [C] improvement or -inf                  (CandidateMove.improvement) */
    uint8_t *feasible;   /* [C]                                      (CandidateMove.feasible)    */
    double *trace_val;   /* [C*T] per-(candidate, period) value, -inf if infeasible (trace CSV)  */
    uint8_t *trace_feas; /* [C*T] per-(candidate, period) feasibility                             */
    double *exp_delta;   /* [C*T] expected delta over scenarios (np.mean of per-scenario deltas)  */
    double *cvar;        /* [C*T] CVaR10 of the per-scenario deltas (saa.py:150-166 semantics)    */
    float *scen_delta;   /* [C*S*T] per-scenario delta, layout [candidate][scenario][period]      */
    pp_best *global;     /* [1] overall best move (evaluate.py:404-421 order)                     */
    /* Sparse statistics: when n_pairs is non-NULL, every feasible (candidate, period) move --
     * precedence window and capacity both satisfied, i.e. trace_feas == 1 -- is appended as
     * (candidate index into cand[], period, expected delta, CVaR10) and *n_pairs receives the
     * count.  Capacity C*T.  The order of the entries is unspecified; the set and every value
     * are deterministic.  About 8% of the moves are feasible at C2, so this is ~12x less
     * device-to-host traffic than exp_delta + cvar. */
    int32_t *pair_cand;   /* [<= C*T] */
    int32_t *pair_period; /* [<= C*T] */
    double *pair_exp;     /* [<= C*T] */
    double *pair_cvar;    /* [<= C*T] */
    int32_t *n_pairs;     /* [1] */
    /* Second selection key (may be NULL): the feasible candidate first in lns_repair's realism
     * fallback order -- geological consistency spatial[b] descending, then block ascending
     * (hybrid.py:256-263) -- as {value = spatial[b], block, period = its best period}; block = -1
     * when no candidate is feasible.  16-byte aligned. */
    pp_best *realism;
} pp_cand_out;

/* Outputs of pp_eval_moves; NULL members are not computed / written.
 * feasible, delta and global are required. */
typedef struct pp_move_out {
    uint8_t *feasible;  /* [M] */
    double *delta;      /* [M] kernel-value delta (parity key), -inf if infeasible */
    double *exp_delta;  /* [M] */
    double *cvar;       /* [M] */
    float *scen_delta;  /* [M*S] layout [move][scenario] */
    pp_best *global;    /* [1] value = best delta, block = move index (lowest on ties) */
} pp_move_out;

/* ---- library / context --------------------------------------------------------- */
PP_API int pp_abi_version(void);
PP_API const char *pp_last_error(void);
PP_API int pp_device_count(int *count);
PP_API int pp_ctx_create(int device, pp_ctx **out);
PP_API int pp_ctx_destroy(pp_ctx *ctx);
PP_API int pp_ctx_stream(pp_ctx *ctx, void **stream);          /* the context's cudaStream_t */
PP_API int pp_synchronize(pp_ctx *ctx, void *stream);
PP_API int pp_host_alloc(size_t bytes, void **ptr);             /* pinned host memory */
PP_API int pp_host_free(void *ptr);
/* Diagnostic (no reference counterpart): in the checked build (libpitplan_b200_checked.so,
 * -DPP_CHECKED) verifies the 512-byte guard zones around every live device buffer and returns the
 * number of overwritten guards found so far (also checked at every free / re-allocation);
 * PP_ERR_STATE in the release build. */
PP_API int pp_debug_check_guards(int64_t *n_bad);

/* ---- static tables (host pointers) ------------------------------------------------
 * Instance: precedence edge list in reference order (blockmodel.py:94, 180-184),
 * masses (blockmodel.py:128), undiscounted mining cost [B][T] (blockmodel.py:137),
 * capacity [T], discount table disc[t] = (1+r)^-t computed by the host (evaluate.py:341).
 * Builds CSR adjacency and topological levels on the device side; PP_ERR_VALIDATION
 * on a cycle (blockmodel.py:228-245). */
PP_API int pp_set_instance(pp_ctx *ctx, int32_t n_blocks, int32_t n_periods, int64_t n_edges,
                    const int32_t *edge_i, const int32_t *edge_j, const double *mass,
                    const double *cost, const double *capacity, const double *discount);
/* spatial[b] = geological_consistency(features_b, params, diameter) (uncertainty.py:185-191,
 * evaluate.py:342-347), computed on the device. */
PP_API int pp_set_geology(pp_ctx *ctx, const double *alteration, const double *structural,
                   const double *dist_intrusion, double w1, double w2, double w3,
                   double diameter);
/* Scenario tables: vmax[S][B] = max over modes of v[s][b][o] (evaluate.py:108-124) in the
 * reference layout (transposed to block-major on the device), sigma[S][T] or NULL
 * (uncertainty.py:276-321).  Derives unit_mean[b] (evaluate.py:302) and the scenario-mean
 * sigma row (evaluate.py:351) on the device. */
PP_API int pp_set_scenarios(pp_ctx *ctx, int32_t n_scenarios, const double *vmax_sb,
                     const double *sigma_st);

/* Device-side ingestion of a scenario set: the value table is built on the
 * device from grades[S][B] as scenario_mode_values does (evaluate.py:116-124),
 *   v[s][b][o] = ((grade * mass) * price) * recovery[o % n_recovery] - mass * proc_cost[o % n_proc_cost],
 * vmax = max over the n_modes modes -- bit-identical to the host computation -- so a freshly sampled
 * set (the DW loop refreshes one per iteration, colgen.py:477-478) crosses PCIe once as grades
 * and never materialises on the host.  sigma_st as pp_set_scenarios. */
PP_API int pp_set_scenarios_grades(pp_ctx *ctx, int32_t n_scenarios, const double *grades_sb, int32_t n_modes,
                                   double price, const double *recovery, int32_t n_recovery, const double *proc_cost,
                                   int32_t n_proc_cost, const double *sigma_st);
/* VAE scenario source on the device (vae.py:91-93, 284-292; the decoder of nn.py:42-53): the
 * decoder's n_layers dense layers with widths[0] = latent dim ... widths[n_layers] = B, params =
 * for each layer W[out][in] (row-major, as Dense.W) then b[out], and the normalisation norm_mean[B],
 * norm_std[B].  The decode agrees with numpy's (BLAS) to rounding, not bit for bit. */
PP_API int pp_set_vae_decoder(pp_ctx *ctx, int32_t n_layers, const int32_t *widths, const double *params,
                              const double *norm_mean, const double *norm_std);
/* grades[S][B] = max(decoder(z) * norm_std + norm_mean, 0) for prior samples z[S][latent]. */
PP_API int pp_vae_decode(pp_ctx *ctx, int32_t n_scenarios, const double *z, double *grades_out, int32_t mem,
                         void *stream);
/* Decode z[S][latent] and bind the grades as the scenario set (the value table built on the device
 * as pp_set_scenarios_grades; the grades never visit the host). */
PP_API int pp_set_scenarios_vae(pp_ctx *ctx, int32_t n_scenarios, const double *z, int32_t n_modes, double price,
                                const double *recovery, int32_t n_recovery, const double *proc_cost,
                                int32_t n_proc_cost, const double *sigma_st);
/* uncertainty_factors (uncertainty.py:276-321) on the device for grades[S][B]: sigma[S][T] =
 * clip(f_spatial[s] * phi[t] * psi, 1e-6, 2), f_spatial = 1 - Moran's I + local CV (1 + local CV
 * for a zero-variance field), Moran's I over the rook pairs of pp_set_rook.  phi[T] =
 * exp(-kappa t) and psi (psi_geological) come from the host.  moran_out[S] (NaN when degenerate)
 * and local_out[S] may be NULL.  Agrees with the reference to rounding: its Moran denominator is a
 * BLAS dot product, here a numpy-order pairwise sum. */
PP_API int pp_uncertainty_sigma(pp_ctx *ctx, int32_t n_scenarios, const double *grades, const double *phi, double psi,
                                double *sigma_out, double *moran_out, double *local_out, int32_t mem, void *stream);
/* The bound value table back in the reference layout vmax[S][B] (host output). */
PP_API int pp_get_scenario_values(pp_ctx *ctx, double *vmax_sb_out);

/* ---- schedule -------------------------------------------------------------------- */
/* Install assign[B] as the current schedule (copied, or borrowed in place with
 * PP_MEM_DEVICE_BORROW until the next call).  period_mass[t] = masses[assign == t].sum()
 * is recomputed bit-exactly (numpy pairwise summation, evaluate.py:334-337) by the next
 * evaluation launch, overlapped with it through programmatic dependent launch.
 * PP_MEM_HOST: the copy is stream-ordered, not synchronous -- a pageable buffer may be
 * reused on return (the driver stages it); a page-locked buffer must stay unchanged until
 * the next synchronous call returns.  Period indices outside [-1, T) are an error
 * (PP_ERR_INVALID_ARGS): checked here, or -- for B <= 65536 and T <= 16 -- on the device by
 * the period-mass kernel and reported by the next host-mode call, after which the context
 * has no schedule until the next pp_set_schedule. */
PP_API int pp_set_schedule(pp_ctx *ctx, const int32_t *assign, int32_t mem, void *stream);
/* Apply accepted deltas assign[blocks[k]] = periods[k] and recompute period_mass. */
PP_API int pp_apply_moves(pp_ctx *ctx, const int32_t *blocks, const int32_t *periods, int32_t n,
                   int32_t mem, void *stream);
PP_API int pp_get_schedule(pp_ctx *ctx, int32_t *assign_out, double *period_mass_out, int32_t mem,
                    void *stream);

/* ---- hot path ---------------------------------------------------------------------- */
/* evaluate_candidates_parallel (evaluate.py:306-430) against the current schedule.
 * scenario: PP_SCENARIO_EXPECTED (s=None) or k in [0, S) (s=k).  Candidates may repeat;
 * results are in input order and independent of any launch geometry.  Candidate ids outside
 * [0, B) are PP_ERR_INVALID_ARGS in PP_MEM_HOST mode; in PP_MEM_DEVICE mode they are skipped
 * (no move, no per-candidate output written).  `global` must be 16-byte aligned (it is updated
 * with a 128-bit compare-and-swap). */
PP_API int pp_eval_candidates(pp_ctx *ctx, const int32_t *cand, int32_t n_cand, int32_t scenario,
                       uint32_t flags, const pp_cand_out *out, int32_t mem, void *stream);
/* Explicit moves against the current schedule: kind PP_MOVE_REASSIGN with (a=block,
 * b=t_new) or PP_MOVE_SWAP with (a=b1, b=b2); feasibility rules of hybrid.py:348-403. */
PP_API int pp_eval_moves(pp_ctx *ctx, int32_t kind, const int32_t *a, const int32_t *b, int32_t n_moves,
                  int32_t scenario, uint32_t flags, const pp_move_out *out, int32_t mem,
                  void *stream);
/* check_feasible (evaluate.py:82-105) for P schedules assign[P][B]. */
PP_API int pp_check_feasible(pp_ctx *ctx, const int32_t *assign, int32_t n_sched, int64_t *pred_count,
                      double *excess, double *violation, double *period_mass, int32_t mem,
                      void *stream);
/* Batched repair of P schedules in place, in topological waves:
 * PP_REPAIR_PUSH_FORWARD = _precedence_repair_pass, PP_REPAIR_UNMINE = the unmine fixpoint
 * (unmined_out[P][B] = 1 where the fixpoint unmined a block; may be NULL). */
PP_API int pp_repair(pp_ctx *ctx, int32_t *assign, int32_t n_sched, int32_t mode, uint8_t *unmined_out,
              int32_t mem, void *stream);
/* lns_repair's over-capacity ejection (hybrid.py:213-235) for P schedules assign[P][B] in place,
 * applied after the unmine fixpoint (pp_repair PP_REPAIR_UNMINE): in every period whose mass
 * (numpy pairwise) exceeds its target -- capacity, or capacity * (1 - destroy_fraction) when
 * destroy_fraction > 0 -- the blocks with no mined successor are unmined in ascending
 * (mean_grade[b] * mass[b], b) order until the mass is within the target (sequential f64
 * subtraction).  mean_grade[B] = scenarios.grades.mean(axis=0).  ejected_out[P][B] (may be
 * NULL) marks the ejected blocks. */
PP_API int pp_eject(pp_ctx *ctx, int32_t *assign, int32_t n_sched, const double *mean_grade, double destroy_fraction,
             uint8_t *ejected_out, int32_t mem, void *stream);
/* lns_repair's rook neighbour map (hybrid.py:159-166, the order of uncertainty.rook_weights) as a
 * CSR: rook_ptr[B+1], rook_idx[rook_ptr[B]]; at most 7 neighbours per block (PP_ERR_SHAPE
 * otherwise: numpy's mean of 8+ values is a pairwise sum, the device ranking does the sequential
 * one).  Instance data, set once. */
PP_API int pp_set_rook(pp_ctx *ctx, const int32_t *rook_ptr, const int32_t *rook_idx);
/* lns_repair's insertion loop (hybrid.py:238-266) on the device: one CUDA-graph launch whose
 * conditional WHILE node runs up to max_iters rounds of -- rank the pool by scheduled-neighbour
 * similarity (hybrid.py:142-156) and take the first candidate_width (<= 64) blocks in
 * (similarity desc, block asc) order; evaluate them as evaluate_candidates_parallel with the
 * expected scenario value (flags: PP_NET_MINING_COST, PP_USE_SIGMA); stop when there is no move
 * (*stalled = 1) or, with only_positive, when the best improvement is <= 0; apply the best move,
 * or the realism fallback's choice when the best block's geological consistency is below
 * realism_threshold; drop the block from the pool -- with no host round trip between rounds.
 * assign[B] (host, in/out): the schedule after the destroy step; pool[B] (host u8, in/out): the
 * unassigned blocks; mean_grade[B] = scenarios.grades.mean(axis=0).  Needs pp_set_geology
 * (consistency), pp_set_scenarios and pp_set_rook.  Returns when assign and pool hold the result. */
PP_API int pp_lns_insert(pp_ctx *ctx, int32_t *assign, uint8_t *pool, const double *mean_grade, int32_t max_iters,
                         int32_t candidate_width, double realism_threshold, int32_t only_positive, uint32_t flags,
                         int32_t *iters, int32_t *stalled);
/* Plant data for the relaxed NPV: plant_hours[T] and the throughput rate of the single operating
 * mode (blockmodel.py:63-97).  Only the stage-2 fast path exists on the device: one mode, one rock
 * type, rate > 0 (evaluate.py:149-150); other instances stay on the reference's LP. */
PP_API int pp_set_plant(pp_ctx *ctx, const double *plant_hours, double rate);
/* ScheduleEvaluator.npv_relaxed (evaluate.py:222-234, 244-246) of P schedules assign[P][B] ->
 * npv_out[P], and per_scenario_npv (248-258) -> per_scen_out[P][S] (may be NULL); flags
 * PP_USE_SIGMA weights the stage-2 values by sigma[s][t] (sigma=None otherwise).  Stage 2 per
 * (s, t) is the greedy fractional knapsack of evaluate.py:166-183, bit-exact, for any period size
 * (periods of more than 6144 mined blocks are sorted in global scratch by a second kernel). */
PP_API int pp_npv_relaxed(pp_ctx *ctx, const int32_t *assign, int32_t n_sched, uint32_t flags, double *npv_out,
                   double *per_scen_out, int32_t mem, void *stream);
/* The stage-2 optimum itself (ScheduleEvaluator.stage2_raw / _solve_stage2, evaluate.py:153-183, sigma = 1)
 * of every (schedule p, period t, scenario s): raw_out[P][T][S], and optionally the period's summed
 * undiscounted mining cost cost_out[P][T] (numpy pairwise over its blocks in block order; 0.0 for an
 * empty period).  In PP_MEM_DEVICE mode cost_out of an empty period is unspecified. */
PP_API int pp_stage2(pp_ctx *ctx, const int32_t *assign, int32_t n_sched, double *raw_out, double *cost_out,
                     int32_t mem, void *stream);
/* Relaxed NPV of M one-block variants of a base schedule assign[B]: variant m moves block
 * blocks[m] to periods[m] (-1 = unmine).  Only the two periods a variant changes are re-solved
 * (S stage-2 problems each); the other periods reuse the base schedule's, and the accumulation is
 * the reference's, so npv_out[m] equals pp_npv_relaxed of the modified schedule bit for bit (the
 * exact move value polish_schedule compares, hybrid.py:369-376). */
PP_API int pp_npv_moves(pp_ctx *ctx, const int32_t *assign, const int32_t *blocks, const int32_t *periods,
                 int32_t n_moves, uint32_t flags, double *npv_out, int32_t mem, void *stream);
/* One single-block sweep of polish_schedule (hybrid.py:357-385) natively: for each block in order
 * its options -- unmine (no mined successor), every other period of its precedence window
 * (hybrid.py:348-355) that fits load[t] + m <= cap[t] -- valued by the incremental exact relaxed NPV
 * (pp_npv_moves) in speculative chunks of blocks, the best option strictly above *cur_val + 1e-9
 * accepted in the reference's order.  assign[B] (host, int32), load[T] (host, the caller's running
 * period loads) and *cur_val are updated in place; *improved_out = 1 if any block moved; *calls_out
 * (may be NULL) = device evaluations.  Results identical to the reference's sweep. */
PP_API int pp_polish_sweep(pp_ctx *ctx, int32_t *assign, double *load, double *cur_val, uint32_t flags,
                           int32_t chunk0, int32_t chunk_max, int32_t *improved_out, int64_t *calls_out);
/* The feasible-sequence greedy of column generation's pricing step (colgen.py:236-254;
 * replaces the Python scan in colgen.price_column, colgen.py:207-293).  score[B][T] (host,
 * row-major) is the dual-adjusted value the caller computed exactly as colgen.py:230-234 does;
 * cap[T] = mining_capacity[t] * capacity_slack.  Writes the column's assignment (period or -1,
 * before the capacity_slack trim of colgen.py:256-268, which stays with the caller) and the
 * expansion count; identical to the reference's sequential scan, including its 1e-12 tolerance
 * and node_cap cut-off.  Synchronous. */
PP_API int pp_price_greedy(pp_ctx *ctx, const double *score, const double *cap, int64_t node_cap,
                           int32_t *assign_out, int64_t *expansions_out);
/* spatial[B] = geological_consistency of every block (uncertainty.py:185-191, the factor
 * pp_set_geology computed on the device), e.g. for lns_repair's realism fallback
 * (hybrid.py:238-244, 256-260). */
PP_API int pp_get_spatial(pp_ctx *ctx, double *spatial_out, int32_t mem, void *stream);
/* Ordered reduction of n pp_best records (e.g. one per GPU after an all-gather) with the
 * selection order of evaluate.py:404-409; records with block < 0 are "none".  This is the
 * deterministic "allreduce-argmax" step of multi-GPU evaluation. */
PP_API int pp_reduce_best(pp_ctx *ctx, const pp_best *records, int32_t n, pp_best *out, int32_t mem,
                          void *stream);
/* Linear expected-NPV table enpv[B][T] of the current scenario set:
 * factored = 0: disc[t]*mean_s(sig[s][t]*vmax[s][b]) - disc[t]*cost[b][t]  (colgen.py:187-204)
 * factored = 1: disc[t]*(mean_s(sig[s][t]*vmax[s][b]) - cost[b][t])        (hybrid.py:673-678,
 *               saa.py:65-69); sig = ones unless PP_USE_SIGMA. */
PP_API int pp_enpv_table(pp_ctx *ctx, uint32_t flags, int32_t factored, double *out, int32_t mem,
                         void *stream);
/* ---- host-native GA helpers (no device work, no context) -------------------------------- */
/* HybridSearch._mutate (hybrid.py:692-714) on assign[n_blocks] (int64, in place) over blocks[n_sel],
 * drawing from a numpy Generator(PCG64) stream supplied as raw 64-bit outputs raw[n_raw] plus the
 * bit generator's uint32 buffer (*has_u32, *uinteger; updated).  *consumed receives the number of raw
 * outputs used, so the caller can leave its Generator exactly where the reference's loop would.
 * CSR adjacency pred_ptr/pred_idx, succ_ptr/succ_idx as BlockModel.csr().  PP_ERR_SHAPE (assign
 * untouched) when raw runs out: retry with a longer block. */
PP_API int pp_host_mutate(int64_t *assign, int32_t n_blocks, const int64_t *blocks, int64_t n_sel,
                          const int32_t *pred_ptr, const int32_t *pred_idx, const int32_t *succ_ptr,
                          const int32_t *succ_idx, int32_t n_periods, double rate, const uint64_t *raw,
                          int64_t n_raw, int32_t *has_u32, uint32_t *uinteger, int64_t *consumed);

/* Topological level of every block (longest predecessor chain), host output. */
PP_API int pp_get_levels(pp_ctx *ctx, int32_t *n_levels, int32_t *level_of_block);

#ifdef __cplusplus
}
#endif
#endif /* PITPLAN_B200_H */
