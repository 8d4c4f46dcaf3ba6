/*
 * oracle.c -- CPU restatement of the pitplan move-evaluation hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links, loads or
 * calls this file; it is the checker used by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs.
 *
 * Every function restates one piece of the reference (paths are relative to
 * /root/reference/pkg/src/pitplan/) with the same IEEE-754 binary64 operation
 * order.  Build with -ffp-contract=off so no multiply-add is fused.
 *
 * Parity pinning: tests/golden/*.npz hold outputs of the reference itself run
 * in the build container (tests/golden/make_golden.py), and
 * tests/test_oracle_golden.py checks this file against them bit for bit.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define UNMINED (-1)

/* numpy's pairwise summation for float64 (numpy/_core/src/umath/loops_utils.h.src,
 * DOUBLE_pairwise_sum), which `ndarray.sum()` / `np.mean` use for a contiguous 1-D
 * reduction; the reduction starts from the additive identity 0.0, see or_np_sum. */
static double pairwise(const double *a, int64_t n) {
    if (n < 8) {
        double res = -0.0;
        for (int64_t i = 0; i < n; i++) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pairwise(a, n2) + pairwise(a + n2, n - n2);
    }
}

/* float(np.asarray(a).sum()) for a contiguous float64 vector. */
double or_np_sum(const double *a, int64_t n) { return 0.0 + pairwise(a, n); }

/* period_mass[t] = masses[assign == t].sum()   (evaluate.py:334-337, also
 * check_feasible evaluate.py:99-101): boolean-mask compaction in block order,
 * then numpy pairwise summation. */
void or_period_mass(int32_t B, int32_t T, const int32_t *assign, const double *mass, double *pm) {
    double *buf = (double *)malloc(sizeof(double) * (size_t)(B > 0 ? B : 1));
    for (int32_t t = 0; t < T; t++) {
        int64_t n = 0;
        for (int32_t b = 0; b < B; b++)
            if (assign[b] == t) buf[n++] = mass[b];
        pm[t] = or_np_sum(buf, n);
    }
    free(buf);
}

/* _unit_values (evaluate.py:291-303).  vmax is v.max(axis=2) laid out [S][B] as in
 * the reference.  s < 0 means s=None: v.max(axis=2).mean(axis=0), which numpy
 * evaluates as a sequential accumulation over the leading axis then / S. */
void or_unit_values(int32_t B, int32_t S, const double *vmax, int32_t s, int32_t literal,
                    const double *mass, double *unit) {
    for (int32_t b = 0; b < B; b++) {
        if (literal) {
            unit[b] = mass[b] * 100.0;
        } else if (s < 0) {
            double acc = 0.0;
            for (int32_t k = 0; k < S; k++) acc += vmax[(size_t)k * B + b];
            unit[b] = acc / (double)S;
        } else {
            unit[b] = vmax[(size_t)s * B + b];
        }
    }
}

/* sig_row (evaluate.py:348-353): ones | sigma.mean(axis=0) | sigma[s]. */
void or_sig_row(int32_t T, int32_t S, const double *sigma, int32_t s, double *sig_row) {
    for (int32_t t = 0; t < T; t++) {
        if (sigma == NULL) {
            sig_row[t] = 1.0;
        } else if (s < 0) {
            double acc = 0.0;
            for (int32_t k = 0; k < S; k++) acc += sigma[(size_t)k * T + t];
            sig_row[t] = acc / (double)S;
        } else {
            sig_row[t] = sigma[(size_t)s * T + t];
        }
    }
}

/* geological_consistency (uncertainty.py:185-191) for every block, with the
 * instance diameter of evaluate.py:342-344 passed in. */
void or_spatial(int32_t B, const double *alt, const double *strc, const double *dist, double w1,
                double w2, double w3, double diameter, double *out) {
    for (int32_t b = 0; b < B; b++) {
        double dn = 0.0;
        if (diameter > 0) {
            dn = dist[b] / diameter;
            if (1.0 < dn) dn = 1.0; /* Python min(x, 1.0) */
        }
        double raw = w1 * alt[b] + w2 * strc[b] + w3 * (1.0 - dn);
        double v = 0.5 + raw;
        /* np.clip(v, 0.5, 1.5) */
        if (v < 0.5) v = 0.5;
        if (v > 1.5) v = 1.5;
        out[b] = v;
    }
}

/* Precedence window of evaluate.py:361-372 for block b and period t. */
static inline int prec_ok(int32_t b, int32_t t, const int32_t *pp, const int32_t *pi,
                          const int32_t *sp, const int32_t *si, const int32_t *assign) {
    for (int32_t k = pp[b]; k < pp[b + 1]; k++) {
        int32_t tp = assign[pi[k]];
        if (tp == UNMINED || tp > t) return 0;
    }
    for (int32_t k = sp[b]; k < sp[b + 1]; k++) {
        int32_t tc = assign[si[k]];
        if (tc != UNMINED && tc < t) return 0;
    }
    return 1;
}

/* `better` (evaluate.py:404-409) restricted to feasible moves. */
static inline int better(double v_new, int32_t b_new, int32_t t_new, double v_old, int32_t b_old,
                         int32_t t_old) {
    if (v_new > v_old) return 1;
    if (v_new == v_old && (b_new < b_old || (b_new == b_old && t_new < t_old))) return 1;
    return 0;
}

/* evaluate_candidates_parallel (evaluate.py:306-430) given the per-call tables
 * (period_mass, unit, discount, spatial, sig_row, optional mining cost [B][T]).
 * Outputs per candidate in input order; optional per-(candidate, period) trace
 * (value, feasible) laid out [C][T]; global best with the (value desc, block asc,
 * period asc) order, g_block = -1 when no candidate is feasible.
 * nthreads > 1 splits candidates over OpenMP threads; the result is independent
 * of it (as worker_count is in the reference). */
void or_eval_candidates(int32_t B, int32_t T, const int32_t *pp, const int32_t *pi,
                        const int32_t *sp, const int32_t *si, const double *mass,
                        const double *cap, const double *disc, const double *spatial,
                        const double *unit, const double *sig_row, const double *cost,
                        const int32_t *assign, const double *pm, const int32_t *cand, int32_t C,
                        int32_t *best_t, double *best_val, uint8_t *feas, double *trace_val,
                        uint8_t *trace_feas, double *g_val, int32_t *g_block, int32_t *g_period,
                        int32_t nthreads) {
    (void)B;
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(static) num_threads(nthreads)
#endif
    for (int32_t i = 0; i < C; i++) {
        int32_t b = cand[i];
        int32_t ab = assign[b];
        double own = (ab != UNMINED) ? mass[b] : 0.0;
        double bv = -INFINITY;
        int32_t bt = -1;
        for (int32_t t = 0; t < T; t++) {
            int ok = prec_ok(b, t, pp, pi, sp, si, assign);
            if (ok) {
                double load = pm[t] + mass[b];
                if (ab == t) load -= own;
                if (load > cap[t]) ok = 0;
            }
            double value;
            if (ok) {
                value = unit[b] * disc[t] * sig_row[t] * spatial[b];
                if (cost != NULL) value -= disc[t] * cost[(size_t)b * T + t];
            } else {
                value = -INFINITY;
            }
            if (trace_val) trace_val[(size_t)i * T + t] = value;
            if (trace_feas) trace_feas[(size_t)i * T + t] = (uint8_t)ok;
            if (ok && value > bv) {
                bv = value;
                bt = t;
            }
        }
        best_t[i] = bt;
        best_val[i] = bv;
        feas[i] = (uint8_t)(bt >= 0);
    }
    double gv = -INFINITY;
    int32_t gb = -1, gt = -1;
    for (int32_t i = 0; i < C; i++) {
        if (!feas[i]) continue;
        if (gb < 0 || better(best_val[i], cand[i], best_t[i], gv, gb, gt)) {
            gv = best_val[i];
            gb = cand[i];
            gt = best_t[i];
        }
    }
    *g_val = gv;
    *g_block = gb;
    *g_period = gt;
}

/* ---- per-scenario / expected / risk-adjusted move value ------------------------
 * Per-scenario value of block b in period t under scenario s: the kernel value of
 * evaluate.py:380-382 evaluated with s=k (unit = vmax[k][b], sig_row = sigma[k]):
 *     val_s(b,t) = ((vmax[s][b] * disc[t]) * sigma[s][t]) * spatial[b]  [- disc[t]*cost[b][t]]
 * Move delta:  d_s = val_s(b,t_new) - val_s(b,t_old)   (t_old = UNMINED contributes 0).
 * Expected delta: np.mean of the per-move vector d_0..d_{S-1} (pairwise sum / S).
 * Risk-adjusted: CVaR10 of d_s, the mean of the ceil(0.1 S) smallest values
 * (saa.py:150-166 risk_metrics: np.sort then srt[:k].mean()).
 */
static inline double val_s(const double *vmax, const double *sigma, const double *disc,
                           const double *spatial, const double *cost, int32_t B, int32_t T,
                           int32_t s, int32_t b, int32_t t) {
    double sg = sigma ? sigma[(size_t)s * T + t] : 1.0;
    double v = vmax[(size_t)s * B + b] * disc[t] * sg * spatial[b];
    if (cost != NULL) v -= disc[t] * cost[(size_t)b * T + t];
    return v;
}

static int cmp_double(const void *x, const void *y) {
    double a = *(const double *)x, b = *(const double *)y;
    return (a > b) - (a < b);
}

static void scen_stats(int32_t B, int32_t T, int32_t S, const double *vmax, const double *sigma,
                       const double *disc, const double *spatial, const double *cost, int32_t b,
                       int32_t t_new, int32_t t_old, int32_t cvar_k, double *tmp,
                       double *exp_out, double *cvar_out, float *scen_out, int64_t scen_stride) {
    for (int32_t s = 0; s < S; s++) {
        double d = 0.0;
        if (t_new != UNMINED) d = val_s(vmax, sigma, disc, spatial, cost, B, T, s, b, t_new);
        if (t_old != UNMINED) d = d - val_s(vmax, sigma, disc, spatial, cost, B, T, s, b, t_old);
        tmp[s] = d;
        if (scen_out) scen_out[(int64_t)s * scen_stride] = (float)d;
    }
    if (exp_out) *exp_out = or_np_sum(tmp, S) / (double)S;
    if (cvar_out) {
        qsort(tmp, (size_t)S, sizeof(double), cmp_double);
        *cvar_out = or_np_sum(tmp, cvar_k) / (double)cvar_k;
    }
}

/* Candidate-mode statistics: for each candidate i and period t, the expected and
 * CVaR delta of moving candidate b = cand[i] from its current period to t;
 * per-scenario deltas (float32) laid out [C][S][T].  Infeasible (i, t) entries
 * (trace_feas == 0) get -inf everywhere. */
void or_candidate_stats(int32_t B, int32_t T, int32_t S, const double *vmax, const double *sigma,
                        const double *disc, const double *spatial, const double *cost,
                        const int32_t *assign, const int32_t *cand, int32_t C,
                        const uint8_t *trace_feas, int32_t cvar_k, double *exp_delta,
                        double *cvar, float *scen_delta, int32_t nthreads) {
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel num_threads(nthreads)
#endif
    {
        double *tmp = (double *)malloc(sizeof(double) * (size_t)(S > 0 ? S : 1));
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
        for (int32_t i = 0; i < C; i++) {
            int32_t b = cand[i];
            for (int32_t t = 0; t < T; t++) {
                size_t m = (size_t)i * T + t;
                float *so = scen_delta ? scen_delta + (size_t)i * S * T + t : NULL;
                if (!trace_feas[m]) {
                    if (exp_delta) exp_delta[m] = -INFINITY;
                    if (cvar) cvar[m] = -INFINITY;
                    if (so)
                        for (int32_t s = 0; s < S; s++) so[(size_t)s * T] = -INFINITY;
                    continue;
                }
                scen_stats(B, T, S, vmax, sigma, disc, spatial, cost, b, t, assign[b], cvar_k, tmp,
                           exp_delta ? exp_delta + m : NULL, cvar ? cvar + m : NULL, so, T);
            }
        }
        free(tmp);
    }
}

/* check_feasible (evaluate.py:82-105). */
void or_check_feasible(int32_t B, int32_t T, const int32_t *pp, const int32_t *pi,
                       const double *mass, const double *cap, const int32_t *assign,
                       int64_t *pred_count, double *excess, double *violation) {
    int64_t cnt = 0;
    for (int32_t j = 0; j < B; j++) {
        int32_t tj = assign[j];
        if (tj == UNMINED) continue;
        for (int32_t k = pp[j]; k < pp[j + 1]; k++) {
            int32_t ti = assign[pi[k]];
            if (ti == UNMINED || ti > tj) cnt++;
        }
    }
    double *pm = (double *)malloc(sizeof(double) * (size_t)(T > 0 ? T : 1));
    or_period_mass(B, T, assign, mass, pm);
    double ex = 0.0;
    for (int32_t t = 0; t < T; t++) {
        double d = pm[t] - cap[t];
        ex += (d > 0.0) ? d : 0.0; /* max(0.0, load - cap) */
    }
    free(pm);
    double mean_cap = or_np_sum(cap, T) / (double)T;
    *pred_count = cnt;
    *excess = ex;
    *violation = (double)cnt + ex / mean_cap;
}

/* Kahn topological order with a sorted ready queue (blockmodel.py:228-245).
 * Returns 0 on success, -1 on a cycle. */
int or_topological_order(int32_t B, const int32_t *pp, const int32_t *sp, const int32_t *si,
                         int32_t *order) {
    int32_t *indeg = (int32_t *)malloc(sizeof(int32_t) * (size_t)(B > 0 ? B : 1));
    int32_t *heap = (int32_t *)malloc(sizeof(int32_t) * (size_t)(B > 0 ? B : 1));
    int32_t hn = 0, n = 0;
    for (int32_t b = 0; b < B; b++) indeg[b] = pp[b + 1] - pp[b];
    /* binary min-heap == "pop(0) of a sorted list" */
#define HPUSH(x)                                                                 \
    do {                                                                         \
        int32_t _i = hn++;                                                       \
        heap[_i] = (x);                                                          \
        while (_i > 0 && heap[(_i - 1) / 2] > heap[_i]) {                        \
            int32_t _p = (_i - 1) / 2, _t = heap[_p];                            \
            heap[_p] = heap[_i];                                                 \
            heap[_i] = _t;                                                       \
            _i = _p;                                                             \
        }                                                                        \
    } while (0)
    for (int32_t b = 0; b < B; b++)
        if (indeg[b] == 0) HPUSH(b);
    while (hn > 0) {
        int32_t top = heap[0];
        heap[0] = heap[--hn];
        int32_t i = 0;
        for (;;) {
            int32_t l = 2 * i + 1, r = l + 1, m = i;
            if (l < hn && heap[l] < heap[m]) m = l;
            if (r < hn && heap[r] < heap[m]) m = r;
            if (m == i) break;
            int32_t tt = heap[m];
            heap[m] = heap[i];
            heap[i] = tt;
            i = m;
        }
        order[n++] = top;
        for (int32_t k = sp[top]; k < sp[top + 1]; k++)
            if (--indeg[si[k]] == 0) HPUSH(si[k]);
    }
#undef HPUSH
    free(indeg);
    free(heap);
    return n == B ? 0 : -1;
}

/* _precedence_repair_pass (hybrid.py:493-510): in-place topological sweep. */
void or_precedence_repair(int32_t B, const int32_t *pp, const int32_t *pi, const int32_t *order,
                          int32_t *assign) {
    for (int32_t k = 0; k < B; k++) {
        int32_t b = order[k];
        int32_t t = assign[b];
        if (t == UNMINED) continue;
        int32_t t_min = 0, ok = 1;
        for (int32_t e = pp[b]; e < pp[b + 1]; e++) {
            int32_t tp = assign[pi[e]];
            if (tp == UNMINED) {
                ok = 0;
                break;
            }
            if (tp > t_min) t_min = tp;
        }
        if (!ok)
            assign[b] = UNMINED;
        else if (t < t_min)
            assign[b] = t_min;
    }
}

/* lns_repair unmine fixpoint (hybrid.py:199-211): sweep the precedence edge list
 * (i must be mined no later than j) until nothing changes.  unmined_out[j] = 1
 * for every block this step unmined (the additions to the repair pool). */
void or_unmine_fixpoint(int32_t B, int64_t E, const int32_t *ei, const int32_t *ej,
                        int32_t *assign, uint8_t *unmined_out) {
    if (unmined_out) memset(unmined_out, 0, (size_t)B);
    int changed = 1;
    while (changed) {
        changed = 0;
        for (int64_t e = 0; e < E; e++) {
            int32_t tj = assign[ej[e]];
            if (tj == UNMINED) continue;
            int32_t ti = assign[ei[e]];
            if (ti == UNMINED || ti > tj) {
                assign[ej[e]] = UNMINED;
                if (unmined_out) unmined_out[ej[e]] = 1;
                changed = 1;
            }
        }
    }
}

/* ---- over-capacity ejection: lns_repair's destroy step (hybrid.py:213-235) -------
 * mean_grade = scenarios.grades.mean(axis=0) (hybrid.py:214).  For each period t in order:
 * load = masses[mined_in(t)].sum() (numpy pairwise, hybrid.py:217); target = cap[t], or
 * cap[t] * (1 - destroy_fraction) when destroy_fraction > 0 and load > cap[t] (218-221);
 * nothing happens when load <= target (222-223).  Otherwise the blocks of t whose successors
 * are all UNMINED (224-228; evaluated before any ejection in t) are sorted by
 * (mean_grade[b] * masses[b], b) (229) and unmined in that order, load -= masses[b] after
 * each, while load > target (230-235).  Ejections in t never change the candidate list of a
 * later period after the unmine fixpoint (successors are mined no earlier than their
 * predecessors), but this restatement simply follows the reference order.  ejected_out[b] = 1
 * for every ejected block (the additions to the repair pool). */
typedef struct {
    double key;
    int32_t b;
} or_ekey;
static int or_ekey_cmp(const void *x, const void *y) {
    const or_ekey *a = (const or_ekey *)x, *b = (const or_ekey *)y;
    if (a->key < b->key) return -1;
    if (a->key > b->key) return 1;
    return (a->b > b->b) - (a->b < b->b);
}
void or_eject(int32_t B, int32_t T, const int32_t *succ_ptr, const int32_t *succ_idx, const double *mass,
              const double *cap, const double *mean_grade, double destroy_fraction, int32_t *assign,
              uint8_t *ejected_out) {
    if (ejected_out) memset(ejected_out, 0, (size_t)B);
    double *buf = (double *)malloc(sizeof(double) * (size_t)(B > 0 ? B : 1));
    or_ekey *ej = (or_ekey *)malloc(sizeof(or_ekey) * (size_t)(B > 0 ? B : 1));
    for (int32_t t = 0; t < T; t++) {
        int64_t n = 0;
        for (int32_t b = 0; b < B; b++)
            if (assign[b] == t) buf[n++] = mass[b];
        double load = or_np_sum(buf, n);
        double target = cap[t];
        if (destroy_fraction > 0 && load > cap[t]) target = cap[t] * (1.0 - destroy_fraction);
        if (load <= target) continue;
        int64_t ne = 0;
        for (int32_t b = 0; b < B; b++) {
            if (assign[b] != t) continue;
            int ok = 1;
            for (int32_t k = succ_ptr[b]; k < succ_ptr[b + 1] && ok; k++) ok = assign[succ_idx[k]] == UNMINED;
            if (ok) {
                ej[ne].key = mean_grade[b] * mass[b];
                ej[ne].b = b;
                ne++;
            }
        }
        qsort(ej, (size_t)ne, sizeof(or_ekey), or_ekey_cmp);
        for (int64_t k = 0; k < ne; k++) {
            if (load <= target) break;
            assign[ej[k].b] = UNMINED;
            if (ejected_out) ejected_out[ej[k].b] = 1;
            load -= mass[ej[k].b];
        }
    }
    free(buf);
    free(ej);
}

/* ---- colgen.price_column's sequence greedy (colgen.py:236-254), literally: per period, scan
 * blocks in id order; skip blocks in the column or over the period's capacity
 * (`masses[b] + load > cap`), skip blocks with a predecessor outside the column or at a later
 * period; every remaining block is one expansion and becomes the pick when its score exceeds
 * best + 1e-12 (best starts at 0.0).  The loop for a period stops when a scan picks nothing;
 * scans start only while expansions < node_cap.  score is [B][T]. ---- */
int64_t or_price_greedy(int32_t B, int32_t T, const int32_t *pred_ptr, const int32_t *pred_idx, const double *mass,
                        const double *score, const double *cap, int64_t node_cap, int32_t *assign) {
    int64_t expansions = 0;
    for (int32_t b = 0; b < B; b++) assign[b] = UNMINED;
    for (int32_t t = 0; t < T; t++) {
        double load = 0.0;
        while (expansions < node_cap) {
            int32_t best_b = -1;
            double best_s = 0.0;
            for (int32_t b = 0; b < B; b++) {
                if (assign[b] != UNMINED || mass[b] + load > cap[t]) continue;
                int ok = 1;
                for (int32_t k = pred_ptr[b]; k < pred_ptr[b + 1] && ok; k++) {
                    const int32_t tp = assign[pred_idx[k]];
                    ok = tp != UNMINED && tp <= t;
                }
                if (!ok) continue;
                expansions++;
                if (score[(size_t)b * T + t] > best_s + 1e-12) {
                    best_b = b;
                    best_s = score[(size_t)b * T + t];
                }
            }
            if (best_b < 0) break;
            assign[best_b] = t;
            load += mass[best_b];
        }
    }
    return expansions;
}

/* ---- relaxed NPV: ScheduleEvaluator.npv_relaxed / per_scenario_npv, single-mode fast path ----
 * stage-2 (evaluate.py:166-183): blocks of period t sorted by density = v[s,b,0] / m[b] with
 * np.argsort(-density, kind="stable") (ties keep block order); greedy: while density > 0 and
 * hours_left > 0: take = min(m, hours_left * rate); total += density * take;
 * hours_left -= take / rate.  _npv (evaluate.py:222-234): total -= disc[t] * costs[mined, t].sum()
 * (numpy pairwise), then total += disc[t] * sigma[s,t] * raw / n_s for s in order;
 * per_scenario_npv (248-258): out[s] += disc[t] * sigma[s,t] * raw - disc[t] * costsum. */
typedef struct {
    double d;
    int32_t k;
} or_dens;
static int or_dens_cmp(const void *x, const void *y) {
    const or_dens *a = (const or_dens *)x, *b = (const or_dens *)y;
    const double na = -a->d, nb = -b->d;
    if (na < nb) return -1;
    if (na > nb) return 1;
    return (a->k > b->k) - (a->k < b->k);
}
static double or_stage2_fast(int64_t n, const int32_t *ids, const double *vrow_s, const double *mass, double hours,
                             double rate, or_dens *buf) {
    for (int64_t k = 0; k < n; k++) {
        buf[k].d = vrow_s[ids[k]] / mass[ids[k]];
        buf[k].k = (int32_t)k;
    }
    qsort(buf, (size_t)n, sizeof(or_dens), or_dens_cmp);
    double hours_left = hours, total = 0.0;
    for (int64_t k = 0; k < n; k++) {
        const double d = buf[k].d;
        if (d <= 0 || hours_left <= 0) break;
        const double m = mass[ids[buf[k].k]];
        const double hr = hours_left * rate;
        const double take = (hr < m) ? hr : m;
        total += d * take;
        hours_left -= take / rate;
    }
    return total;
}
void or_npv_relaxed(int32_t B, int32_t T, int32_t S, const int32_t *assign, const double *mass, const double *cost,
                    const double *vmax_sb, const double *sigma_st, const double *disc, const double *plant_hours,
                    double rate, double *npv_out, double *per_scen_out) {
    int32_t *ids = (int32_t *)malloc(sizeof(int32_t) * (size_t)(B > 0 ? B : 1));
    double *buf = (double *)malloc(sizeof(double) * (size_t)(B > 0 ? B : 1));
    or_dens *db = (or_dens *)malloc(sizeof(or_dens) * (size_t)(B > 0 ? B : 1));
    double total = 0.0;
    if (per_scen_out)
        for (int32_t s = 0; s < S; s++) per_scen_out[s] = 0.0;
    for (int32_t t = 0; t < T; t++) {
        int64_t n = 0;
        for (int32_t b = 0; b < B; b++)
            if (assign[b] == t) ids[n++] = b;
        double costv = 0.0;
        if (n) {
            for (int64_t k = 0; k < n; k++) buf[k] = cost[(size_t)ids[k] * T + t];
            const double csum = or_np_sum(buf, n);
            total -= disc[t] * csum;
            costv = disc[t] * csum;
        }
        for (int32_t s = 0; s < S; s++) {
            const double raw = n ? or_stage2_fast(n, ids, vmax_sb + (size_t)s * B, mass, plant_hours[t], rate, db) : 0.0;
            const double sg = sigma_st ? sigma_st[(size_t)s * T + t] : 1.0;
            total += disc[t] * sg * raw / S;
            if (per_scen_out) per_scen_out[s] += disc[t] * sg * raw - costv;
        }
    }
    *npv_out = total;
    free(ids);
    free(buf);
    free(db);
}

/* ---- explicit moves (reassign / unmine / swap) ---------------------------------
 * Reassign move (b, t_new), t_old = assign[b]:
 *   t_new == t_old                 -> not a move (infeasible), as polish skips t == orig
 *                                     (hybrid.py:369-370)
 *   t_new == UNMINED               -> feasible iff mined and no mined successor
 *                                     (hybrid.py:362-367)
 *   t_new >= 0                     -> precedence window of evaluate.py:361-372 and the
 *                                     capacity test (pm[t] + m) > cap (evaluate.py:373-378)
 *   delta = val(b,t_new) - val(b,t_old), val from evaluate.py:380-382, val(UNMINED) = 0.
 * Swap (b1, b2) with t1 = assign[b1], t2 = assign[b2] both mined and different:
 *   capacity  ((pm[t1] - m1) + m2) <= cap[t1] and ((pm[t2] - m2) + m1) <= cap[t2]
 *   (hybrid.py:396-399), windows re-evaluated with the swap applied (hybrid.py:400-403),
 *   delta = (val(b1,t2) - val(b1,t1)) + (val(b2,t1) - val(b2,t2)).
 * Best: feasible move with the largest delta, lowest move index on ties. */
static inline double kval(const double *unit, const double *disc, const double *sig_row,
                          const double *spatial, const double *cost, int32_t T, int32_t b,
                          int32_t t) {
    double v = unit[b] * disc[t] * sig_row[t] * spatial[b];
    if (cost != NULL) v -= disc[t] * cost[(size_t)b * T + t];
    return v;
}

/* window(b) of hybrid.py:348-355 with an optional override of one block's period. */
static inline void window(int32_t b, const int32_t *pp, const int32_t *pi, const int32_t *sp,
                          const int32_t *si, const int32_t *assign, int32_t T, int32_t ob,
                          int32_t ot, int32_t *lo, int32_t *hi) {
    int32_t l = 0, h = T - 1, none = 0;
    for (int32_t k = pp[b]; k < pp[b + 1]; k++) {
        int32_t p = pi[k];
        int32_t tp = (p == ob) ? ot : assign[p];
        if (tp == UNMINED) none = 1;
        else if (tp > l) l = tp;
    }
    for (int32_t k = sp[b]; k < sp[b + 1]; k++) {
        int32_t c = si[k];
        int32_t tc = (c == ob) ? ot : assign[c];
        if (tc != UNMINED && tc < h) h = tc;
    }
    *lo = none ? -2 : l; /* -2 encodes "None" */
    *hi = h;
}

void or_eval_moves(int32_t B, int32_t T, int32_t S, const int32_t *pp, const int32_t *pi,
                   const int32_t *sp, const int32_t *si, const double *mass, const double *cap,
                   const double *disc, const double *spatial, const double *unit,
                   const double *sig_row, const double *cost, const double *vmax,
                   const double *sigma, const int32_t *assign, const double *pm,
                   const int32_t *mv_a, const int32_t *mv_b, int32_t M, int32_t is_swap,
                   int32_t cvar_k, uint8_t *feas, double *delta, double *exp_delta, double *cvar,
                   float *scen_delta, double *g_val, int32_t *g_index, int32_t nthreads) {
    (void)B;
#ifdef _OPENMP
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel num_threads(nthreads)
#endif
    {
        double *tmp = (double *)malloc(sizeof(double) * (size_t)(S > 0 ? S : 1));
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
        for (int32_t i = 0; i < M; i++) {
            int ok = 0;
            double d = -INFINITY;
            if (!is_swap) {
                int32_t b = mv_a[i], tn = mv_b[i], to = assign[b];
                if (tn == to) {
                    ok = 0;
                } else if (tn == UNMINED) {
                    ok = 1;
                    for (int32_t k = sp[b]; k < sp[b + 1]; k++)
                        if (assign[si[k]] != UNMINED) ok = 0;
                } else {
                    ok = prec_ok(b, tn, pp, pi, sp, si, assign);
                    if (ok) {
                        double load = pm[tn] + mass[b];
                        if (load > cap[tn]) ok = 0;
                    }
                }
                if (ok) {
                    double vn = (tn != UNMINED) ? kval(unit, disc, sig_row, spatial, cost, T, b, tn) : 0.0;
                    double vo = (to != UNMINED) ? kval(unit, disc, sig_row, spatial, cost, T, b, to) : 0.0;
                    d = vn - vo;
                    if (vmax && S > 0)
                        scen_stats(B, T, S, vmax, sigma, disc, spatial, cost, b, tn, to, cvar_k, tmp,
                                   exp_delta ? exp_delta + i : NULL, cvar ? cvar + i : NULL,
                                   scen_delta ? scen_delta + (size_t)i * S : NULL, 1);
                }
            } else {
                int32_t b1 = mv_a[i], b2 = mv_b[i];
                int32_t t1 = assign[b1], t2 = assign[b2];
                if (b1 != b2 && t1 != UNMINED && t2 != UNMINED && t1 != t2) {
                    double l1 = pm[t1] - mass[b1] + mass[b2];
                    double l2 = pm[t2] - mass[b2] + mass[b1];
                    if (!(l1 > cap[t1]) && !(l2 > cap[t2])) {
                        int32_t lo1, hi1, lo2, hi2;
                        window(b1, pp, pi, sp, si, assign, T, b2, t1, &lo1, &hi1);
                        window(b2, pp, pi, sp, si, assign, T, b1, t2, &lo2, &hi2);
                        ok = lo1 != -2 && lo1 <= t2 && t2 <= hi1 && lo2 != -2 && lo2 <= t1 && t1 <= hi2;
                    }
                }
                if (ok) {
                    double v12 = kval(unit, disc, sig_row, spatial, cost, T, b1, t2);
                    double v11 = kval(unit, disc, sig_row, spatial, cost, T, b1, t1);
                    double v21 = kval(unit, disc, sig_row, spatial, cost, T, b2, t1);
                    double v22 = kval(unit, disc, sig_row, spatial, cost, T, b2, t2);
                    d = (v12 - v11) + (v21 - v22);
                    if (vmax && S > 0) {
                        for (int32_t s = 0; s < S; s++) {
                            double a1 = val_s(vmax, sigma, disc, spatial, cost, B, T, s, b1, t2) -
                                        val_s(vmax, sigma, disc, spatial, cost, B, T, s, b1, t1);
                            double a2 = val_s(vmax, sigma, disc, spatial, cost, B, T, s, b2, t1) -
                                        val_s(vmax, sigma, disc, spatial, cost, B, T, s, b2, t2);
                            double ds = a1 + a2;
                            tmp[s] = ds;
                            if (scen_delta) scen_delta[(size_t)i * S + s] = (float)ds;
                        }
                        if (exp_delta) exp_delta[i] = or_np_sum(tmp, S) / (double)S;
                        if (cvar) {
                            qsort(tmp, (size_t)S, sizeof(double), cmp_double);
                            cvar[i] = or_np_sum(tmp, cvar_k) / (double)cvar_k;
                        }
                    }
                }
            }
            feas[i] = (uint8_t)ok;
            delta[i] = d;
            if (!ok && vmax && S > 0) {
                if (exp_delta) exp_delta[i] = -INFINITY;
                if (cvar) cvar[i] = -INFINITY;
                if (scen_delta)
                    for (int32_t s = 0; s < S; s++) scen_delta[(size_t)i * S + s] = -INFINITY;
            }
        }
        free(tmp);
    }
    double gv = -INFINITY;
    int32_t gi = -1;
    for (int32_t i = 0; i < M; i++) {
        if (!feas[i]) continue;
        if (gi < 0 || delta[i] > gv) {
            gv = delta[i];
            gi = i;
        }
    }
    *g_val = gv;
    *g_index = gi;
}

/* Linear ENPV table, [B][T]:
 *   factored = 0: disc[t] * mean_s(sig[s][t] * v[s][b]) - disc[t] * cost[b][t]   (colgen.py:187-204)
 *   factored = 1: disc[t] * (mean_s(sig[s][t] * v[s][b]) - cost[b][t])           (hybrid.py:673-678)
 * mean_s = numpy .mean(axis=0) of the [S][B] product array: sequential in s, then / S. */
void or_enpv_table(int32_t B, int32_t T, int32_t S, const double *vmax, const double *sigma,
                   const double *disc, const double *cost, int32_t factored, double *out) {
    for (int32_t b = 0; b < B; b++) {
        for (int32_t t = 0; t < T; t++) {
            double acc = 0.0;
            for (int32_t s = 0; s < S; s++) {
                double sg = sigma ? sigma[(size_t)s * T + t] : 1.0;
                acc += sg * vmax[(size_t)s * B + b];
            }
            double mean = acc / (double)S;
            double c = cost[(size_t)b * T + t];
            out[(size_t)b * T + t] = factored ? disc[t] * (mean - c) : disc[t] * mean - disc[t] * c;
        }
    }
}
