/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into, loaded by, or
 * called from the product path (paper_2401_07886_b200/).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may use it, and
 * only as the checker / CPU baseline.
 *
 * Plain-C scalar restatement of the reference's greedy-rollout hot path:
 *
 *   run_eval loop          pkg/src/besteffort/evalkit.py:154-209
 *   ClusterSim.submit      pkg/src/besteffort/simcore.py:94-111
 *   ClusterSim.advance     pkg/src/besteffort/simcore.py:113-149
 *   ClusterSim.observe     pkg/src/besteffort/simcore.py:155-157
 *   RateEstimator          pkg/src/besteffort/workload.py:212-255
 *   encode                 pkg/src/besteffort/policy.py:52-65
 *   QNetwork.forward       pkg/src/besteffort/policy.py:111-118
 *   argmax (first max)     pkg/src/besteffort/evalkit.py:201
 *   request_reward         pkg/src/besteffort/reward.py:94-126
 *
 * The reference keeps one global event heap; events of different replicas
 * never interact (a replica's events only touch its own active/queue), so
 * this restatement advances every replica independently with the exact same
 * per-replica event order: END before START at equal times, an END exactly at
 * the horizon is processed, a START exactly at the horizon stays pending
 * (simcore.py:18, :120).  Completions are identified by request id, so the
 * cross-replica completion order (which differs from the heap's) does not
 * affect any rollout output (records are indexed by id, evalkit.py:178-183).
 *
 * Float semantics are kept literally: end time = (t + alpha) + (beta * n)
 * with no contraction (simcore.py:146; build with -ffp-contract=off),
 * realized = (t - arrival) / tokens (simcore.py:135), estimator
 * 1 / max(((w[-1]-w[0]) / (n-1)) / 1000, 1e-6) (workload.py:246-247).
 *
 * Parity: pinned against golden records produced by the reference itself
 * (tests/golden/make_golden.py) and against the reference's known-answer
 * tests (pkg/tests/test_simcore.py:24-139), see tests/test_oracle_golden.py.
 * The Q-network sums in plain sequential order; the reference's OpenBLAS
 * order is not reproducible, so routing decisions are
 * compared tie-aware.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define K_NONE 0
#define K_START 1
#define K_END 2

typedef struct {
    double arrival;
    int32_t id;
    int32_t task;
    int64_t join; /* iteration count at the START that first included it; -1 = not running */
} slot_t;

typedef struct {
    slot_t* buf;
    int64_t cap, head, count; /* FIFO = active (first min(count,max_batch)) ++ queue */
    int64_t n_running;        /* prefix of the FIFO that joined an iteration */
    int kind;
    double t;
    int64_t iters; /* END events so far */
} replica_t;

typedef struct {
    int replicas;
    double alpha, beta;
    int max_batch, tokens;
} or_tier_t;

static void fifo_push(replica_t* r, slot_t s) {
    if (r->count == r->cap) {
        int64_t ncap = r->cap ? r->cap * 2 : 64;
        slot_t* nb = (slot_t*)malloc(sizeof(slot_t) * (size_t)ncap);
        for (int64_t k = 0; k < r->count; ++k) nb[k] = r->buf[(r->head + k) % r->cap];
        free(r->buf);
        r->buf = nb;
        r->cap = ncap;
        r->head = 0;
    }
    r->buf[(r->head + r->count) % r->cap] = s;
    r->count++;
}

static slot_t* fifo_at(replica_t* r, int64_t k) { return &r->buf[(r->head + k) % r->cap]; }

typedef struct {
    int T, M;
    const double* deadline;
    const int32_t* soft;
    const double* matrix;
    double decay, cutoff;
    uint8_t* tier_out;
    double* reward_out;
    double* realized_out;
} scorer_t;

/* reward.py:94-126 */
static double score(const scorer_t* sc, int task, int tier, double realized) {
    double dl = sc->deadline[task];
    double w;
    if (!sc->soft[task]) {
        w = realized <= dl ? 1.0 : 0.0;
    } else {
        double excess = realized - dl;
        if (excess <= 0) w = 1.0;
        else if (excess <= sc->cutoff * dl) {
            volatile double prod = sc->decay * excess; /* rounded before the subtract */
            double v = 1.0 - prod;
            w = v > 0.0 ? v : 0.0;
        } else w = 0.0;
    }
    return w * sc->matrix[task * sc->M + tier];
}

/* One replica's share of ClusterSim.advance (simcore.py:113-149). */
static void advance_replica(replica_t* r, const or_tier_t* spec, int tier, double until,
                            const scorer_t* sc) {
    while (r->kind != K_NONE) {
        if (r->kind == K_START) {
            if (!(r->t < until)) break; /* START exactly at the horizon stays pending */
            int64_t n_active = r->count < spec->max_batch ? r->count : spec->max_batch;
            for (int64_t k = r->n_running; k < n_active; ++k) fifo_at(r, k)->join = r->iters;
            r->n_running = n_active;
            volatile double a = r->t + spec->alpha;
            volatile double b = spec->beta * (double)n_active;
            r->t = a + b; /* (time + alpha) + beta * len(members), simcore.py:146 */
            r->kind = K_END;
        } else {
            if (!(r->t <= until)) break;
            r->iters++;
            while (r->n_running > 0) {
                slot_t* h = fifo_at(r, 0);
                if (r->iters - h->join < spec->tokens) break;
                double realized = (r->t - h->arrival) / (double)spec->tokens;
                int id = h->id;
                sc->tier_out[id] = (uint8_t)tier;
                sc->reward_out[id] = score(sc, h->task, tier, realized);
                if (sc->realized_out) sc->realized_out[id] = realized;
                r->head = (r->head + 1) % r->cap;
                r->count--;
                r->n_running--;
            }
            int64_t n_active = r->count < spec->max_batch ? r->count : spec->max_batch;
            r->kind = n_active > 0 ? K_START : K_NONE; /* START at the same time */
        }
    }
}

/*
 * Returns 0 on success, -1 on invalid input.
 * Policy: w1 [D x H] row-major, b1 [H], w2 [H x M], b2 [M]; D = T + M + 1.
 * static_tier >= 0 routes everything to that tier; forced_actions (nullable)
 * overrides both.  seg_start/seg_rate: the trace's SegmentMarks.
 */
int oracle_run_eval(int M, const or_tier_t* tiers, int T, const double* deadline,
                    const int32_t* soft, const double* matrix, double decay, double cutoff,
                    const double* enc_scales, double rate_scale, const double* w1,
                    const double* b1, const double* w2, const double* b2, int hidden,
                    int static_tier, const uint8_t* forced_actions, int64_t N,
                    const double* arrival, const uint8_t* task, int64_t S,
                    const int64_t* seg_start, const double* seg_rate, int estimator_true_rate,
                    double prior_rate, int reset_between_segments, uint8_t* tier_out,
                    double* reward_out, double* realized_out, int32_t* obs_out,
                    double* rate_out, double* q_out) {
    if (M < 1 || T < 1) return -1;
    int R = 0;
    int base[64];
    for (int m = 0; m < M; ++m) {
        base[m] = R;
        R += tiers[m].replicas;
    }
    replica_t* reps = (replica_t*)calloc((size_t)R, sizeof(replica_t));
    scorer_t sc = {T, M, deadline, soft, matrix, decay, cutoff, tier_out, reward_out, realized_out};
    int D = T + M + 1;
    double* x = (double*)malloc(sizeof(double) * (size_t)D);
    double* h = (double*)malloc(sizeof(double) * (size_t)(hidden > 0 ? hidden : 1));
    double q[64];
    double win[5];
    int wn = 0;
    int64_t seg = 0;
    double cur_rate = NAN;

    for (int64_t i = 0; i < N; ++i) {
        /* segment boundaries (evalkit.py:186-192) */
        while (seg < S && i >= seg_start[seg]) {
            if (reset_between_segments && i == seg_start[seg] && i > 0) {
                for (int m = 0; m < M; ++m)
                    for (int rr = 0; rr < tiers[m].replicas; ++rr)
                        advance_replica(&reps[base[m] + rr], &tiers[m], m, INFINITY, &sc);
                for (int k = 0; k < R; ++k) {
                    free(reps[k].buf);
                    memset(&reps[k], 0, sizeof(replica_t));
                }
                wn = 0;
            }
            cur_rate = seg_rate[seg];
            seg++;
        }
        double t_arr = arrival[i];
        for (int m = 0; m < M; ++m)
            for (int rr = 0; rr < tiers[m].replicas; ++rr)
                advance_replica(&reps[base[m] + rr], &tiers[m], m, t_arr, &sc);
        /* RateEstimator.observe (workload.py:234-247) */
        if (wn == 5) {
            memmove(win, win + 1, sizeof(double) * 4);
            wn = 4;
        }
        win[wn++] = t_arr;
        double rate;
        if (estimator_true_rate) rate = cur_rate;
        else if (wn < 2) rate = prior_rate;
        else {
            double gap = ((win[wn - 1] - win[0]) / (double)(wn - 1)) / 1000.0;
            rate = 1.0 / (gap > 1e-6 ? gap : 1e-6);
        }
        int obs[64];
        for (int m = 0; m < M; ++m) {
            int s = 0;
            for (int rr = 0; rr < tiers[m].replicas; ++rr) s += (int)reps[base[m] + rr].count;
            obs[m] = s;
            if (obs_out) obs_out[i * M + m] = s;
        }
        if (rate_out) rate_out[i] = rate;
        int tier;
        if (forced_actions) tier = forced_actions[i];
        else if (static_tier >= 0) tier = static_tier;
        else {
            /* encode (policy.py:52-65) + forward (policy.py:111-118) */
            for (int d = 0; d < D; ++d) x[d] = 0.0;
            x[task[i]] = 1.0;
            for (int m = 0; m < M; ++m) x[T + m] = (double)obs[m] / enc_scales[m];
            x[D - 1] = rate / rate_scale;
            for (int j = 0; j < hidden; ++j) {
                double acc = 0.0;
                for (int d = 0; d < D; ++d) acc += x[d] * w1[d * hidden + j];
                acc += b1[j];
                h[j] = acc > 0.0 ? acc : 0.0;
            }
            tier = 0;
            for (int m = 0; m < M; ++m) {
                double acc = 0.0;
                for (int j = 0; j < hidden; ++j) acc += h[j] * w2[j * M + m];
                acc += b2[m];
                q[m] = acc;
                if (q_out) q_out[i * M + m] = acc;
                if (acc > q[tier]) tier = m; /* np.argmax: first maximum */
            }
        }
        if (tier < 0 || tier >= M) {
            free(x); free(h);
            for (int k = 0; k < R; ++k) free(reps[k].buf);
            free(reps);
            return -1;
        }
        /* ClusterSim.submit (simcore.py:94-111): min (len(active), len(queue), id) */
        int best = 0;
        int64_t best_key = -1;
        for (int rr = 0; rr < tiers[tier].replicas; ++rr) {
            replica_t* r = &reps[base[tier] + rr];
            int64_t mb = tiers[tier].max_batch;
            int64_t act = r->count < mb ? r->count : mb;
            int64_t que = r->count - act;
            int64_t key = act * ((int64_t)1 << 40) + que;
            if (best_key < 0 || key < best_key) {
                best_key = key;
                best = rr;
            }
        }
        replica_t* r = &reps[base[tier] + best];
        slot_t s = {t_arr, (int32_t)i, (int32_t)task[i], -1};
        int was_idle = r->kind == K_NONE;
        fifo_push(r, s);
        if (r->count <= tiers[tier].max_batch && was_idle) {
            r->kind = K_START; /* scheduled at clock_ms == this arrival */
            r->t = t_arr;
        }
    }
    for (int m = 0; m < M; ++m)
        for (int rr = 0; rr < tiers[m].replicas; ++rr)
            advance_replica(&reps[base[m] + rr], &tiers[m], m, INFINITY, &sc);
    for (int k = 0; k < R; ++k) free(reps[k].buf);
    free(reps);
    free(x);
    free(h);
    return 0;
}
