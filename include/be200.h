/*
 * be200.h — C ABI of the B200-native best-effort serving hot path.
 *
 * The reference (`besteffort`, pure Python + numpy) has no FFI layer: its
 * "interface" is the Python call surface in pkg/src/besteffort.  Each entry
 * point below replaces one piece of that surface for a whole batch of
 * independent environments (one environment = one reference `ClusterSim`
 * driven by one `run_eval` / `run_training` loop):
 *
 *   be_env_create / be_env_destroy   ClusterSim.__init__          simcore.py:72-84
 *   be_env_reset                     ClusterSim(tiers) (re-create) evalkit.py:189-191
 *   be_env_step                      advance + observe + encode +  evalkit.py:185-205,
 *                                    forward/argmax + submit        simcore.py:94-157
 *   be_env_step_observe / _submit    the same, split around any    evalkit.py:185-205
 *                                    router (e.g. be_qnet_route_tc)
 *   be_env_drain                     ClusterSim.drain              simcore.py:151-153
 *   be_env_new_segment               segment reset of run_eval     evalkit.py:186-192
 *   be_rollout_greedy                run_eval (whole trace)        evalkit.py:154-209
 *   be_qnet_route_f64                select_action / argmax(forward) policy.py:111-132
 *   be_qnet_route_tc                 the same on the tensor cores   policy.py:111-132
 *                                    (tcgen05 tf32, certified, fp64 fallback)
 *   be_reduce_eval                   windowed + threshold_counts,  evalkit.py:217-241,
 *                                    miss_fractions_by_rate        evalkit.py:61-68
 *   be_reduce_selection              selection_distribution counts evalkit.py:244-262
 *   be_windowed                      windowed series               evalkit.py:217-226
 *   be_trace_gen_stable              gen_stable (Philox, on device) workload.py:120-141
 *   be_trace_gen                     gen_stable / gen_unpredictable_* workload.py:94-209
 *   be_learner_*                     train_step / _StepKernel /    trainer.py:211-290
 *                                    Adam                          trainer.py:177-199
 *   be_replay_*                      ReplayBuffer                  trainer.py:101-163
 *
 * Conventions
 *  - All data pointers are DEVICE pointers (e.g. torch.Tensor.data_ptr()),
 *    borrowed, caller-owned and valid until `stream` reaches the call.
 *    `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *  - Handles own their device state; no allocation happens inside step /
 *    rollout calls.
 *  - Every function returns a be_status.  On failure be_last_error() returns
 *    a thread-local message.  Device-side failures (FIFO ring overflow,
 *    non-finite router input) are latched in the handle and reported by
 *    be_env_check() after a stream sync; they are never silently ignored.
 *  - Per-env arrays are env-major: element (e, i) lives at [e * ld + i].
 */
#ifndef BE200_H
#define BE200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BE_MAX_TIERS 8
#define BE_MAX_TASKS 16
#define BE_MAX_LANES 32 /* sum of replicas over tiers: one warp lane per replica */

typedef enum {
    BE_OK = 0,
    BE_EINVAL = 1,    /* bad argument -> reference ValueError / InvalidParameterError */
    BE_ECAPACITY = 2, /* a replica FIFO ring overflowed (simcore.py never drops) */
    BE_ECUDA = 3,     /* CUDA runtime error */
    BE_ENONFINITE = 4 /* non-finite router input (policy.py:115-116) */
} be_status;

/* ModelTierSpec (simcore.py:21-37) */
typedef struct {
    int32_t replicas;
    int32_t max_batch;
    int32_t tokens_per_request;
    int32_t _pad;
    double alpha_ms;
    double beta_ms;
} be_tier;

/* Everything a ClusterSim + RewardSpec + StateEncoding + RateEstimator need. */
typedef struct {
    int32_t n_tiers;                 /* M */
    int32_t n_tasks;                 /* T */
    be_tier tiers[BE_MAX_TIERS];
    double deadline[BE_MAX_TASKS];   /* TaskSpec.deadline_ms_per_token (reward.py:32-42) */
    int32_t soft[BE_MAX_TASKS];      /* 1 = soft deadline kind */
    double matrix[BE_MAX_TASKS * BE_MAX_TIERS]; /* RewardSpec.matrix, [T][M] */
    double decay_per_ms;             /* RewardSpec.decay_per_ms */
    double cutoff_fraction;          /* RewardSpec.cutoff_fraction */
    double batch_scales[BE_MAX_TIERS]; /* StateEncoding.batch_scales (policy.py:23-42) */
    double rate_scale;               /* StateEncoding.rate_scale */
    int32_t estimator_true_rate;     /* RateEstimator mode: 0 estimated, 1 true-rate */
    int32_t reset_between_segments;  /* run_eval(reset_between_segments=...) */
    double prior_rate;               /* RateEstimator.prior_rate */
    int32_t ring_capacity;           /* per-replica FIFO slots (power of two) */
    int32_t skip_ahead;              /* 1 = exact closed-form iteration skipping (default) */
    int32_t q_screen;                /* 1 = greedy rollout decides with a certified fp32 screen and
                                        falls back to fp64 where it cannot certify (default;
                                        decisions identical); 0 = fp64 for every decision */
    int32_t _pad2;
} be_cfg;

/* Trace batch: WorkloadTrace (workload.py:39-91) for E envs, SoA, env-major. */
typedef struct {
    int32_t n_envs;
    int32_t _pad;
    int64_t ld;                  /* row stride (elements) of arrival/task/outputs */
    const double* arrival_ms;    /* [E][ld] nondecreasing per env */
    const uint8_t* task;         /* [E][ld] */
    const int64_t* n_events;     /* [E] or NULL (= ld for every env) */
    const int64_t* seg_offsets;  /* [E+1] CSR into seg_start/seg_rate */
    const int64_t* seg_start;    /* SegmentMark.start_index */
    const double* seg_rate;      /* SegmentMark.rate */
    const int32_t* seg_bucket;   /* per segment reducer bucket id, or NULL */
    /* Streamed upload (optional, be_rollout_greedy): env e's arrival/task rows are
     * read only after env_ready[e / envs_per_ready] >= ready_value — the caller's
     * copy stream writes that flag after the rows' copy (e.g. a 4-byte
     * cudaMemcpyAsync), so the rollout starts on the first envs while the rest of
     * the batch is still in flight.  NULL: the rows are resident. */
    const int32_t* env_ready;
    int32_t envs_per_ready;
    int32_t ready_value;
} be_trace_soa;

/* QNetwork parameters (policy.py:68-118), fp64, BEQN1 order/layout. */
typedef struct {
    int32_t hidden;      /* even, in [2, 1024] (the tensor-core router: multiple of 32, <= 256) */
    int16_t n_tasks;     /* QNetwork.n_tasks: must equal the env's / router's T */
    int16_t n_tiers;     /* QNetwork.n_tiers: must equal M (policy.py:111-116 rejects
                            an input of the wrong dimension; a mismatched net would
                            read past w1 / w2) */
    const double* w1;    /* [D][H], D = T + M + 1 */
    const double* b1;    /* [H] */
    const double* w2;    /* [H][M] */
    const double* b2;    /* [M] */
} be_qweights;

/* Per-request records (RequestRecord, evalkit.py:37-45), env-major [E][ld].
 * flags = tier_id | (deadline_miss << 7).  Optional per-step router inputs. */
typedef struct {
    uint8_t* flags;      /* required */
    double* reward;      /* required */
    double* realized;    /* nullable: realized ms/token */
    int32_t* obs;        /* nullable: [E][ld][M] observed per-tier batch */
    double* rate;        /* nullable: [E][ld] rate signal */
    double* q;           /* nullable: [E][ld][M] Q-values (policy mode) */
} be_records;

typedef struct be_env be_env;

const char* be_last_error(void);
int32_t be_abi_version(void);

/* Environment handle: E envs, device state (replica headers, FIFO rings). */
int32_t be_env_create(const be_cfg* cfg, int32_t n_envs, int32_t device, be_env** out);
int32_t be_env_destroy(be_env* env);
size_t be_env_device_bytes(const be_env* env);
/* Re-initialise envs whose mask byte is nonzero (all if mask == NULL). */
int32_t be_env_reset(be_env* env, const uint8_t* mask, void* stream);
/* Sync `stream` and report latched device errors (ring overflow, ...). */
int32_t be_env_check(be_env* env, void* stream);
/* The latched device status {code, env} copied to dst (host pinned or device int32[2])
 * in stream order, without a synchronisation: a pipelined caller (StreamingEvaluator)
 * reads it with the batch's results and calls be_env_check only when it is nonzero. */
int32_t be_env_status_async(be_env* env, int32_t* dst, void* stream);
/* Counters of the certified fp32 decision screen of be_rollout_greedy, summed
 * over all rollouts since the last reset: out[0] = screened decisions,
 * out[1] = decisions that fell back to fp64.  Synchronises the device. */
int32_t be_env_screen_stats(be_env* env, int64_t* out, int32_t reset);

/* One env step for all E envs (evalkit.py:193-205 / trainer.py:375-395):
 * advance every replica to arrival_ms[e], score completions into `rec`
 * (indexed by each env's request id), update the rate estimator, observe,
 * route (forced_action[e] if non-NULL, else static_tier if >= 0, else greedy
 * argmax of W; epsilon-greedy with Philox(seed, counter) when epsilon > 0),
 * submit.  Outputs obs [E][M], rate [E], action [E], q [E][M] (nullable). */
int32_t be_env_step(be_env* env, const double* arrival_ms, const uint8_t* task,
                    const double* true_rate, const uint8_t* forced_action,
                    const be_qweights* W, int32_t static_tier, double epsilon,
                    uint64_t philox_seed, uint64_t philox_counter, int64_t rec_ld,
                    be_records* rec, int32_t* obs_out, double* rate_out,
                    uint8_t* action_out, double* q_out, double* x_out, void* stream);
/* The same step split around a router of the caller's choice (the reference's
 * own order, evalkit.py:185-205: advance / observe / encode, then select_action,
 * then submit).  be_env_step_observe advances every env to its arrival (scoring
 * completions into rec), updates the estimator and writes the encoded state
 * x_out [E][D] (required), obs_out [E][M] and rate_out [E] (nullable); it makes
 * no decision.  be_env_step_submit then submits request `next id` of every env
 * to the tier in action [E] (e.g. the output of be_qnet_route_tc on x_out) — the
 * same arrival/task arrays as the observe call.  observe + route + submit ==
 * be_env_step with that router's decisions. */
int32_t be_env_step_observe(be_env* env, const double* arrival_ms, const uint8_t* task,
                            const double* true_rate, int64_t rec_ld, be_records* rec, double* x_out,
                            int32_t* obs_out, double* rate_out, void* stream);
int32_t be_env_step_submit(be_env* env, const double* arrival_ms, const uint8_t* task, const uint8_t* action,
                           int64_t rec_ld, be_records* rec, void* stream);
/* Run every replica to completion (simcore.py:151-153). */
int32_t be_env_drain(be_env* env, int64_t rec_ld, be_records* rec, void* stream);
/* Stable-segment reset of run_eval (evalkit.py:186-192) for the envs with
 * mask[e] != 0 (device u8 [E]; NULL = all): drain every replica (completions
 * scored into rec), then a fresh ClusterSim (simcore.py:72-84) and an empty
 * estimator window (workload.py:249-250).  Request ids continue (they index
 * the trace), unlike be_env_reset, which also restarts them at 0. */
int32_t be_env_new_segment(be_env* env, const uint8_t* mask, int64_t rec_ld, be_records* rec,
                           void* stream);

/* Whole greedy rollout (run_eval) of E envs over a trace batch, fused in one
 * persistent kernel: one warp per env, one lane per replica.  Routing:
 * forced_action [E][ld] if non-NULL, else static_tier if >= 0, else W. */
int32_t be_rollout_greedy(be_env* env, const be_trace_soa* trace, const be_qweights* W,
                          int32_t static_tier, const uint8_t* forced_action, be_records* rec,
                          void* stream);

/* What the last be_rollout_greedy on this handle launched (host-side record,
 * no sync): out[0] = n_tiers (template M), [1] lanes per env (16 | 32),
 * [2] 1 = true-rate estimator variant, [3] 1 = the throughput variant
 * (BE_ROLLOUT_MINB CTAs/SM, fewer registers; chosen when the batch fills them),
 * [4] 1 = skip table staged in shared memory (0 = read through L1),
 * [5] 1 = certified fp32 decision screen, [6] resident CTAs per SM, [7] CTAs. */
int32_t be_env_rollout_plan(const be_env* env, int32_t* out /* [8] */);

/* Batched router: q = relu(x W1 + b1) W2 + b2; action = argmax (first max),
 * or uniform random with probability epsilon (Philox4x32-10). x: [B][D]. */
int32_t be_qnet_route_f64(const be_qweights* W, int32_t n_tasks, int32_t n_tiers,
                          const double* x, int32_t batch, double epsilon, uint64_t philox_seed,
                          uint64_t philox_counter, double* q_out, uint8_t* action_out,
                          void* stream);

/* The same router on the tensor cores (route_tc.cu): layer 1 as
 * tcgen05.mma.kind::tf32 with a 3xTF32 split over 256-state tiles (TMEM
 * accumulators, weights staged in shared memory by one bulk async copy),
 * relu + layer 2 in fp32; each greedy decision is certified by an error bound
 * or re-evaluated with the exact arithmetic of be_qnet_route_f64, so actions
 * equal be_qnet_route_f64's.  q_out (nullable) is fp32 [batch][n_tiers]
 * (within 1e-5 relative of the fp64 router).  Requires n_tiers <= 4,
 * n_tasks + n_tiers + 2 <= 16, hidden a multiple of 32 in [32, 256]
 * (be_qnet_route_tc_supported); `workspace` = device scratch of
 * be_qnet_route_tc_workspace_bytes(hidden) bytes (16-byte aligned, not shared
 * by concurrent calls); stats (nullable, device int64[2]) accumulates
 * (states, fp64 re-evaluations). */
int32_t be_qnet_route_tc_supported(int32_t n_tasks, int32_t n_tiers, int32_t hidden);
size_t be_qnet_route_tc_workspace_bytes(int32_t hidden);
int32_t be_qnet_route_tc(const be_qweights* W, int32_t n_tasks, int32_t n_tiers, const double* x,
                         int32_t batch, double epsilon, uint64_t philox_seed, uint64_t philox_counter,
                         float* q_out, uint8_t* action_out, void* workspace, int64_t* stats,
                         void* stream);

/* Evaluation reducer (evalkit.py:212-241, :61-74): per env a sequential fp64
 * prefix sum of rewards in request order, trailing `window` means, counts of
 * windows >= theta (== 1.0 for theta == 1.0); per (env, bucket) miss and
 * request counts and reward sums.  Outputs:
 *   win_counts [E][n_theta] int64, n_windows [E] int64,
 *   bucket_miss / bucket_req [E][n_buckets] int64, bucket_reward [E][n_buckets] f64
 * Buckets come from trace->seg_bucket (NULL -> everything in bucket 0).
 * The thresholds travel BY VALUE (no host/device pointer ambiguity; the
 * library turns each theta into an exact cut-off on the window sum, see
 * reduce.cu).  Miss flags are the rollout's per-request flags bit 7
 * (realized > deadline[task], evalkit.py:65-67, decided where realized is made). */
#define BE_MAX_THETA 8
typedef struct {
    int32_t n;                      /* number of thresholds, 1..BE_MAX_THETA */
    int32_t _pad;
    double theta[BE_MAX_THETA];     /* each in [0, 1]; 1.0 counts exact peaks only */
} be_thresholds;

int32_t be_reduce_eval(const be_trace_soa* trace, const uint8_t* flags, const double* reward,
                       int32_t window, be_thresholds thresholds,
                       int32_t n_buckets, int64_t* win_counts, int64_t* n_windows,
                       int64_t* bucket_miss, int64_t* bucket_req, double* bucket_reward,
                       void* stream);

/* Selection counts for selection_distribution (evalkit.py:244-262): counts
 * [T][K][M] int64 (ADDED to: zero them first) of requests per (task, rate
 * bucket of the request's segment = trace->seg_bucket, tier = flags & 0x3f). */
int32_t be_reduce_selection(const be_trace_soa* trace, const uint8_t* flags, int32_t n_tasks,
                            int32_t n_tiers, int32_t n_buckets, int64_t* counts, void* stream);

/* windowed (evalkit.py:217-226) per env: out[e][k] = (c[k+w] - c[k]) / w for
 * k in [0, n_e - w], c the sequential fp64 prefix sum of reward[e][:]. */
int32_t be_windowed(const be_trace_soa* trace, const double* reward, int32_t window, double* out,
                    void* stream);

/* On-device gen_stable (workload.py:120-141) with Philox4x32-10 keyed by
 * (seed, env_offset + e): per env one Poisson segment at rate[e] req/s, exponential gaps
 * of mean 1000/rate ms accumulated sequentially in fp64, uniform task ids;
 * the first n events of the segment (truncated).  Writes arrival/task [E][ld]. */
int32_t be_trace_gen_stable(int32_t n_envs, int64_t env_offset, int64_t n, int64_t ld,
                            const double* rate, int32_t n_tasks, uint64_t seed,
                            double* arrival_ms, uint8_t* task, void* stream);

/* On-device workload generators (workload.py:94-209) with Philox4x32-10 keyed
 * by (seed, env_offset + e) — every global env id gets the same trace on any
 * number of GPUs.  Kinds:
 *   BE_GEN_STABLE        gen_stable (workload.py:120-141): segment k holds
 *                        rates[e][k] for hold_ms on [k*hold, (k+1)*hold)
 *                        (Poisson arrivals, workload.py:94-111); with
 *                        truncate = 1 the trace stops at ld events (config 1),
 *                        else more than ld events is BE_ECAPACITY;
 *   BE_GEN_UNPRED_TIME   gen_unpredictable_time_based (workload.py:144-171):
 *                        band 90/8/2 %, rate uniform in the band, shifted-
 *                        geometric count of mean 20 * rate, n requests;
 *   BE_GEN_UNPRED_REQ    gen_unpredictable_request_based (workload.py:174-198):
 *                        rate uniform on [1, 48], geometric count of mean 500.
 * Tasks are uniform over task_ids[0..n_task_ids) (all of [0, n_tasks) when
 * n_task_ids == 0), workload.py:201-209.  Outputs (device, env-major):
 * arrival/task [E][ld], n_events [E], seg_count [E], seg_start/seg_rate
 * [E][seg_capacity].  More than seg_capacity segments -> BE_ECAPACITY (latched
 * in *status, a device int32[2] = {code, first env}, checked by the caller). */
#define BE_GEN_STABLE 0
#define BE_GEN_UNPRED_TIME 1
#define BE_GEN_UNPRED_REQ 2
typedef struct {
    int32_t kind;
    int32_t n_tasks;
    int32_t n_task_ids;
    int32_t task_ids[BE_MAX_TASKS];
    int32_t n_rates;          /* BE_GEN_STABLE: segments per env */
    int32_t truncate;         /* BE_GEN_STABLE: stop at ld events instead of failing */
    int64_t rate_ld;          /* row stride of rates (0 = one row shared by every env) */
    const double* rates;      /* BE_GEN_STABLE: device [E or 1][rate_ld] req/s */
    double hold_ms;           /* BE_GEN_STABLE: segment duration */
    int64_t n;                /* BE_GEN_UNPRED_*: requests per env (<= ld) */
    int64_t seg_capacity;     /* segments per env the outputs can hold */
} be_gen_cfg;

int32_t be_trace_gen(const be_gen_cfg* cfg, int32_t n_envs, int64_t env_offset, int64_t ld,
                     uint64_t seed, double* arrival_ms, uint8_t* task, int64_t* n_events,
                     int64_t* seg_count, int64_t* seg_start, double* seg_rate, int32_t* status,
                     void* stream);

/* ---------------------------------------------------------------- training
 * Replay + learner (trainer.py:101-290) and the training workload
 * (trainer.py:293-316) for E envs stepping in lockstep (request id = step).
 * All learner arithmetic is fp64; updates are deterministic for a batch. */
typedef struct {
    int32_t n_tasks, n_tiers, hidden, n_envs;
    int64_t replay_capacity;    /* TrainConfig.buffer_capacity */
    int32_t pending_capacity;   /* P: max decisions a request may stay unresolved */
    int32_t batch;              /* TrainConfig.batch_size */
    int64_t warmup;             /* TrainConfig.warmup */
    int64_t target_sync_every;  /* TrainConfig.target_sync_every */
    double discount, learning_rate;
    int32_t adam;               /* 1 = Adam (beta 0.9/0.999, eps 1e-8), 0 = SGD */
    int32_t huber;              /* 1 = huber (delta 1), 0 = squared */
    double rate_low, rate_high; /* TrainingWorkload rate range (log-uniform) */
    int32_t regime_equal_time;  /* 1 = "equal-time" cadence, 0 = "requests" */
    int32_t _pad;
    double regime_mean_seconds, regime_mean_requests;
} be_learner_cfg;

typedef struct be_learner be_learner;

/* Device views into a learner (all device pointers). */
typedef struct {
    be_qweights online, target;  /* routing weights for be_env_step */
    double* params;              /* online w1 | b1 | w2 | b2, contiguous (nparam) */
    double* grad;                /* gradient of the last backward (nparam): all-reduce here */
    int32_t nparam;
    int32_t _pad;
    double* loss;                /* [0] loss of the last backward, [1] loss of the last update */
    int64_t* counters;           /* [0] Adam t, [1] gradient steps, [2] any update applied,
                                    [3] iteration index (be_train_iteration) */
    double* ring_states;         /* [C][D] */
    double* ring_next_states;    /* [C][D] */
    uint8_t* ring_actions;       /* [C] */
    double* ring_rewards;        /* [C] */
    double* ring_cont;           /* [C] */
    int64_t* ring_state;         /* [0] cursor, [1] size, [2] total commits, [3] commits of the
                                    last step, [4] most decisions a request stayed in flight */
    double* pending_x;           /* [P][E][D]: x_out of be_env_step for request id = step */
    uint8_t* pending_action;     /* [P][E]:    action_out of be_env_step */
    uint8_t* pending_flags;      /* [E][P]:    be_records.flags with rec_ld = P */
    double* pending_reward;      /* [E][P]:    be_records.reward with rec_ld = P */
    double* workload_state;      /* [E][3] time_ms, rate, requests left in the regime */
    int64_t* gate;               /* [1] update gate for be_train_iteration(use_gate = 1) */
} be_learner_views_t;

int32_t be_learner_create(const be_learner_cfg* cfg, int32_t device, be_learner** out);
int32_t be_learner_destroy(be_learner* learner);
/* Online = target = the given parameters (host or device pointers); Adam state reset. */
int32_t be_learner_set_params(be_learner* learner, const double* w1, const double* b1,
                              const double* w2, const double* b2, void* stream);
int32_t be_learner_views(be_learner* learner, be_learner_views_t* views);
/* TrainingWorkload.next_arrival for every env (Philox keyed by seed, counter step). */
int32_t be_learner_workload(be_learner* learner, uint64_t seed, int64_t step, double* arrival_ms,
                            uint8_t* task, double* true_rate, void* stream);
/* Commit every transition whose reward and next state are both known after the
 * decision for request `step` (trainer.py:143-156); ring slots by env-order scan. */
int32_t be_learner_commit(be_learner* learner, int64_t step, void* stream);
/* Sample a batch (Philox(seed, counter)) and compute loss + gradients into views.grad
 * (no-op while the ring holds fewer than max(batch, warmup) transitions). */
int32_t be_learner_backward(be_learner* learner, uint64_t seed, uint64_t counter,
                            int64_t* sample_idx /* nullable [batch] */, void* stream);
/* Same on an explicit batch (states/next_states [B][D], actions u8, rewards, cont). */
int32_t be_learner_backward_batch(be_learner* learner, const double* states,
                                  const uint8_t* actions, const double* rewards,
                                  const double* next_states, const double* cont,
                                  int32_t batch, void* stream);
/* Adam/SGD on views.grad, then the target sync every target_sync_every steps. */
int32_t be_learner_apply(be_learner* learner, int32_t explicit_batch, void* stream);
int32_t be_learner_check(be_learner* learner, void* stream);

/* Data-parallel learner without a collective library (be_train_iteration
 * phase 4): every rank's update kernel publishes its tile-reduced gradients in
 * an exchange buffer, waits for every rank's publication of the same update
 * (release/acquire at system scope over NVLink peer memory, bounded wait), sums
 * all ranks' gradients in rank order, scales by 1/W and applies Adam — the
 * replicas stay bit-identical and no NCCL launch sits on the update path.
 *   be_learner_exchange_buffer: this learner's exchange allocation (device);
 *   be_learner_ipc_handle:      its cudaIpcMemHandle_t (64 bytes) for other processes;
 *   be_learner_set_peers:       the device pointers (valid in this process) of every
 *                               rank's exchange allocation, xmems[rank] = own;
 *   be_learner_open_peers_ipc:  the same from world x 64-byte IPC handles. */
int32_t be_learner_exchange_buffer(be_learner* learner, void** xmem, size_t* bytes);
int32_t be_learner_ipc_handle(be_learner* learner, void* handle_out);
int32_t be_learner_set_peers(be_learner* learner, int32_t world, int32_t rank, const uint64_t* xmems);
int32_t be_learner_open_peers_ipc(be_learner* learner, int32_t world, int32_t rank, const void* handles);

/* One iteration of run_training's loop (trainer.py:374-401) for all E envs,
 * with EVERY per-iteration value read from device memory — the iteration index
 * `it` (views.counters[3]), epsilon_at(it) (trainer.py:85-90), the Philox
 * counters — so a CUDA graph of K iterations replays unchanged:
 *   workload(it) -> be_env_step(epsilon_at(it), counter it; x/action into the
 *   pending slot it % P) -> commit(it) -> update(s) -> it += 1.
 * Bit-identical to driving be_learner_workload / be_env_step / be_learner_commit
 * / be_learner_backward / be_learner_apply from the host with the same seeds.
 * phase 0: whole iteration in two launches when the env has <= 16 replicas and
 *          input dim <= 16: the env step with the arrivals and the replay commit
 *          fused in, then per update one kernel — row tiles (Double-Q targets, Huber
 *          backward) whose last CTAs reduce the tiles, apply Adam and repack the
 *          step's weights (else: separate step, commit and tile + reduce/Adam launches).
 *          Weights written outside the learner (be_learner_set_params) are repacked
 *          by the next phase-0 call.
 * phase 4: whole iteration with the peer-memory gradient exchange (data-parallel,
 *          be_learner_set_peers first): no host round trip, graph-capturable.
 * phase 3: the env part only (workload, env step, commits; with
 *          updates_per_step == 0 it also advances the iteration);
 * phase 1: the gradients of update `update_index` into views.grad — all-reduce
 *          them here (DP learner);
 * phase 2: optimizer step of update `update_index`; the last one advances it.
 * use_gate = 1 (phases 1/2): the update runs iff *views.gate != 0 instead of the
 * local "replay holds max(batch, warmup) transitions" test — the DP learner
 * all-reduces (MIN) that readiness so every rank updates in the same iterations. */
typedef struct {
    uint64_t workload_seed, policy_seed, sample_seed;
    double epsilon_start, epsilon_end;
    int64_t epsilon_decay_steps;  /* int(epsilon_decay_fraction * total_iterations) */
    int32_t updates_per_step;
    int32_t phase;
    int32_t update_index;
    int32_t use_gate;
    int32_t router;   /* BE_ROUTER_FP64: the decision inside the env step (fp64 Q);
                         BE_ROUTER_TC: the decision on tcgen05 inside the env step
                         (<= 16 replicas; else observe -> be_qnet_route_tc -> submit),
                         certified + fp64 fallback: the same decisions */
    int32_t _pad;
} be_train_iter_cfg;
#define BE_ROUTER_FP64 0
#define BE_ROUTER_TC 1

int32_t be_train_iteration(be_learner* learner, be_env* env, const be_train_iter_cfg* cfg,
                           void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BE200_H */
