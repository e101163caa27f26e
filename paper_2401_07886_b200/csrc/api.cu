// api.cu — the extern "C" boundary (include/be200.h): argument validation,
// handle lifetime, error reporting.  All compute is in the other .cu files.
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "be200.h"
#include "be_internal.h"

namespace be {

static thread_local char g_err[512] = "";

int set_error(int code, const char* msg) {
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return code;
}

int set_cuda_error(cudaError_t e, const char* where) {
    snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
    return BE_ECUDA;
}

void make_score_aux(const be_cfg& c, ScoreAux* aux) {
    for (int k = 0; k < BE_MAX_TASKS * BE_MAX_TIERS; ++k) aux->hit_tau[k] = -INFINITY;
    for (int t = 0; t < c.n_tasks; ++t)
        for (int m = 0; m < c.n_tiers; ++m)
            aux->hit_tau[t * BE_MAX_TIERS + m] = tau_le(c.deadline[t], (double)c.tiers[m].tokens_per_request);
}

// round(x * 2^(52 - e)) to an integer (x >= 0); false on a rounding tie or overflow
static bool scaled_round(double x, int e, long long& out) {
    if (x == 0.0) {
        out = 0;
        return true;
    }
    long long bits;
    memcpy(&bits, &x, 8);
    int ex = (int)((bits >> 52) & 0x7ff);
    if (ex == 0 || ex == 0x7ff || bits < 0) return false;
    long long mx = (bits & 0xfffffffffffffLL) | (1LL << 52);
    int s = e - (ex - 1023);  // right shift
    if (s <= 0) {
        if (s < -9) return false;
        out = mx << (-s);
        return true;
    }
    if (s >= 60) {
        out = 0;
        return true;
    }
    long long q = mx >> s;
    long long rem = mx & ((1LL << s) - 1);
    long long half = 1LL << (s - 1);
    if (rem == half) return false;
    out = q + (rem > half ? 1 : 0);
    return true;
}

// D(tier m, n, e) = (RN_u(alpha_m) + RN_u(RN(beta_m * n))) with u = 2^(e - 52): the
// exact per-cycle advance of a replica with n running requests while its clock
// stays in binade e (be_env.cuh, skip_cycles).  0 where a rounding tie makes the
// advance parity-dependent (the kernel then steps one iteration at a time).
int build_skip_table(const be_cfg& c, double* out) {
    int rows = 0;
    for (int m = 0; m < c.n_tiers; ++m) {
        const be_tier& t = c.tiers[m];
        for (int n = 0; n <= t.max_batch; ++n, ++rows) {
            if (!out) continue;
            const double cn = t.beta_ms * (double)n;  // simcore.py:146, beta * n
            for (int k = 0; k < SKIP_NB; ++k) {
                const int e = SKIP_ELO + k;
                long long a, b;
                double D = 0.0;
                if (n > 0 && scaled_round(t.alpha_ms, e, a) && scaled_round(cn, e, b) && a + b > 0 &&
                    a + b < (1LL << 53))
                    D = ldexp((double)(a + b), e - 52);
                out[(size_t)rows * SKIP_NB + k] = D;
            }
        }
    }
    return rows;
}

static int validate_cfg(const be_cfg* c, int* lanes) {
    if (!c) return set_error(BE_EINVAL, "cfg is NULL");
    if (c->n_tiers < 1 || c->n_tiers > BE_MAX_TIERS)
        return set_error(BE_EINVAL, "n_tiers must be in [1, 8]");
    if (c->n_tasks < 1 || c->n_tasks > BE_MAX_TASKS)
        return set_error(BE_EINVAL, "n_tasks must be in [1, 16]");
    int R = 0;
    for (int m = 0; m < c->n_tiers; ++m) {
        const be_tier& t = c->tiers[m];
        // ModelTierSpec.__post_init__ (simcore.py:31-37)
        if (t.replicas < 1) return set_error(BE_EINVAL, "replicas must be >= 1");
        if (!(t.alpha_ms > 0) || !(t.beta_ms >= 0) || !isfinite(t.alpha_ms) || !isfinite(t.beta_ms))
            return set_error(BE_EINVAL, "alpha_ms must be > 0 and beta_ms >= 0");
        if (t.max_batch < 1 || t.tokens_per_request < 1)
            return set_error(BE_EINVAL, "max_batch and tokens_per_request must be >= 1");
        R += t.replicas;
    }
    if (R > BE_MAX_LANES) return set_error(BE_EINVAL, "total replicas per env must be <= 32 (one warp)");
    for (int k = 0; k < c->n_tasks; ++k) {
        if (!(c->deadline[k] > 0)) return set_error(BE_EINVAL, "deadline must be positive");
        for (int m = 0; m < c->n_tiers; ++m) {
            double v = c->matrix[k * c->n_tiers + m];
            if (!(v >= 0 && v <= 1)) return set_error(BE_EINVAL, "matrix entries must lie in [0, 1]");
        }
    }
    if (!(c->decay_per_ms > 0 && c->decay_per_ms <= 1) || !(c->cutoff_fraction > 0 && c->cutoff_fraction <= 1))
        return set_error(BE_EINVAL, "decay_per_ms and cutoff_fraction must lie in (0, 1]");
    if (!(c->rate_scale > 0)) return set_error(BE_EINVAL, "rate_scale must be positive");
    for (int m = 0; m < c->n_tiers; ++m)
        if (!(c->batch_scales[m] > 0)) return set_error(BE_EINVAL, "batch_scales must be positive");
    if (!(c->prior_rate > 0)) return set_error(BE_EINVAL, "prior_rate must be positive");
    int cap = c->ring_capacity;
    if (cap < 2 || (cap & (cap - 1)) != 0 || cap > (1 << 24))
        return set_error(BE_EINVAL, "ring_capacity must be a power of two in [2, 2^24]");
    *lanes = R;
    return BE_OK;
}

static int validate_weights(const be_qweights* W, const be_cfg& c) {
    if (!W || !W->w1 || !W->b1 || !W->w2 || !W->b2) return set_error(BE_EINVAL, "policy weights missing");
    if (W->n_tasks != c.n_tasks || W->n_tiers != c.n_tiers)
        return set_error(BE_EINVAL, "expected input dim: the policy network's (n_tasks, n_tiers) differ from "
                                    "the environment's");
    // any even width (the packed layouts pair hidden units); the fused rollout's fp32
    // decision screen switches itself off unless H is a multiple of 2 x lanes per env
    if (W->hidden < 2 || W->hidden % 2 != 0 || W->hidden > 1024)
        return set_error(BE_EINVAL, "hidden must be even, in [2, 1024]");
    size_t smem = rollout_smem_bytes(c.n_tasks, c.n_tiers, W->hidden, true);
    if (smem > 200 * 1024) return set_error(BE_EINVAL, "Q-network too large for shared memory");
    return BE_OK;
}

}  // namespace be

using namespace be;

extern "C" {

const char* be_last_error(void) { return g_err; }

int32_t be_abi_version(void) { return 1; }

int32_t be_env_create(const be_cfg* cfg, int32_t n_envs, int32_t device, be_env** out) {
    if (!out) return set_error(BE_EINVAL, "out is NULL");
    *out = nullptr;
    int R = 0;
    int rc = validate_cfg(cfg, &R);
    if (rc) return rc;
    if (n_envs < 1) return set_error(BE_EINVAL, "n_envs must be >= 1");
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaSetDevice");
    be_env* env = new be_env();
    memset(env, 0, sizeof(*env));
    env->cfg = *cfg;
    env->E = n_envs;
    env->R = R;
    env->device = device;
    int cap_log2 = 0;
    while ((1 << cap_log2) < cfg->ring_capacity) ++cap_log2;
    env->cap_log2 = cap_log2;
    cudaDeviceGetAttribute(&env->sms, cudaDevAttrMultiProcessorCount, device);
    env->ring_bytes = (size_t)n_envs * R * ((size_t)1 << cap_log2) * 16;
    size_t state = env_state_bytes_per_env(R) * (size_t)n_envs;
    if ((e = cudaMalloc(&env->rings, env->ring_bytes)) != cudaSuccess ||
        (e = cudaMalloc(&env->reps, state)) != cudaSuccess ||
        (e = cudaMalloc((void**)&env->d_counter, 64)) != cudaSuccess ||
        (e = cudaMalloc((void**)&env->d_status, 64)) != cudaSuccess ||
        (e = cudaMalloc((void**)&env->d_screen, 16)) != cudaSuccess ||
        (e = cudaMalloc((void**)&env->d_qpack, QPACK_MAX_DOUBLES * sizeof(double))) != cudaSuccess) {
        be_env_destroy(env);
        return set_cuda_error(e, "be_env_create: cudaMalloc");
    }
    cudaMemset(env->d_status, 0, 64);
    cudaMemset(env->d_screen, 0, 16);
    env->envs = nullptr;
    // a replica holds at most `capacity` requests, so obs_m <= replicas_m x capacity
    env->exact_mul = 1;
    for (int m = 0; m < cfg->n_tiers && env->exact_mul; ++m) {
        const double s = cfg->batch_scales[m], inv = 1.0 / s;
        const long long top = (long long)cfg->tiers[m].replicas << cap_log2;
        for (long long o = 0; o <= top; ++o) {
            volatile double a = (double)o * inv, b = (double)o / s;
            if (a != b) {
                env->exact_mul = 0;
                break;
            }
        }
    }
    if (cfg->skip_ahead) {
        env->skip_rows = build_skip_table(*cfg, nullptr);
        const size_t tb = (size_t)env->skip_rows * SKIP_NB * sizeof(double);
        double* h = (double*)malloc(tb);
        build_skip_table(*cfg, h);
        if ((e = cudaMalloc((void**)&env->d_skip, tb)) != cudaSuccess ||
            (e = cudaMemcpy(env->d_skip, h, tb, cudaMemcpyHostToDevice)) != cudaSuccess) {
            free(h);
            be_env_destroy(env);
            return set_cuda_error(e, "be_env_create: skip table");
        }
        free(h);
    }
    rc = launch_env_reset(env, nullptr, 0);
    if (rc) {
        be_env_destroy(env);
        return rc;
    }
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        be_env_destroy(env);
        return set_cuda_error(e, "be_env_create: reset");
    }
    *out = env;
    return BE_OK;
}

int32_t be_env_destroy(be_env* env) {
    if (!env) return BE_OK;
    cudaFree(env->rings);
    cudaFree(env->reps);
    cudaFree(env->d_counter);
    cudaFree(env->d_status);
    cudaFree(env->d_skip);
    cudaFree(env->d_screen);
    cudaFree(env->d_qpack);
    delete env;
    return BE_OK;
}

size_t be_env_device_bytes(const be_env* env) {
    if (!env) return 0;
    return env->ring_bytes + env_state_bytes_per_env(env->R) * (size_t)env->E + 128;
}

int32_t be_env_reset(be_env* env, const uint8_t* mask, void* stream) {
    if (!env) return set_error(BE_EINVAL, "env is NULL");
    return launch_env_reset(env, mask, (cudaStream_t)stream);
}

int32_t be_env_status_async(be_env* env, int32_t* dst, void* stream) {
    if (!env || !dst) return set_error(BE_EINVAL, "NULL argument");
    cudaError_t e = cudaMemcpyAsync(dst, env->d_status, 2 * sizeof(int32_t), cudaMemcpyDefault, (cudaStream_t)stream);
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "be_env_status_async");
}

int32_t be_env_check(be_env* env, void* stream) {
    if (!env) return set_error(BE_EINVAL, "env is NULL");
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e != cudaSuccess) return set_cuda_error(e, "be_env_check: sync");
    int32_t st[2];
    e = cudaMemcpy(st, env->d_status, sizeof(st), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return set_cuda_error(e, "be_env_check: copy");
    if (st[0] == 0) return BE_OK;
    cudaMemset(env->d_status, 0, 64);
    char msg[256];
    if (st[0] == BE_ECAPACITY)
        snprintf(msg, sizeof(msg),
                 "env %d: replica FIFO ring overflow (capacity %d) or iteration counter "
                 "overflow; recreate the env with a larger ring_capacity",
                 st[1], 1 << env->cap_log2);
    else if (st[0] == BE_EINVAL)
        snprintf(msg, sizeof(msg), "env %d: action / tier or task id out of range", st[1]);
    else if (st[0] == BE_ENONFINITE)
        snprintf(msg, sizeof(msg), "env %d: non-finite network input", st[1]);
    else if (st[0] == BE_ECUDA)
        snprintf(msg, sizeof(msg), "env %d: streamed trace rows never became ready (env_ready flag)", st[1]);
    else
        snprintf(msg, sizeof(msg), "env %d: device error %d", st[1], st[0]);
    return set_error(st[0], msg);
}

int32_t be_env_screen_stats(be_env* env, int64_t* out, int32_t reset) {
    if (!env || !out) return set_error(BE_EINVAL, "NULL argument");
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return set_cuda_error(e, "be_env_screen_stats: sync");
    unsigned long long h[2];
    e = cudaMemcpy(h, env->d_screen, sizeof(h), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return set_cuda_error(e, "be_env_screen_stats: copy");
    out[0] = (int64_t)h[0];
    out[1] = (int64_t)h[1];
    if (reset) cudaMemset(env->d_screen, 0, sizeof(h));
    return BE_OK;
}

int32_t be_env_rollout_plan(const be_env* env, int32_t* out) {
    if (!env || !out) return set_error(BE_EINVAL, "NULL argument");
    for (int k = 0; k < 8; ++k) out[k] = env->last_plan[k];
    return BE_OK;
}

int32_t be_rollout_greedy(be_env* env, const be_trace_soa* trace, const be_qweights* W,
                          int32_t static_tier, const uint8_t* forced_action, be_records* rec,
                          void* stream) {
    if (!env || !trace || !rec) return set_error(BE_EINVAL, "NULL argument");
    if (trace->n_envs < 1 || trace->n_envs > env->E)
        return set_error(BE_EINVAL, "trace has more envs than the env handle");
    if (!trace->arrival_ms || !trace->task || !trace->seg_offsets)
        return set_error(BE_EINVAL, "trace arrays missing");
    if (trace->ld < 0 || trace->ld > (1 << 24)) return set_error(BE_EINVAL, "trace length must be <= 2^24");
    if (!rec->flags || !rec->reward) return set_error(BE_EINVAL, "records.flags/reward required");
    if (static_tier >= env->cfg.n_tiers) return set_error(BE_EINVAL, "static tier out of range");
    if (!forced_action && static_tier < 0) {
        int rc = validate_weights(W, env->cfg);
        if (rc) return rc;
    }
    if (rec->q && (forced_action || static_tier >= 0)) rec->q = nullptr;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != env->device) cudaSetDevice(env->device);
    return launch_rollout(env, trace, W, static_tier, forced_action, rec, (cudaStream_t)stream);
}

int32_t be_env_step(be_env* env, const double* arrival_ms, const uint8_t* task,
                    const double* true_rate, const uint8_t* forced_action, const be_qweights* W,
                    int32_t static_tier, double epsilon, uint64_t philox_seed,
                    uint64_t philox_counter, int64_t rec_ld, be_records* rec, int32_t* obs_out,
                    double* rate_out, uint8_t* action_out, double* q_out, double* x_out,
                    void* stream) {
    if (!env || !arrival_ms || !task || !rec || !rec->flags || !rec->reward)
        return set_error(BE_EINVAL, "NULL argument");
    if (rec_ld < 1) return set_error(BE_EINVAL, "rec_ld must be >= 1");
    if (!(epsilon >= 0.0 && epsilon <= 1.0)) return set_error(BE_EINVAL, "epsilon must lie in [0, 1]");
    if (static_tier >= env->cfg.n_tiers) return set_error(BE_EINVAL, "static tier out of range");
    if (env->cfg.estimator_true_rate && !true_rate) return set_error(BE_EINVAL, "true-rate mode needs true_rate");
    if (!forced_action && static_tier < 0) {
        int rc = validate_weights(W, env->cfg);
        if (rc) return rc;
    }
    return launch_env_step(env, arrival_ms, task, true_rate, forced_action, W, static_tier, epsilon,
                           philox_seed, philox_counter, rec_ld, rec, obs_out, rate_out, action_out,
                           q_out, x_out, (cudaStream_t)stream);
}

int32_t be_env_step_observe(be_env* env, const double* arrival_ms, const uint8_t* task,
                            const double* true_rate, int64_t rec_ld, be_records* rec, double* x_out,
                            int32_t* obs_out, double* rate_out, void* stream) {
    if (!env || !arrival_ms || !task || !rec || !rec->flags || !rec->reward || !x_out)
        return set_error(BE_EINVAL, "NULL argument");
    if (rec_ld < 1) return set_error(BE_EINVAL, "rec_ld must be >= 1");
    if (env->cfg.estimator_true_rate && !true_rate) return set_error(BE_EINVAL, "true-rate mode needs true_rate");
    return launch_env_step_split(env, 1, arrival_ms, task, true_rate, nullptr, x_out, obs_out, rate_out, rec_ld,
                                 rec, (cudaStream_t)stream);
}

int32_t be_env_step_submit(be_env* env, const double* arrival_ms, const uint8_t* task, const uint8_t* action,
                           int64_t rec_ld, be_records* rec, void* stream) {
    if (!env || !arrival_ms || !task || !action || !rec || !rec->flags || !rec->reward)
        return set_error(BE_EINVAL, "NULL argument");
    if (rec_ld < 1) return set_error(BE_EINVAL, "rec_ld must be >= 1");
    return launch_env_step_split(env, 2, arrival_ms, task, nullptr, const_cast<uint8_t*>(action), nullptr, nullptr,
                                 nullptr, rec_ld, rec, (cudaStream_t)stream);
}

int32_t be_env_drain(be_env* env, int64_t rec_ld, be_records* rec, void* stream) {
    if (!env || !rec || !rec->flags || !rec->reward) return set_error(BE_EINVAL, "NULL argument");
    if (rec_ld < 1) return set_error(BE_EINVAL, "rec_ld must be >= 1");
    return launch_env_drain(env, rec_ld, rec, (cudaStream_t)stream);
}

int32_t be_env_new_segment(be_env* env, const uint8_t* mask, int64_t rec_ld, be_records* rec, void* stream) {
    if (!env || !rec || !rec->flags || !rec->reward) return set_error(BE_EINVAL, "NULL argument");
    if (rec_ld < 1) return set_error(BE_EINVAL, "rec_ld must be >= 1");
    return launch_env_drain(env, rec_ld, rec, (cudaStream_t)stream, mask, 1);
}

int32_t be_qnet_route_f64(const be_qweights* W, int32_t n_tasks, int32_t n_tiers, const double* x,
                          int32_t batch, double epsilon, uint64_t philox_seed,
                          uint64_t philox_counter, double* q_out, uint8_t* action_out,
                          void* stream) {
    if (!W || !W->w1 || !W->b1 || !W->w2 || !W->b2 || !x || !action_out)
        return set_error(BE_EINVAL, "NULL argument");
    if (n_tasks < 1 || n_tasks > BE_MAX_TASKS || n_tiers < 1 || n_tiers > BE_MAX_TIERS)
        return set_error(BE_EINVAL, "dimensions out of range");
    if (W->n_tasks != n_tasks || W->n_tiers != n_tiers)
        return set_error(BE_EINVAL, "expected input dim: the network's (n_tasks, n_tiers) differ from the router's");
    if (W->hidden < 1 || W->hidden > 4096) return set_error(BE_EINVAL, "hidden out of range");
    if (!(epsilon >= 0.0 && epsilon <= 1.0)) return set_error(BE_EINVAL, "epsilon must lie in [0, 1]");
    if (batch < 0) return set_error(BE_EINVAL, "batch must be >= 0");
    if (batch == 0) return BE_OK;
    return launch_route(W, n_tasks, n_tiers, x, batch, epsilon, philox_seed, philox_counter, q_out,
                        action_out, (cudaStream_t)stream);
}

int32_t be_qnet_route_tc_supported(int32_t n_tasks, int32_t n_tiers, int32_t hidden) {
    return route_tc_supported(n_tasks, n_tiers, hidden) ? 1 : 0;
}

size_t be_qnet_route_tc_workspace_bytes(int32_t hidden) {
    return hidden >= 32 && hidden <= 256 ? route_tc_workspace_bytes(hidden) : 0;
}

int32_t be_qnet_route_tc(const be_qweights* W, int32_t n_tasks, int32_t n_tiers, const double* x,
                         int32_t batch, double epsilon, uint64_t philox_seed, uint64_t philox_counter,
                         float* q_out, uint8_t* action_out, void* workspace, int64_t* stats,
                         void* stream) {
    if (!W || !W->w1 || !W->b1 || !W->w2 || !W->b2 || !x || !action_out || !workspace)
        return set_error(BE_EINVAL, "NULL argument");
    if (n_tasks < 1 || n_tasks > BE_MAX_TASKS || n_tiers < 1 || n_tiers > BE_MAX_TIERS)
        return set_error(BE_EINVAL, "dimensions out of range");
    if (W->n_tasks != n_tasks || W->n_tiers != n_tiers)
        return set_error(BE_EINVAL, "expected input dim: the network's (n_tasks, n_tiers) differ from the router's");
    if (!route_tc_supported(n_tasks, n_tiers, W->hidden))
        return set_error(BE_EINVAL, "route_tc needs n_tiers <= 4, n_tasks + n_tiers + 2 <= 16 and hidden a "
                                    "multiple of 32 in [32, 256]; use be_qnet_route_f64");
    if (((uintptr_t)workspace & 15) != 0) return set_error(BE_EINVAL, "workspace must be 16-byte aligned");
    if (!(epsilon >= 0.0 && epsilon <= 1.0)) return set_error(BE_EINVAL, "epsilon must lie in [0, 1]");
    if (batch < 0) return set_error(BE_EINVAL, "batch must be >= 0");
    return launch_route_tc(W, n_tasks, n_tiers, x, batch, epsilon, philox_seed, philox_counter, q_out,
                           action_out, workspace, stats, (cudaStream_t)stream);
}

int32_t be_reduce_eval(const be_trace_soa* trace, const uint8_t* flags, const double* reward,
                       int32_t window, be_thresholds thresholds, int32_t n_buckets,
                       int64_t* win_counts, int64_t* n_windows, int64_t* bucket_miss,
                       int64_t* bucket_req, double* bucket_reward, void* stream) {
    if (!trace || !flags || !reward || !win_counts || !n_windows || !bucket_miss || !bucket_req ||
        !bucket_reward)
        return set_error(BE_EINVAL, "NULL argument");
    if (window < 1) return set_error(BE_EINVAL, "window must be >= 1");
    if (thresholds.n < 1 || thresholds.n > BE_MAX_THETA)
        return set_error(BE_EINVAL, "the number of thresholds must be in [1, 8]");
    if (n_buckets < 1) return set_error(BE_EINVAL, "n_buckets must be >= 1");
    if (!trace->seg_offsets) return set_error(BE_EINVAL, "trace segments missing");
    return launch_reduce(trace, flags, reward, window, thresholds.theta, thresholds.n, n_buckets, win_counts,
                         n_windows, bucket_miss, bucket_req, bucket_reward, (cudaStream_t)stream);
}

int32_t be_trace_gen_stable(int32_t n_envs, int64_t env_offset, int64_t n, int64_t ld,
                            const double* rate, int32_t n_tasks, uint64_t seed,
                            double* arrival_ms, uint8_t* task, void* stream) {
    if (!rate || !arrival_ms || !task) return set_error(BE_EINVAL, "NULL argument");
    if (n_envs < 1 || n < 0 || ld < n || n_tasks < 1 || n_tasks > 255 || env_offset < 0)
        return set_error(BE_EINVAL, "bad sizes");
    return launch_tracegen(n_envs, env_offset, n, ld, rate, n_tasks, seed, arrival_ms, task,
                           (cudaStream_t)stream);
}

int32_t be_trace_gen(const be_gen_cfg* cfg, int32_t n_envs, int64_t env_offset, int64_t ld,
                     uint64_t seed, double* arrival_ms, uint8_t* task, int64_t* n_events,
                     int64_t* seg_count, int64_t* seg_start, double* seg_rate, int32_t* status,
                     void* stream) {
    if (!cfg || !arrival_ms || !task || !n_events || !seg_count || !seg_start || !seg_rate || !status)
        return set_error(BE_EINVAL, "NULL argument");
    // InvalidParameterError cases of workload.py:131-134, :152-153, :181-182, :201-209
    if (n_envs < 1 || ld < 1 || env_offset < 0 || cfg->seg_capacity < 1)
        return set_error(BE_EINVAL, "bad sizes");
    if (cfg->n_tasks < 1 || cfg->n_tasks > 255) return set_error(BE_EINVAL, "n_tasks must be >= 1");
    if (cfg->n_task_ids < 0 || cfg->n_task_ids > BE_MAX_TASKS)
        return set_error(BE_EINVAL, "too many task_ids");
    for (int k = 0; k < cfg->n_task_ids; ++k)
        if (cfg->task_ids[k] < 0 || cfg->task_ids[k] >= cfg->n_tasks)
            return set_error(BE_EINVAL, "task_ids must be a nonempty subset of [0, n_tasks)");
    if (cfg->kind == BE_GEN_STABLE) {
        if (!cfg->rates || cfg->n_rates < 1) return set_error(BE_EINVAL, "rates must be nonempty and positive");
        if (!(cfg->hold_ms > 0) || !isfinite(cfg->hold_ms)) return set_error(BE_EINVAL, "hold_seconds must be positive");
        if (cfg->rate_ld != 0 && cfg->rate_ld < cfg->n_rates) return set_error(BE_EINVAL, "bad rate_ld");
    } else if (cfg->kind == BE_GEN_UNPRED_TIME || cfg->kind == BE_GEN_UNPRED_REQ) {
        if (cfg->n < 1) return set_error(BE_EINVAL, "n_requests must be >= 1");
        if (cfg->n > ld) return set_error(BE_EINVAL, "n_requests exceeds ld");
    } else {
        return set_error(BE_EINVAL, "unknown generator kind");
    }
    return launch_tracegen_general(cfg, n_envs, env_offset, ld, seed, arrival_ms, task, n_events,
                                   seg_count, seg_start, seg_rate, status, (cudaStream_t)stream);
}

}  // extern "C"
