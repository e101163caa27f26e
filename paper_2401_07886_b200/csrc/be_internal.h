// be_internal.h — host-side internals shared by the translation units.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "be200.h"

// Skip table (exact iteration skipping, be_env.cuh): D per (tier, n in
// [0, max_batch], binade e in [SKIP_ELO, SKIP_ELO + SKIP_NB)), doubles.
constexpr int SKIP_NB = 32;
constexpr int SKIP_ELO = -2;
// largest packed fp64 Q-weight block (QLayout: (T + 2M + 1) H + M doubles)
constexpr size_t QPACK_MAX_DOUBLES = (size_t)(BE_MAX_TASKS + 2 * BE_MAX_TIERS + 1) * 1024 + BE_MAX_TIERS;

struct be_env {
    be_cfg cfg;
    int32_t E;        // environments
    int32_t R;        // replicas per env (lanes used per warp)
    int32_t device;
    int32_t sms;      // multiprocessor count
    int32_t cap_log2; // per-replica FIFO ring capacity = 1 << cap_log2
    void* rings;      // [E][R][cap] Slot (16 B)
    size_t ring_bytes;
    void* reps;       // step API: [E][R] Rep
    void* envs;       // step API: [E] EnvState
    int32_t* d_counter;
    int32_t* d_status;  // [0] code, [1] env
    double* d_skip;     // skip table [sum_m (max_batch_m + 1)][SKIP_NB], NULL = skipping off
    int32_t skip_rows;
    unsigned long long* d_screen;  // [2] screened decisions, fp64 fallbacks (rollout)
    double* d_qpack;    // packed fp64 Q weights for the screened rollout's fallback (max size)
    int32_t last_plan[8];  // be_env_rollout_plan: what the last be_rollout_greedy launched
    int32_t exact_mul;     // obs * (1/s_m) == obs / s_m for every reachable obs (<= R_m x ring
                           // capacity) and tier m: encode may multiply (policy.py:63)
};

namespace be {
// Programmatic dependent launch (PDL): a kernel launched with launch_pdl may be
// scheduled while its stream predecessor is still running; it calls pdl_wait()
// before touching anything the predecessor wrote, and pdl_trigger() lets its own
// successor be scheduled early.  Hides the kernel-boundary latency of the
// launch-bound training iteration (six dependent kernels per iteration).
#ifndef BE_PDL_IN_GRAPHS
#define BE_PDL_IN_GRAPHS 1
#endif
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = BE_PDL_IN_GRAPHS ? 1 : 0;
    if (!BE_PDL_IN_GRAPHS) {  // programmatic edges only for eager launches
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(st, &cs);
        cfg.numAttrs = cs == cudaStreamCaptureStatusNone ? 1 : 0;
    }
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
#endif

// Host-side derived reward constants shipped in kernel parameters (see Score).
struct ScoreAux {
    double hit_tau[BE_MAX_TASKS * BE_MAX_TIERS];
};
void make_score_aux(const be_cfg& c, ScoreAux* aux);
double tau_le(double theta, double w);
double tau_ge(double theta, double w);
int set_error(int code, const char* msg);
// Host: tabulate the per-cycle increment D(tier, n, binade) (0 = do not skip).
int build_skip_table(const be_cfg& c, double* out /* [rows][SKIP_NB] or NULL */);
int set_cuda_error(cudaError_t e, const char* where);
int launch_rollout(be_env* env, const be_trace_soa* tr, const be_qweights* W, int static_tier,
                   const uint8_t* forced, const be_records* rec, cudaStream_t st);
size_t rollout_smem_bytes(int T, int M, int H, bool policy, int skip_rows = 0, bool screen = false);
int launch_env_reset(be_env* env, const uint8_t* mask, cudaStream_t st);
int launch_env_step(be_env* env, const double* arrival, const uint8_t* task,
                    const double* true_rate, const uint8_t* forced, const be_qweights* W,
                    int static_tier, double epsilon, uint64_t seed, uint64_t counter,
                    int64_t rec_ld, const be_records* rec, int32_t* obs_out, double* rate_out,
                    uint8_t* action_out, double* q_out, double* x_out, cudaStream_t st);
int launch_env_drain(be_env* env, int64_t rec_ld, const be_records* rec, cudaStream_t st,
                     const uint8_t* mask = nullptr, int new_segment = 0);
// be_train_iteration with the fp64 router: the replay commit (ReplayBuffer
// resolve_reward / resolve_next_state -> push, trainer.py:143-156) fused into the env
// step — the step's completed transitions go straight into the ring (same slots as
// commit_fused_kernel: env-id order, request-id order within an env)
struct StepCommitArgs {
    int64_t capacity;
    double *rs, *rs2, *rr, *rc;  // ring states / next states / rewards / continue flags
    uint8_t* ra;                 // ring actions
    int64_t* low;                // [E] oldest request still in flight
    int64_t* ring_state;         // cursor, size, total, last count, in-flight high-water mark
    int32_t* status;             // learner status (pending-store overflow)
    unsigned long long* scan;    // [ceil(E / 16)] decoupled look-back state
    unsigned* epoch;             // scan epoch (advanced by the last block)
    int32_t list_cap;            // block transition-list entries used (<= SC_LIST; set at launch)
    // virtual block ids from a ticket (when the grid may exceed the CTAs resident at once):
    // [2] counters used by alternate launches (epoch parity), each reset one launch ahead
    unsigned* vticket;
    int32_t use_ticket;
};
int launch_env_step_dev(be_env* env, const double* arrival, const uint8_t* task,
                        const double* true_rate, const be_qweights* W, uint64_t seed,
                        const int64_t* iter_dev, double eps_start, double eps_end, int64_t eps_decay,
                        int32_t pending_P, int64_t rec_ld, const be_records* rec, uint8_t* action_base,
                        double* x_base, cudaStream_t st, const struct WorkloadArgs* wl = nullptr,
                        int phase = 0, float* tc_img = nullptr, int64_t* crange = nullptr,
                        const StepCommitArgs* commit = nullptr);
bool env_step_commit_supported(const be_env* env);
// pack W into env->d_qpack (QLayout) for the env step's fp64 decision
int launch_stage_qpack(be_env* env, const be_qweights* W, cudaStream_t st);
// the training step with the decision on the tensor cores (tc_img != NULL above):
// shared-memory size and the kernel attribute (set before any graph capture)
size_t step_tc_smem_bytes(int H);
void step_tc_prepare(int M, int H);
// split step: phase 1 = advance + observe + encode into x_out (no decision), phase 2 =
// submit the decisions in `action` (a router runs in between)
int launch_env_step_split(be_env* env, int phase, const double* arrival, const uint8_t* task,
                          const double* true_rate, uint8_t* action, double* x_out, int32_t* obs_out,
                          double* rate_out, int64_t rec_ld, const be_records* rec, cudaStream_t st);
size_t env_state_bytes_per_env(int R);
int launch_reduce(const be_trace_soa* tr, const uint8_t* flags, const double* reward, int window,
                  const double* thetas, int n_theta, int n_buckets, int64_t* win_counts,
                  int64_t* n_windows, int64_t* bucket_miss, int64_t* bucket_req,
                  double* bucket_reward, cudaStream_t st);
int launch_route(const be_qweights* W, int T, int M, const double* x, int B, double eps,
                 uint64_t seed, uint64_t counter, double* q_out, uint8_t* a_out, cudaStream_t st);
bool route_tc_supported(int T, int M, int H);
// sets the router kernel's shared-memory attribute ahead of any CUDA-graph capture
void route_tc_prepare(int T, int M, int H);
size_t route_tc_workspace_bytes(int H);
int launch_route_tc(const be_qweights* W, int T, int M, const double* x, int B, double eps, uint64_t seed,
                    uint64_t counter, float* q_out, uint8_t* a_out, void* workspace, int64_t* stats,
                    cudaStream_t st);
// device-iteration form (be_train_iteration, router = tensor cores): x / a_out are the
// pending store's bases, slot *iter_dev % pending_P; epsilon_at(*iter_dev) and the
// Philox counter *iter_dev are read on the device, so a CUDA graph replays it unchanged
int launch_route_tc_dev(const be_qweights* W, int T, int M, const double* x_base, int B, uint64_t seed,
                        const int64_t* iter_dev, double eps_start, double eps_end, int64_t eps_decay,
                        int32_t pending_P, uint8_t* a_base, void* workspace, int64_t* stats, cudaStream_t st);
int launch_tracegen(int E, int64_t env_offset, int64_t n, int64_t ld, const double* rate, int n_tasks, uint64_t seed,
                    double* arrival, uint8_t* task, cudaStream_t st);
int launch_tracegen_general(const be_gen_cfg* cfg, int E, int64_t env_offset, int64_t ld,
                            uint64_t seed, double* arrival, uint8_t* task, int64_t* n_events,
                            int64_t* seg_count, int64_t* seg_start, double* seg_rate,
                            int32_t* status, cudaStream_t st);
int launch_selection(const be_trace_soa* tr, const uint8_t* flags, int T, int M, int K,
                     int64_t* counts, cudaStream_t st);
int launch_windowed(const be_trace_soa* tr, const double* reward, int w, double* out, cudaStream_t st);
}  // namespace be
