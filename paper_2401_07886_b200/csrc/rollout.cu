// rollout.cu — fused greedy rollout (run_eval, evalkit.py:154-209) and the
// step-synchronous env API (ClusterSim reset/advance/observe/submit).
//
// be_rollout_greedy runs ONE persistent kernel for the whole trace batch:
// each warp pulls an environment id from a global counter, keeps the
// replica state in registers (one lane per replica) and walks its trace
// request by request — advance (with exact iteration skipping), score
// completions, estimate the rate, observe, Q-network forward + argmax in fp64,
// submit — then drains.  Trace reads are coalesced 32-request blocks
// broadcast with shuffles; per-tier sums and the replica argmin are REDUX ops.
#include <cuda_runtime.h>
#include <stdint.h>

#include "be_env.cuh"
#include "be_internal.h"

namespace be {

struct RolloutParams {
    be_cfg cfg;
    int32_t E;
    int64_t ld;
    const double* arrival;
    const uint8_t* task;
    const int64_t* n_events;
    const int64_t* seg_off;
    const int64_t* seg_start;
    const double* seg_rate;
    const uint8_t* forced;
    int32_t static_tier;
    int32_t H;
    const double* w1;
    const double* b1;
    const double* w2;
    const double* b2;
    be_records rec;
    Slot* rings;
    int32_t cap_log2;
    int32_t R;  // replicas per env (= active lanes)
    int32_t* env_counter;
    int32_t* status;  // [0] = error code, [1] = first failing env
};

__device__ __forceinline__ void raise_status(int32_t* status, int code, int env) {
    if (atomicCAS(&status[0], 0, code) == 0) status[1] = env;
}

// Shared-memory staging: Score, then W1 [D][H], b1 [H], W2^T [M][H], b2 [M].
template <int M>
__device__ void stage_weights(const RolloutParams& p, double* sw, int T) {
    const int H = p.H, D = T + M + 1;
    for (int k = threadIdx.x; k < D * H; k += blockDim.x) sw[k] = p.w1[k];
    double* sb1 = sw + D * H;
    for (int k = threadIdx.x; k < H; k += blockDim.x) sb1[k] = p.b1[k];
    double* sw2t = sb1 + H;
    for (int k = threadIdx.x; k < M * H; k += blockDim.x) {
        int m = k / H, j = k % H;
        sw2t[k] = p.w2[j * M + m];
    }
    double* sb2 = sw2t + M * H;
    for (int k = threadIdx.x; k < M; k += blockDim.x) sb2[k] = p.b2[k];
}

template <int M>
__global__ void __launch_bounds__(256) rollout_kernel(const RolloutParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Score& sc = *reinterpret_cast<Score*>(smem_raw);
    double* sw = reinterpret_cast<double*>(smem_raw + ((sizeof(Score) + 15) & ~size_t(15)));
    const int T = p.cfg.n_tasks;
    const bool policy = p.forced == nullptr && p.static_tier < 0;
    if (threadIdx.x < 32) load_score(sc, p.cfg);
    if (policy) stage_weights<M>(p, sw, T);
    __syncthreads();
    const int H = p.H, D = T + M + 1;
    const double* sW1 = sw;
    const double* sb1 = sw + D * H;
    const double* sW2t = sb1 + H;
    const double* sb2 = sW2t + M * H;

    const int lane = threadIdx.x & 31;
    const TierC tc = lane_tier(p.cfg, lane);
    const bool active_lane = tc.tier >= 0;
    const uint32_t mask = (1u << p.cap_log2) - 1u;
    const bool skip = p.cfg.skip_ahead != 0;
    const bool true_rate = p.cfg.estimator_true_rate != 0;
    const bool reset_segs = p.cfg.reset_between_segments != 0;

    for (;;) {
        int env = 0;
        if (lane == 0) env = atomicAdd(p.env_counter, 1);
        env = __shfl_sync(FULL, env, 0);
        if (env >= p.E) break;

        Slot* ring = p.rings + ((size_t)env * p.R + (active_lane ? lane : 0)) * ((size_t)mask + 1);
        RecOut out{p.rec.flags, p.rec.reward, p.rec.realized, (int64_t)env * p.ld};
        const int64_t base = (int64_t)env * p.ld;
        const int64_t n = p.n_events ? p.n_events[env] : p.ld;
        int64_t seg = p.seg_off[env];
        const int64_t seg_end = p.seg_off[env + 1];
        int64_t next_seg = seg < seg_end ? p.seg_start[seg] : INT64_MAX;
        double cur_rate = __longlong_as_double(0x7ff8000000000000LL);  // NaN until a mark applies
        Rep r;
        rep_reset(r);
        r.head = 0;
        Estimator est;
        est.n = 0;
#pragma unroll
        for (int k = 0; k < 5; ++k) est.w[k] = 0.0;
        bool ok = true;   // ring capacity / iteration counter
        bool bad = false; // forced action out of range

        double pf_arr = 0.0;
        int pf_task = 0, pf_forced = 0;
        for (int64_t i = 0; i < n; ++i) {
            const int sub = (int)(i & 31);
            if (sub == 0) {  // coalesced 32-request prefetch
                int64_t ii = i + lane;
                if (ii < n) {
                    pf_arr = __ldg(p.arrival + base + ii);
                    pf_task = __ldg(p.task + base + ii);
                    if (p.forced) pf_forced = __ldg(p.forced + base + ii);
                }
            }
            const double U = __shfl_sync(FULL, pf_arr, sub);
            const int task = __shfl_sync(FULL, pf_task, sub);
            // segment boundaries (evalkit.py:186-192)
            while (i >= next_seg) {
                if (reset_segs && i == next_seg && i > 0) {
                    if (active_lane) ok &= advance_lane(r, tc, __longlong_as_double(0x7ff0000000000000LL), ring, mask, sc, out, skip);
                    rep_reset(r);
                    est.n = 0;
                }
                cur_rate = p.seg_rate[seg];
                ++seg;
                next_seg = seg < seg_end ? p.seg_start[seg] : INT64_MAX;
            }
            if (active_lane) ok &= advance_lane(r, tc, U, ring, mask, sc, out, skip);
            const double rate = estimator_observe(est, U, true_rate, cur_rate, p.cfg.prior_rate);
            int obs[M];
#pragma unroll
            for (int m = 0; m < M; ++m) obs[m] = (int)__reduce_add_sync(FULL, (tc.tier == m) ? (unsigned)r.count : 0u);
            int tier;
            if (p.forced) {
                tier = __shfl_sync(FULL, pf_forced, sub);
            } else if (p.static_tier >= 0) {
                tier = p.static_tier;
            } else {
                double xt[M], q[M];
#pragma unroll
                for (int m = 0; m < M; ++m) xt[m] = __ddiv_rn((double)obs[m], p.cfg.batch_scales[m]);
                const double xr = __ddiv_rn(rate, p.cfg.rate_scale);
                qnet_warp<M>(sW1, sb1, sW2t, sb2, T, H, task, xt, xr, q);
                tier = argmax_first<M>(q);
                if (p.rec.q && lane < M) {
#pragma unroll
                    for (int m = 0; m < M; ++m)
                        if (lane == m) p.rec.q[(base + i) * M + m] = q[m];
                }
            }
            if (p.rec.obs && lane < M) {
#pragma unroll
                for (int m = 0; m < M; ++m)
                    if (lane == m) p.rec.obs[(base + i) * M + m] = obs[m];
            }
            if (p.rec.rate && lane == 0) p.rec.rate[base + i] = rate;
            // replica argmin of (len(active), len(queue), id) == argmin (count, lane)
            unsigned key = (tc.tier == tier) ? (((unsigned)r.count << 5) | (unsigned)lane) : 0xffffffffu;
            unsigned best = __reduce_min_sync(FULL, key);
            if (best == 0xffffffffu) {  // tier out of range (forced action)
                bad = true;
            } else if ((int)(best & 31u) == lane) {
                ok &= submit_lane(r, tc, U, (uint32_t)i | ((uint32_t)task << 24), ring, mask);
            }
            if (!__all_sync(FULL, ok) || bad) break;
        }
        if (active_lane && ok && !bad)
            ok &= advance_lane(r, tc, __longlong_as_double(0x7ff0000000000000LL), ring, mask, sc, out, skip);
        if (bad && lane == 0) raise_status(p.status, BE_EINVAL, env);
        else if (!__all_sync(FULL, ok) && lane == 0) raise_status(p.status, BE_ECAPACITY, env);
    }
}

size_t rollout_smem_bytes(int T, int M, int H, bool policy) {
    size_t s = (sizeof(Score) + 15) & ~size_t(15);
    if (policy) s += sizeof(double) * ((size_t)(T + M + 1) * H + H + (size_t)M * H + M);
    return s;
}

template <int M>
static int launch_rollout_m(const RolloutParams& p, size_t smem, cudaStream_t st, int sms) {
    auto kern = rollout_kernel<M>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute");
    }
    const int threads = 256;
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    if (e != cudaSuccess) return set_cuda_error(e, "occupancy");
    if (per_sm < 1) per_sm = 1;
    long long warps_needed = p.E;
    long long blocks = (long long)sms * per_sm;
    long long max_blocks = (warps_needed + threads / 32 - 1) / (threads / 32);
    if (blocks > max_blocks) blocks = max_blocks;
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, threads, smem, st>>>(p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e, "rollout launch");
    return BE_OK;
}

int launch_rollout(be_env* env, const be_trace_soa* tr, const be_qweights* W, int static_tier,
                   const uint8_t* forced, const be_records* rec, cudaStream_t st) {
    RolloutParams p{};
    p.cfg = env->cfg;
    p.E = tr->n_envs;
    p.ld = tr->ld;
    p.arrival = tr->arrival_ms;
    p.task = tr->task;
    p.n_events = tr->n_events;
    p.seg_off = tr->seg_offsets;
    p.seg_start = tr->seg_start;
    p.seg_rate = tr->seg_rate;
    p.forced = forced;
    p.static_tier = static_tier;
    p.rec = *rec;
    p.rings = reinterpret_cast<Slot*>(env->rings);
    p.cap_log2 = env->cap_log2;
    p.R = env->R;
    p.env_counter = env->d_counter;
    p.status = env->d_status;
    bool policy = forced == nullptr && static_tier < 0;
    int T = env->cfg.n_tasks, M = env->cfg.n_tiers;
    if (policy) {
        p.H = W->hidden;
        p.w1 = W->w1;
        p.b1 = W->b1;
        p.w2 = W->w2;
        p.b2 = W->b2;
    }
    size_t smem = rollout_smem_bytes(T, M, policy ? p.H : 0, policy);
    cudaError_t e = cudaMemsetAsync(env->d_counter, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return set_cuda_error(e, "memset counter");
    switch (M) {
        case 1: return launch_rollout_m<1>(p, smem, st, env->sms);
        case 2: return launch_rollout_m<2>(p, smem, st, env->sms);
        case 3: return launch_rollout_m<3>(p, smem, st, env->sms);
        case 4: return launch_rollout_m<4>(p, smem, st, env->sms);
        case 5: return launch_rollout_m<5>(p, smem, st, env->sms);
        case 6: return launch_rollout_m<6>(p, smem, st, env->sms);
        case 7: return launch_rollout_m<7>(p, smem, st, env->sms);
        case 8: return launch_rollout_m<8>(p, smem, st, env->sms);
        default: return set_error(BE_EINVAL, "n_tiers out of range");
    }
}

}  // namespace be
