// rollout.cu — fused greedy rollout (run_eval, evalkit.py:154-209).
//
// be_rollout_greedy runs ONE persistent kernel for the whole trace batch.
// Each warp hosts 32 / LPE environments (LPE = lanes per env: 16 when the
// cluster has <= 16 replicas — the shipped 3 x 4 — else 32); each group of
// LPE lanes pulls an environment id from a global counter, keeps one replica
// per lane in registers and walks that env's trace request by request:
// advance (with exact iteration skipping), score completions, rate signal,
// observe, Q-network forward + argmax in fp64, submit — then drains and
// pulls the next env.  Two envs per warp halve the per-env cost of every
// warp-wide instruction (the Q-network, reductions, bookkeeping).  Trace
// reads are coalesced LPE-request blocks broadcast with shuffles; per-tier
// sums and the replica argmin are REDUX ops.
#include <cuda_runtime.h>
#include <stdint.h>
#include <climits>
#include <math.h>
#include <stdlib.h>

#include "be_env.cuh"
#include "be_internal.h"

// Occupancy (A/B on B200, config-4 bench, rollout ms): 256 threads x 3 CTAs per SM
// (80 registers, small spills) with the skip table read through L1 373; 128 x 6 377;
// 256 x 2 (128 registers) 393; 256 x 3 with the skip table staged in shared memory
// 433 (the staging shrinks L1, which caches the skip table and the FIFO rings);
// 128 x 7 / x 8 420 / 416 (spills).
// The estimated-rate variant keeps the 5-arrival window live and spills at 80
// registers (config 2, 4096 unpredictable-1 envs: 1.21e9 at 2 CTAs/SM with the skip
// table in shared memory, 0.84e9 at 3 CTAs/SM), so it keeps 2 CTAs/SM and stages the
// skip table; the true-rate variant runs 3 CTAs/SM and reads it through L1 when the
// batch fills them (config 4), else 2 CTAs/SM (config 1: 18 envs, latency-bound).
#ifndef BE_RING_PER_GROUP
#define BE_RING_PER_GROUP 1
#endif
#ifndef BE_TRACE_EVICT_FIRST
#define BE_TRACE_EVICT_FIRST 1
#endif
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ double ld_stream_f64(const double* p, uint64_t pol) {
    double v;
    asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int ld_stream_u8(const uint8_t* p, uint64_t pol) {
    unsigned short v;
    asm volatile("ld.global.cg.L2::cache_hint.u8 %0, [%1], %2;" : "=h"(v) : "l"(p), "l"(pol));
    return (int)v;
}
#ifndef BE_ROLLOUT_MINB
#define BE_ROLLOUT_MINB 3  // resident CTAs per SM the register allocation is capped for (true rate)
#endif
#ifndef BE_ROLLOUT_MINB_EST
#define BE_ROLLOUT_MINB_EST 2  // the same for the estimated-rate variant
#endif
#ifndef BE_ROLLOUT_THREADS
#define BE_ROLLOUT_THREADS 256
#endif
#ifndef BE_SKIP_SMEM_MAX
#define BE_SKIP_SMEM_MAX 0  // true rate: stage the skip table if the CTA's shared memory stays below (0: never)
#endif
#ifndef BE_SKIP_SMEM_MAX_EST
#define BE_SKIP_SMEM_MAX_EST (100 * 1024)  // estimated rate: the same bound
#endif

namespace be {

struct RolloutParams {
    be_cfg cfg;
    ScoreAux aux;
    int32_t E;
    int64_t ld;
    const double* arrival;
    const uint8_t* task;
    const int64_t* n_events;
    const int64_t* seg_off;
    const int64_t* seg_start;
    const double* seg_rate;
    const uint8_t* forced;
    const int32_t* env_ready;  // streamed upload: wait for env_ready[env / envs_per_ready] >= ready_value
    int32_t envs_per_ready, ready_value;
    int32_t static_tier;
    int32_t H;
    const double* w1;
    const double* b1;
    const double* w2;
    const double* b2;
    be_records rec;
    Slot* rings;
    int32_t cap_log2;
    int32_t R;  // replicas per env (= active lanes per group)
    int32_t* env_counter;
    int32_t* status;  // [0] = error code, [1] = first failing env
    const double* skip;  // skip table (global), NULL = skipping off
    int32_t skip_rows;
    int32_t skip_smem;   // 1 = stage the skip table in shared memory
    int32_t screen;      // 1 = certified fp32 decision screen (qnet_screen) + fp64 fallback
    double inv_scale[BE_MAX_TIERS];  // 1 / batch_scales[m] (host IEEE division)
    double inv_rate_scale;           // 1 / rate_scale
    int32_t ring_per_group;  // 1: replica rings indexed by the persistent group, else by env
    int32_t throughput;      // 1: the throughput variant (3 CTAs/SM) — set by launch_rollout
    int32_t exact_mul;   // 1 = obs * (1/s) == obs / s for every reachable obs and tier
                         // (be_env.exact_mul; always so for power-of-two scales); the
                         // throughput variant (OCC = 1) is launched only then
    unsigned long long* screen_stats;  // [2] decisions screened, fp64 fallbacks (nullable)
    int32_t pack_obs;    // 1: per-tier queue sums fit 10-bit fields (observe with one REDUX)
    const double* qpack;  // screen on: the fp64 fallback's packed weights (QLayout) in global
                          // memory (L1/L2-resident), so shared memory holds only the screen
};

__device__ __forceinline__ void raise_status(int32_t* status, int code, int env) {
    if (atomicCAS(&status[0], 0, code) == 0) status[1] = env;
}

// TR: 1 = true-rate estimator (the arrival window is never read, so its registers
// are not allocated), 0 = estimated rate (workload.py:234-247).
// OCC: 1 = the throughput variant (BE_ROLLOUT_MINB CTAs/SM, fewer registers), for
// batches with enough envs to fill them; 0 = the latency variant (2 CTAs/SM, 128
// registers, no spills) — a small batch is bound by its slowest env's serial chain.
template <int M, int LPE, int TR, int OCC>
__global__ void __launch_bounds__(BE_ROLLOUT_THREADS, OCC ? BE_ROLLOUT_MINB : BE_ROLLOUT_MINB_EST)
    rollout_kernel(const RolloutParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Score& sc = *reinterpret_cast<Score*>(smem_raw);
    double* sw = reinterpret_cast<double*>(smem_raw + ((sizeof(Score) + 15) & ~size_t(15)));
    const int T = p.cfg.n_tasks;
    const bool policy = p.forced == nullptr && p.static_tier < 0;
    if (threadIdx.x < 32) load_score(sc, p.cfg, p.aux);
    const int H = p.H;
    // screen on: [Score | fp32 screen tables | skip table], fp64 weights in global (qpack);
    // screen off: [Score | fp64 weights | skip table]
    const bool screen = policy && p.screen;
    if (policy && !screen) stage_qnet<M>(p.w1, p.b1, p.w2, p.b2, T, H, sw);
    const double* qw = screen ? p.qpack : sw;
    float* sf = reinterpret_cast<float*>(sw);
    if (screen) stage_qscreen<M, LPE>(p.w1, p.b1, p.w2, p.b2, T, H, sf);
    const double* skip_tab = p.skip;
    if (p.skip && p.skip_smem) {  // after the weights (policy) or right after Score
        double* st = screen ? reinterpret_cast<double*>(sf + ((QsLayout<M>::floats(T, H) + 3) & ~size_t(3)))
                            : sw + (policy ? QLayout<M>::doubles(T, H) : 0);
        for (int k = threadIdx.x; k < p.skip_rows * SKIP_NB; k += blockDim.x) st[k] = p.skip[k];
        skip_tab = st;
    }
    __syncthreads();
    unsigned n_screened = 0, n_fallback = 0;  // per group leader (screen_stats)

    const int lane = threadIdx.x & 31;
    const int gl = lane & (LPE - 1);       // lane within the env group
    const int grp = LPE == 32 ? 0 : lane / LPE;
    const int g0 = grp * LPE;              // first lane of the group
    const int my_group = (int)((blockIdx.x * blockDim.x + threadIdx.x) / LPE);  // persistent group id
    const unsigned gmask = LPE == 32 ? FULL : (0xffffu << g0);
    const TierC tc = lane_tier(p.cfg, gl, skip_tab);
    const bool active_lane = tc.tier >= 0;
    const uint32_t mask = (1u << p.cap_log2) - 1u;
#if BE_TRACE_EVICT_FIRST
    const uint64_t l2_first = l2_policy_evict_first();
#endif
    constexpr bool true_rate = TR != 0;
    const bool reset_segs = p.cfg.reset_between_segments != 0;
    const double INF = __longlong_as_double(0x7ff0000000000000LL);
    // encode (policy.py:63-64) divides by the scales: a / s as a * (1/s) plus one
    // Markstein correction step (residual a - q s exact by FMA, q + r (1/s) rounded
    // once) — the correctly rounded quotient, bit-identical to __ddiv_rn for every
    // scale (not only the power-of-two ones), two DFMA instead of a DDIV sequence
    // 1/s precomputed on the host (IEEE division there too) and read as constant-bank
    // operands: no registers held across the request loop
#define INV_SCALE(m) p.inv_scale[m]
#define INV_RATE_SCALE p.inv_rate_scale
    auto div_by = [](double a, double s, double inv) {
        const double q = __dmul_rn(a, inv);
        return __fma_rn(__fma_rn(-q, s, a), inv, q);
    };
    // the product IS the quotient for every reachable obs (the shipped 128/32/8 are
    // powers of two); the throughput variant relies on it (host-checked)
    const bool mul_ok = OCC ? true : p.exact_mul != 0;

    // per-group ("group-uniform") env state
    int env = -1;
    bool need = true, dead = false;
    // request indices are 32-bit (ld <= 2^24, checked at the API); segment CSR offsets 64-bit
    int64_t base = 0, seg = 0, seg_end = 0;

    int n = 0, i = 0, next_seg = INT_MAX;
    auto seg_mark = [&](int64_t k) { return k < seg_end ? (int)min(p.seg_start[k], (int64_t)INT_MAX) : INT_MAX; };
    double cur_xr = 0.0;  // true-rate mode: the current segment's rate / rate_scale (NaN before a mark)
    Slot* ring = p.rings;
    Rep r;
    rep_reset(r);
    Estimator est;
    est.n = 0;
#pragma unroll
    for (int k = 0; k < 5; ++k) est.w[k] = 0.0;
    bool ok = true, bad = false;
    double pf_arr = 0.0;
    int pf_task = 0, pf_forced = 0;

    for (;;) {
        // ---- (re)fill groups that finished their env
        int got = (need && gl == 0) ? atomicAdd(p.env_counter, 1) : 0;
        if (p.env_ready && need && gl == 0 && got < p.E) {
            // streamed upload: this env's rows are readable once its chunk's flag is set
            const int32_t* f = p.env_ready + got / p.envs_per_ready;
            unsigned long long t0, now;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            for (;;) {
                int v;
                asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
                if (v >= p.ready_value) break;
                if (*(volatile int32_t*)p.status != 0) break;  // already failed: do not wait again
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                if (now - t0 > 5000000000ull) {  // 5 s: the upload never arrived
                    raise_status(p.status, BE_ECUDA, got);
                    break;
                }
                __nanosleep(256);
            }
        }
        got = __shfl_sync(FULL, got, g0);
        if (need) {
            need = false;
            if (got >= p.E) {
                dead = true;
            } else {
                env = got;
                base = (int64_t)env * p.ld;

                n = (int)(p.n_events ? p.n_events[env] : p.ld);
                i = 0;
                seg = p.seg_off[env];
                seg_end = p.seg_off[env + 1];
                next_seg = seg_mark(seg);
                cur_xr = __longlong_as_double(0x7ff8000000000000LL);  // NaN until a mark applies
                ring = p.rings + ((size_t)(p.ring_per_group ? my_group : env) * p.R + (active_lane ? gl : 0)) *
                                     ((size_t)mask + 1);
                rep_reset(r);
                r.head = 0;
                est.n = 0;
                ok = true;
                bad = false;
            }
        }
        if (__all_sync(FULL, dead)) break;
        const bool live = !dead && i < n;
        const RecOut out = RecOut::row(p.rec, base);

        // ---- one request for every live group (evalkit.py:185-205)
        const int sub = (int)(i & (LPE - 1));
        if (live && sub == 0) {  // coalesced LPE-request prefetch
            const int ii = i + gl;
            if (ii < n) {
                // through L2 only (ld.global.cg): rows that arrive during the kernel
                // (streamed upload) are never served from a stale L1 line; read-once
                // rows gain nothing from L1 anyway (A/B: 1% faster than a branch)
#if BE_TRACE_EVICT_FIRST
                // read-once trace rows: evict-first in L2, so the 9 B/request stream does
                // not push the FIFO rings, records and spill lines of the envs in flight out
                pf_arr = ld_stream_f64(p.arrival + base + ii, l2_first);
                pf_task = ld_stream_u8(p.task + base + ii, l2_first);
#else
                pf_arr = __ldcg(p.arrival + base + ii);
                pf_task = __ldcg(p.task + base + ii);
#endif
                if (pf_task >= T) {  // task id outside the reward spec (encode raises,
                    bad = true;      // policy.py:57-58): the env fails with BE_EINVAL
                    pf_task = 0;
                }
                if (p.forced) pf_forced = __ldg(p.forced + base + ii);
            }
        }
        const double U = __shfl_sync(FULL, pf_arr, g0 + sub);
        int task = __shfl_sync(FULL, pf_task, g0 + sub);
        const int ftier = p.forced ? __shfl_sync(FULL, pf_forced, g0 + sub) : 0;
        if (!live) task = 0;  // keep idle groups' shared-memory reads in range
        double rate = 0.0;
        if (live) {
            while (i >= next_seg) {  // segment boundaries (evalkit.py:186-192)
                if (reset_segs && i == next_seg && i > 0) {
                    if (active_lane) ok &= advance_lane(r, tc, INF, ring, mask, sc, out);
                    rep_reset(r);
                    est.n = 0;
                }
                if (true_rate) cur_xr = __ddiv_rn(p.seg_rate[seg], p.cfg.rate_scale);  // once per segment
                ++seg;
                next_seg = seg_mark(seg);
            }
            if (active_lane) ok &= advance_lane(r, tc, U, ring, mask, sc, out);
            // true-rate mode never reads the arrival window (workload.py:241-242)
            if (!true_rate) rate = estimator_observe(est, U, false, 0.0, p.cfg.prior_rate);
        }
        int obs[M];
        if (M <= 3 && p.pack_obs) {
            // one REDUX per group: tier m's replica counts in bits [10m, 10m + 10) (the host
            // checked replicas x ring capacity < 1024 for every tier, so no field overflows)
            const unsigned s = group_sum<LPE>(live && active_lane ? (unsigned)r.count << (10 * tc.tier) : 0u, grp);
#pragma unroll
            for (int m = 0; m < M; ++m) obs[m] = (int)((s >> (10 * m)) & 1023u);
        } else {
#pragma unroll
            for (int m = 0; m < M; ++m)
                obs[m] = (int)group_sum<LPE>((live && tc.tier == m) ? (unsigned)r.count : 0u, grp);
        }
        int tier;
        if (p.forced) {
            tier = ftier;
        } else if (p.static_tier >= 0) {
            tier = p.static_tier;
        } else {
            double xt[M], q[M];
#pragma unroll
            for (int m = 0; m < M; ++m)
                xt[m] = mul_ok ? __dmul_rn((double)obs[m], INV_SCALE(m))
                                    : div_by((double)obs[m], p.cfg.batch_scales[m], INV_SCALE(m));
            const double xr = true_rate ? cur_xr : div_by(rate, p.cfg.rate_scale, INV_RATE_SCALE);
            if (screen) {
                // certified fp32 decision; exact fp64 evaluation only where it cannot certify
                const bool sure = qnet_screen<M, LPE>(sf, T, H, task, xt, xr, tier);
                if (__ballot_sync(FULL, live && !sure)) {
                    qnet_group<M, LPE>(qw, T, H, task, xt, xr, q);
                    if (!sure) tier = argmax_first<M>(q);
                }
                if (live && gl == 0) {
                    ++n_screened;
                    n_fallback += sure ? 0u : 1u;
                }
            } else {
                qnet_group<M, LPE>(sw, T, H, task, xt, xr, q);
                tier = argmax_first<M>(q);
            }
            if (live && p.rec.q && gl < M) {
#pragma unroll
                for (int m = 0; m < M; ++m)
                    if (gl == m) p.rec.q[(base + i) * M + m] = q[m];
            }
        }
        if (live && p.rec.obs && gl < M) {
#pragma unroll
            for (int m = 0; m < M; ++m)
                if (gl == m) p.rec.obs[(base + i) * M + m] = obs[m];
        }
        if (live && p.rec.rate && gl == 0) {  // true-rate mode: the segment's rate (NaN before a mark)
            p.rec.rate[base + i] = !true_rate ? rate : cur_xr == cur_xr ? p.seg_rate[seg - 1] : cur_xr;
        }
        // replica argmin of (len(active), len(queue), id) == argmin (count, replica)
        const unsigned key = (live && tc.tier == tier) ? (((unsigned)r.count << 5) | (unsigned)gl) : 0xffffffffu;
        const unsigned best = group_min<LPE>(key, grp);
        if (live) {
            if (best == 0xffffffffu) {  // tier out of range (forced action)
                bad = true;
            } else if ((int)(best & 31u) == gl) {
                ok &= submit_lane(r, tc, U, (uint32_t)i | ((uint32_t)task << 24), ring, mask);
            }
            ++i;
        }
        // ---- group bookkeeping: failure or end of trace -> drain, next env
        const unsigned fb = __ballot_sync(FULL, live && (!ok || bad));
        const bool gfail = (fb & gmask) != 0;
        const bool gbad = fb != 0 && (__ballot_sync(FULL, live && bad) & gmask) != 0;  // fb: warp-uniform
        if (!dead && (gfail || i >= n)) {
            if (!gfail && active_lane) ok &= advance_lane(r, tc, INF, ring, mask, sc, out);
            const bool drain_fail = (__ballot_sync(gmask, !ok) & gmask) != 0;
            if (gl == 0) {
                if (gbad) raise_status(p.status, BE_EINVAL, env);
                else if (gfail || drain_fail) raise_status(p.status, BE_ECAPACITY, env);
            }
            need = true;
        }
    }
    if (p.screen_stats && screen) {
        const unsigned a = __reduce_add_sync(FULL, n_screened), b = __reduce_add_sync(FULL, n_fallback);
        if (lane == 0) {
            atomicAdd(&p.screen_stats[0], (unsigned long long)a);
            atomicAdd(&p.screen_stats[1], (unsigned long long)b);
        }
    }
}

size_t rollout_smem_bytes(int T, int M, int H, bool policy, int skip_rows, bool screen) {
    size_t s = (sizeof(Score) + 15) & ~size_t(15);
    if (policy && !screen) s += sizeof(double) * ((size_t)(T + 2 * M + 1) * H + M);  // QLayout<M>::doubles
    if (policy && screen)  // QsLayout<M>::floats, rounded to 16 bytes
        s += sizeof(float) * (((size_t)(2 * T + 2 * M) * H + T + (M + 1) + M + 3) & ~size_t(3));
    s += sizeof(double) * (size_t)skip_rows * SKIP_NB;
    return s;
}

template <int M, int LPE>
static int launch_rollout_m(const RolloutParams& p, size_t smem, cudaStream_t st, int sms, int32_t* plan) {
    const bool many = p.throughput != 0;  // chosen by launch_rollout
    auto kern = !p.cfg.estimator_true_rate ? rollout_kernel<M, LPE, 0, 0>
                : many                     ? rollout_kernel<M, LPE, 1, 1>
                                           : rollout_kernel<M, LPE, 1, 0>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute");
    }
    const int threads = BE_ROLLOUT_THREADS;
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    if (e != cudaSuccess) return set_cuda_error(e, "occupancy");
    if (per_sm < 1) per_sm = 1;
    const long long groups_per_block = threads / LPE;
    long long blocks = (long long)sms * per_sm;
    const long long max_blocks = (p.E + groups_per_block - 1) / groups_per_block;
    if (blocks > max_blocks) blocks = max_blocks;
    if (blocks < 1) blocks = 1;
    RolloutParams q = p;
    // FIFO rings per persistent group when every group id indexes the allocation (the
    // next env of a group reuses its predecessor's L1/L2-warm ring lines; rings by env
    // id touch cold lines at every env start and leave dead dirty lines to be evicted)
    q.ring_per_group = BE_RING_PER_GROUP && blocks * groups_per_block <= (long long)p.E;
    kern<<<(unsigned)blocks, threads, smem, st>>>(q);
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e, "rollout launch");
    const int32_t pl[8] = {M, LPE, p.cfg.estimator_true_rate ? 1 : 0,
                           (p.cfg.estimator_true_rate && many) ? 1 : 0, p.skip_smem, p.screen, per_sm,
                           (int32_t)blocks};
    for (int k = 0; k < 8; ++k) plan[k] = pl[k];
    return BE_OK;
}

template <int M>
static int launch_rollout_lpe(const RolloutParams& p, size_t smem, cudaStream_t st, int sms, int32_t* plan) {
    if (p.screen) {
        stage_qpack_kernel<M><<<QPACK_CTAS, 256, 0, st>>>(p.w1, p.b1, p.w2, p.b2, p.cfg.n_tasks, p.H,
                                                 const_cast<double*>(p.qpack));
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return set_cuda_error(e, "stage_qpack launch");
    }
    if (p.R <= 16 && (p.H == 0 || p.H % 32 == 0)) return launch_rollout_m<M, 16>(p, smem, st, sms, plan);
    return launch_rollout_m<M, 32>(p, smem, st, sms, plan);
}

int launch_rollout(be_env* env, const be_trace_soa* tr, const be_qweights* W, int static_tier,
                   const uint8_t* forced, const be_records* rec, cudaStream_t st) {
    RolloutParams p{};
    p.cfg = env->cfg;
    make_score_aux(env->cfg, &p.aux);
    p.E = tr->n_envs;
    p.ld = tr->ld;
    p.arrival = tr->arrival_ms;
    p.task = tr->task;
    p.n_events = tr->n_events;
    p.seg_off = tr->seg_offsets;
    p.seg_start = tr->seg_start;
    p.seg_rate = tr->seg_rate;
    p.forced = forced;
    p.env_ready = tr->env_ready;
    p.envs_per_ready = tr->envs_per_ready > 0 ? tr->envs_per_ready : 1;
    p.ready_value = tr->ready_value;
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
    // the screen needs H % (2 LPE) == 0 (LPE = 16 for <= 16 replicas, else 32); runs that
    // record Q values use the fp64 path throughout
    const int lpe = (env->R <= 16 && (!policy || p.H % 32 == 0)) ? 16 : 32;
    p.screen = policy && env->cfg.q_screen && !rec->q && p.H % (2 * lpe) == 0 &&
               rollout_smem_bytes(T, M, p.H, true, 0, true) <= 200 * 1024;
    p.screen_stats = p.screen ? env->d_screen : nullptr;
    p.qpack = env->d_qpack;
    p.exact_mul = env->exact_mul;
    for (int m = 0; m < M; ++m) p.inv_scale[m] = 1.0 / env->cfg.batch_scales[m];
    p.inv_rate_scale = 1.0 / env->cfg.rate_scale;
    {
        int ok_pack = M <= 3;
        for (int m = 0; m < M; ++m)
            if ((long long)env->cfg.tiers[m].replicas << env->cap_log2 >= 1024) ok_pack = 0;
        p.pack_obs = ok_pack;
    }
    p.skip = env->d_skip;
    p.skip_rows = env->skip_rows;
    // True rate: the variant with the shortest expected makespan.  One wave of the
    // latency variant (2 CTAs/SM, 128 registers, the skip table staged in shared memory)
    // beats everything; then one wave of the throughput variant (3 CTAs/SM, 80 registers,
    // the skip table through L1); up to two waves of the latency variant still beat a
    // throughput wave plus a partial second one (measured, tools/probe_occ.py: 8,192 envs
    // — config 4's shard on 8 GPUs — 57.6 vs 67.2 ms); beyond, the throughput variant.
    const long long gpb = BE_ROLLOUT_THREADS / (env->R <= 16 ? 16 : 32);
    const long long g_lat = (long long)env->sms * BE_ROLLOUT_MINB_EST * gpb;
    const long long g_many = (long long)env->sms * BE_ROLLOUT_MINB * gpb;
    const long long E64 = p.E;
    bool many = env->cfg.estimator_true_rate && env->exact_mul && !(E64 <= g_lat || (E64 > g_many && E64 <= 2 * g_lat));
    if (const char* f = getenv("BE_ROLLOUT_FORCE_OCC"))  // probes (tools/probe_occ.py)
        many = env->cfg.estimator_true_rate && env->exact_mul && atoi(f) != 0;
    p.throughput = many ? 1 : 0;
    p.skip_smem = p.skip && rollout_smem_bytes(T, M, policy ? p.H : 0, policy, p.skip_rows, p.screen) <=
                              (size_t)(env->cfg.estimator_true_rate && many ? BE_SKIP_SMEM_MAX : BE_SKIP_SMEM_MAX_EST);
    size_t smem = rollout_smem_bytes(T, M, policy ? p.H : 0, policy, p.skip_smem ? p.skip_rows : 0, p.screen);
    cudaError_t e = cudaMemsetAsync(env->d_counter, 0, sizeof(int32_t), st);
    if (e != cudaSuccess) return set_cuda_error(e, "memset counter");
    switch (M) {
        case 1: return launch_rollout_lpe<1>(p, smem, st, env->sms, env->last_plan);
        case 2: return launch_rollout_lpe<2>(p, smem, st, env->sms, env->last_plan);
        case 3: return launch_rollout_lpe<3>(p, smem, st, env->sms, env->last_plan);
        case 4: return launch_rollout_lpe<4>(p, smem, st, env->sms, env->last_plan);
        case 5: return launch_rollout_lpe<5>(p, smem, st, env->sms, env->last_plan);
        case 6: return launch_rollout_lpe<6>(p, smem, st, env->sms, env->last_plan);
        case 7: return launch_rollout_lpe<7>(p, smem, st, env->sms, env->last_plan);
        case 8: return launch_rollout_lpe<8>(p, smem, st, env->sms, env->last_plan);
        default: return set_error(BE_EINVAL, "n_tiers out of range");
    }
}

}  // namespace be
