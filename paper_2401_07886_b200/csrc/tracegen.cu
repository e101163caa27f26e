// tracegen.cu — on-device synthetic workload.
//
// gen_stable (workload.py:120-141) for one segment per env: Poisson arrivals
// at rate[e] req/s starting at 0 ms — exponential gaps of mean 1000/rate
// (workload.py:94-111) accumulated sequentially in fp64 exactly like
// `t0 + np.cumsum(gaps)` with t0 = 0 — and task ids uniform over [0, T)
// (workload.py:136).  numpy's PCG64 + ziggurat cannot be reproduced, so the
// draws come from Philox4x32-10 keyed by the seed with counter (request, env):
// the trace of env e is the same for any GPU count.  Parity is statistical
// (mean gap, KS, task frequencies — tests/test_tracegen_gpu.py), and traces
// can be exported to the reference CSV format to replay on the CPU.
#include <cuda_runtime.h>
#include <stdint.h>

#include "be_internal.h"
#include "be_philox.cuh"

constexpr unsigned FULL = 0xffffffffu;

namespace be {

__global__ void tracegen_stable_kernel(int E, int64_t env_offset, int64_t n, int64_t ld,
                                       const double* rate, int T,
                                       uint64_t seed, double* arrival, uint8_t* task) {
    // one warp per env: lanes draw 32 gaps in parallel, the prefix sum is
    // done sequentially (lane order) so times equal the left-to-right cumsum
    const int env = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (env >= E) return;
    const double mean_gap = __ddiv_rn(1000.0, rate[env]);
    double t = 0.0;
    for (int64_t i0 = 0; i0 < n; i0 += 32) {
        const int64_t i = i0 + lane;
        P4 r = philox4x32_10((uint64_t)i, (uint64_t)(env_offset + env), seed);
        // Exp(mean) by inversion: -log(1 - u) * mean, u in [0, 1)
        const double u = u01(r.x[0], r.x[1]);
        const double gap = __dmul_rn(-log1p(-u), mean_gap);
        const uint8_t tk = (uint8_t)below(r.x[2], (uint32_t)T);
        // sequential fp64 accumulation in request order (cumsum semantics)
        double ti = 0.0;
        for (int k = 0; k < 32; ++k) {
            const double g = __shfl_sync(0xffffffffu, gap, k);
            t = __dadd_rn(t, g);
            if (k == lane) ti = t;
        }
        if (i < n) {
            arrival[(int64_t)env * ld + i] = ti;
            task[(int64_t)env * ld + i] = tk;
        }
    }
}

int launch_tracegen(int E, int64_t env_offset, int64_t n, int64_t ld, const double* rate, int n_tasks, uint64_t seed,
                    double* arrival, uint8_t* task, cudaStream_t st) {
    const int threads = 256;
    const int blocks = (int)(((int64_t)E * 32 + threads - 1) / threads);
    tracegen_stable_kernel<<<blocks, threads, 0, st>>>(E, env_offset, n, ld, rate, n_tasks, seed, arrival, task);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "tracegen launch");
}


// ---------------------------------------------------------------------------
// General generator (be_trace_gen): gen_stable with several timed segments and
// the two unpredictable workloads.  One warp per env walks its segments in
// order; per segment the warp draws 32 exponential gaps at a time (counter =
// gap index, key = seed, counter_hi = global env id), adds them to the
// segment's running sum sequentially in lane order (`t0 + np.cumsum(gaps)`,
// workload.py:105-106, :114-117) and keeps the events inside the segment
// (time < end for gen_stable, count for the unpredictable kinds).  Segment
// draws (band, rate, geometric count) use the substream counter_hi | 2^48.
namespace {

constexpr uint64_t SUB_SEGMENT = 1ull << 48;

// numpy Generator.geometric(p) = number of Bernoulli(p) trials up to the first
// success (>= 1); inversion k = ceil(log(1 - u) / log(1 - p)).
__device__ __forceinline__ int64_t geometric_draw(double u, double p) {
    if (p >= 1.0) return 1;
    double k = ceil(__ddiv_rn(log1p(-u), log1p(-p)));
    if (!(k >= 1.0)) return 1;
    if (k > 4.0e15) k = 4.0e15;
    return (int64_t)k;
}

__device__ __forceinline__ void latch(int32_t* status, int code, int env) {
    if (atomicCAS(&status[0], 0, code) == 0) status[1] = env;
}

}  // namespace

__global__ void tracegen_kernel(const be_gen_cfg cfg, int E, int64_t env_offset, int64_t ld,
                                uint64_t seed, double* arrival, uint8_t* task, int64_t* n_events,
                                int64_t* seg_count, int64_t* seg_start, double* seg_rate,
                                int32_t* status) {
    const int env = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (env >= E) return;
    const uint64_t gid = (uint64_t)(env_offset + env);
    const int n_choices = cfg.n_task_ids > 0 ? cfg.n_task_ids : cfg.n_tasks;
    double* arr = arrival + (int64_t)env * ld;
    uint8_t* tsk = task + (int64_t)env * ld;
    int64_t* sst = seg_start + (int64_t)env * cfg.seg_capacity;
    double* srt = seg_rate + (int64_t)env * cfg.seg_capacity;
    const bool stable = cfg.kind == BE_GEN_STABLE;
    const double INF = __longlong_as_double(0x7ff0000000000000LL);
    // TIME_BASED_PROBS cumulated as np.cumsum does (workload.py:159)
    const double c0 = 0.90, c1 = __dadd_rn(c0, 0.08), c2 = __dadd_rn(c1, 0.02);
    int64_t i = 0, s = 0;
    uint64_t draw = 0;
    double t = 0.0;
    int fail = 0;
    for (;;) {
        double rate, t0, end = INF;
        int64_t count = INT64_MAX;
        if (stable) {
            if (s >= cfg.n_rates || (cfg.truncate && i >= ld)) break;
            rate = cfg.rates[(int64_t)env * cfg.rate_ld + s];
            t0 = __dmul_rn((double)s, cfg.hold_ms);  // k * hold_ms (workload.py:139)
            end = __dadd_rn(t0, cfg.hold_ms);        // t0 + duration (workload.py:100)
        } else {
            if (i >= cfg.n) break;
            const P4 r = philox4x32_10((uint64_t)s, gid | SUB_SEGMENT, seed);
            const double u0 = u01(r.x[0], r.x[1]);
            const double u1 = u01(r.x[2], r.x[3]);
            const P4 r2 = philox4x32_10((uint64_t)s, gid | (2 * SUB_SEGMENT), seed);
            const double u2 = u01(r2.x[0], r2.x[1]);
            double lo, hi, mean;
            if (cfg.kind == BE_GEN_UNPRED_TIME) {  // workload.py:160-163
                const int band = (u0 >= c0) + (u0 >= c1) + (u0 >= c2);
                lo = band == 0 ? 0.25 : (band == 1 ? 2.0 : 40.0);
                hi = band == 0 ? 2.0 : (band == 1 ? 40.0 : 48.0);
                rate = __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u1));
                mean = __dmul_rn(20.0, rate);
            } else {  // workload.py:189-191
                lo = 1.0;
                hi = 48.0;
                rate = __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u1));
                mean = 500.0;
            }
            count = geometric_draw(u2, __ddiv_rn(1.0, mean));
            if (count > cfg.n - i) count = cfg.n - i;  // workload.py:164
            t0 = t;                                    // t = times[-1] (workload.py:169)
        }
        if (!(rate > 0.0) || !isfinite(rate)) {
            fail = BE_EINVAL;
            break;
        }
        if (s >= cfg.seg_capacity) {
            fail = BE_ECAPACITY;
            break;
        }
        if (lane == 0) {
            sst[s] = i;
            srt[s] = rate;
        }
        ++s;
        const double mean_gap = __ddiv_rn(1000.0, rate);
        double run = 0.0;  // np.cumsum(gaps) of this segment so far
        int64_t k0 = 0;
        bool stop_all = false;
        for (;;) {
            const P4 r = philox4x32_10(draw + (uint64_t)lane, gid, seed);
            draw += 32;
            const double gap = __dmul_rn(-log1p(-u01(r.x[0], r.x[1])), mean_gap);
            const int tk = cfg.n_task_ids > 0 ? cfg.task_ids[below(r.x[2], (uint32_t)n_choices)]
                                              : (int)below(r.x[2], (uint32_t)n_choices);
            double mine = 0.0;
            for (int k = 0; k < 32; ++k) {
                run = __dadd_rn(run, __shfl_sync(FULL, gap, k));
                if (k == lane) mine = run;
            }
            const double a = __dadd_rn(t0, mine);
            const bool inside = stable ? (a < end) : (k0 + lane < count);
            const int nin = __popc(__ballot_sync(FULL, inside));  // a prefix: a is monotone
            int64_t room = ld - i;
            int keep = nin;
            if (nin > room) {
                if (stable && cfg.truncate) {
                    keep = (int)room;
                    stop_all = true;
                } else {
                    fail = BE_ECAPACITY;
                    break;
                }
            }
            if (lane < keep) {
                arr[i + lane] = a;
                tsk[i + lane] = (uint8_t)tk;
            }
            if (keep > 0) t = __shfl_sync(FULL, a, keep - 1);
            i += keep;
            k0 += keep;
            if (nin < 32 || stop_all) break;
        }
        if (fail || stop_all) break;
    }
    if (lane == 0) {
        n_events[env] = i;
        seg_count[env] = s;
        if (fail) latch(status, fail, env);
    }
}

int launch_tracegen_general(const be_gen_cfg* cfg, int E, int64_t env_offset, int64_t ld,
                            uint64_t seed, double* arrival, uint8_t* task, int64_t* n_events,
                            int64_t* seg_count, int64_t* seg_start, double* seg_rate,
                            int32_t* status, cudaStream_t st) {
    const int threads = 256;
    const int blocks = (int)(((int64_t)E * 32 + threads - 1) / threads);
    tracegen_kernel<<<blocks, threads, 0, st>>>(*cfg, E, env_offset, ld, seed, arrival, task,
                                                 n_events, seg_count, seg_start, seg_rate, status);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "tracegen launch");
}

}  // namespace be
