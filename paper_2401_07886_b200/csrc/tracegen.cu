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

}  // namespace be
