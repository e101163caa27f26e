// be_workload.cuh — TrainingWorkload.next_arrival (trainer.py:304-316) for one env,
// shared by train_workload_kernel (learner.cu) and the fused weight-packing +
// workload launch of be_train_iteration (step.cu).  State [E][3] = (time_ms,
// rate, requests left in the regime); Philox counter (step, env), key seed.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "be_philox.cuh"

namespace be {

struct WorkloadArgs {
    int E;
    double* state;
    double log_lo, log_hi;
    int equal_time;
    double mean_seconds, mean_requests;
    int n_tasks;
    uint64_t seed, step;
    double* arrival;
    uint8_t* task;
    double* rate_out;
    const int64_t* step_dev;  // be_train_iteration: iteration index on device (else `step`)
};

// Next arrival of env e: (arrival time, task, regime rate); `store` = write the state
// and the outputs (the fused training step computes it on every lane of the env's
// group and lets one lane store).
__device__ __forceinline__ void train_workload_next(const WorkloadArgs& w, int e, bool store, double& t_out,
                                                    int& task_out, double& rate_out) {
    const uint64_t step = w.step_dev ? (uint64_t)*w.step_dev : w.step;
    double t = w.state[3 * e], rate = w.state[3 * e + 1], left = w.state[3 * e + 2];
    P4 a = philox4x32_10(step * 2, (uint64_t)e, w.seed);
    if (left <= 0.0) {
        rate = exp(w.log_lo + (w.log_hi - w.log_lo) * u01(a.x[0], a.x[1]));
        double mean = w.equal_time ? fmax(1.0, w.mean_seconds * rate) : w.mean_requests;
        double p = 1.0 / mean;
        // numpy geometric(p): trials to the first success, >= 1 (inversion)
        double u = u01(a.x[2], a.x[3]);
        left = p >= 1.0 ? 1.0 : fmax(1.0, ceil(log1p(-u) / log1p(-p)));
    }
    left -= 1.0;
    P4 b = philox4x32_10(step * 2 + 1, (uint64_t)e, w.seed);
    const double gap = -log1p(-u01(b.x[0], b.x[1])) * (1000.0 / rate);
    t = t + gap;
    const int task = (int)below(b.x[2], (uint32_t)w.n_tasks);
    if (store) {
        w.state[3 * e] = t;
        w.state[3 * e + 1] = rate;
        w.state[3 * e + 2] = left;
        w.arrival[e] = t;
        w.task[e] = (uint8_t)task;
        w.rate_out[e] = rate;
    }
    t_out = t;
    task_out = task;
    rate_out = rate;
}

__device__ __forceinline__ void train_workload_env(const WorkloadArgs& w, int e) {
    double t, rate;
    int task;
    train_workload_next(w, e, true, t, task, rate);
}

}  // namespace be
