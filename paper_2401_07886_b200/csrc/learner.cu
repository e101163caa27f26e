// learner.cu — DQN training on the device (K3 replay + K4 learner).
//
//   TrainingWorkload.next_arrival    trainer.py:293-316   -> train_workload_kernel
//   ReplayBuffer pending store       trainer.py:93-156    -> pending ring [P][E] + commit kernels
//   ReplayBuffer ring / sample       trainer.py:101-163   -> ring [C] + Philox sampling
//   _StepKernel.compute              trainer.py:211-267   -> learner_partial_kernel (+ reduce)
//   td_targets_double_q              trainer.py:166-174
//   Adam / SGD, target sync          trainer.py:177-208, :276-290 -> learner_apply_kernel
//
// All learner arithmetic is fp64 (an fp32 learner misses 1e-5 on
// gradients by cancellation over the batch).  Gradients are reduced over row
// tiles in a fixed order, so an update is deterministic for a given batch.
// Transitions commit once their reward (request completion) and next state
// (the env's next decision) are both known (trainer.py:143-156); the ring slot
// of every commit comes from an exclusive scan over per-env commit counts in
// env-id order, never from an atomic cursor, so training
// is reproducible for a fixed seed.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "be200.h"
#include "be_internal.h"
#include "be_philox.cuh"

namespace be {

constexpr int LROWS = 32;      // rows per learner CTA
constexpr int LTHREADS = 256;  // one thread per hidden unit (looping for H > 256)

// --------------------------------------------------------------- workload
// TrainingWorkload.next_arrival (trainer.py:304-316) per env; state [E][3] =
// (time_ms, rate, segment_left).  Philox counter (step, env), key seed.
__global__ void train_workload_kernel(int E, double* state, double log_lo, double log_hi,
                                      int equal_time, double mean_seconds, double mean_requests,
                                      int n_tasks, uint64_t seed, uint64_t step, double* arrival,
                                      uint8_t* task, double* rate_out, const int64_t* step_dev) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    if (step_dev) step = (uint64_t)*step_dev;  // be_train_iteration: iteration index on device
    double t = state[3 * e], rate = state[3 * e + 1], left = state[3 * e + 2];
    P4 a = philox4x32_10(step * 2, (uint64_t)e, seed);
    if (left <= 0.0) {
        rate = exp(log_lo + (log_hi - log_lo) * u01(a.x[0], a.x[1]));
        double mean = equal_time ? fmax(1.0, mean_seconds * rate) : mean_requests;
        double p = 1.0 / mean;
        // numpy geometric(p): trials to the first success, >= 1 (inversion)
        double u = u01(a.x[2], a.x[3]);
        left = p >= 1.0 ? 1.0 : fmax(1.0, ceil(log1p(-u) / log1p(-p)));
    }
    left -= 1.0;
    P4 b = philox4x32_10(step * 2 + 1, (uint64_t)e, seed);
    const double gap = -log1p(-u01(b.x[0], b.x[1])) * (1000.0 / rate);
    t = t + gap;
    state[3 * e] = t;
    state[3 * e + 1] = rate;
    state[3 * e + 2] = left;
    arrival[e] = t;
    task[e] = (uint8_t)below(b.x[2], (uint32_t)n_tasks);
    rate_out[e] = rate;
}

// --------------------------------------------------------------- commits
struct CommitParams {
    int32_t E, D, P;
    int64_t step;            // id of the request just submitted in every env
    const double* px;        // pending states [P][E][D]
    const uint8_t* pa;       // pending actions [P][E]
    uint8_t* pflags;         // [E][P] completion flags (bit 6 = reward known)
    const double* preward;   // [E][P]
    int64_t* low;            // [E] oldest uncommitted request id
    int32_t* count;          // [E] commits this step
    const int64_t* offset;   // [E] exclusive scan of count (pass 2)
    int64_t* ring_state;     // [0] cursor, [1] size, [2] total commits
    int64_t capacity;
    double* rs;              // ring states [C][D]
    double* rs2;             // ring next states [C][D]
    uint8_t* ra;             // ring actions [C]
    double* rr;              // ring rewards [C]
    double* rc;              // ring continue flags [C]
    int32_t* status;
    const int64_t* step_dev;  // be_train_iteration: `step` read from device memory
};

// A transition j is ready when its reward is known and j <= step - 1 (its next
// state x_{j+1} exists).  Pass 1 counts per env, pass 2 writes in id order.
template <bool WRITE>
__global__ void commit_kernel(const CommitParams p) {
    const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (e >= p.E) return;
    int64_t lo = p.low[e];
    const int64_t step = p.step_dev ? *p.step_dev : p.step;
    const int64_t hi = step - 1;  // inclusive upper candidate
    int64_t base = WRITE ? p.offset[e] : 0;
    int total = 0;
    int64_t new_low = lo;
    bool blocked = false;  // first not-ready id seen: low cannot pass it
    for (int64_t j0 = lo; j0 <= hi; j0 += 32) {
        const int64_t j = j0 + lane;
        bool ready = false, pend = false;
        if (j <= hi) {
            // 0 = in flight (cleared at submit), 0x40|tier|miss = completed, 0x20 = committed
            const uint8_t f = p.pflags[(int64_t)e * p.P + (j % p.P)];
            ready = (f & 0x40) != 0;
            pend = (f & 0x60) == 0;
        }
        const unsigned rb = __ballot_sync(0xffffffffu, ready);
        const unsigned pb = __ballot_sync(0xffffffffu, pend);
        if (WRITE && ready) {
            const int rank = __popc(rb & ((1u << lane) - 1u));
            const int64_t slot = (p.ring_state[0] + base + total + rank) % p.capacity;
            const int64_t sj = (j % p.P), sj1 = ((j + 1) % p.P);
            for (int d = 0; d < p.D; ++d) {
                p.rs[slot * p.D + d] = p.px[(sj * p.E + e) * p.D + d];
                p.rs2[slot * p.D + d] = p.px[(sj1 * p.E + e) * p.D + d];
            }
            p.ra[slot] = p.pa[sj * p.E + e];
            p.rr[slot] = p.preward[(int64_t)e * p.P + sj];
            p.rc[slot] = 1.0;  // no episode boundaries in training
            p.pflags[(int64_t)e * p.P + sj] = 0x20;  // committed (cleared again at the next submit)
        }
        total += __popc(rb);
        if (!blocked) {
            if (pb) {
                new_low = j0 + __ffs(pb) - 1;
                blocked = true;
            } else {
                new_low = (j0 + 32 <= hi + 1) ? j0 + 32 : hi + 1;
            }
        }
    }
    if (lane == 0) {
        if (!WRITE) {
            p.count[e] = total;
        } else {
            p.low[e] = new_low;
            // the pending ring must hold every uncommitted request
            if (step + 1 - new_low >= p.P && atomicCAS(&p.status[0], 0, BE_ECAPACITY) == 0)
                p.status[1] = e;
        }
    }
}

// single-CTA exclusive scan of the per-env commit counts (env-id order)
__global__ void commit_scan_kernel(int E, const int32_t* count, int64_t* offset, int64_t* ring_state,
                                   int64_t capacity) {
    __shared__ int64_t part[1024];
    const int t = threadIdx.x;
    const int per = (E + blockDim.x - 1) / blockDim.x;
    int64_t s = 0;
    for (int k = 0; k < per; ++k) {
        const int e = t * per + k;
        if (e < E) s += count[e];
    }
    part[t] = s;
    __syncthreads();
    if (t == 0) {
        int64_t acc = 0;
        for (int k = 0; k < (int)blockDim.x; ++k) {
            const int64_t v = part[k];
            part[k] = acc;
            acc += v;
        }
        part[blockDim.x] = acc;  // blockDim <= 1023
    }
    __syncthreads();
    int64_t acc = part[t];
    for (int k = 0; k < per; ++k) {
        const int e = t * per + k;
        if (e < E) {
            offset[e] = acc;
            acc += count[e];
        }
    }
    __syncthreads();
    if (t == 0) ring_state[3] = part[blockDim.x];  // commits this step (applied after pass 2)
}

__global__ void commit_finish_kernel(int64_t* ring_state, int64_t capacity) {
    const int64_t n = ring_state[3];
    ring_state[0] = (ring_state[0] + n) % capacity;
    ring_state[1] = ring_state[1] + n < capacity ? ring_state[1] + n : capacity;
    ring_state[2] += n;
}

// --------------------------------------------------------------- learner
struct LearnParams {
    int32_t D, H, M, B;
    const double* w1;  // online [D][H]
    const double* b1;
    const double* w2;  // [H][M]
    const double* b2;
    const double* tw1;  // target
    const double* tb1;
    const double* tw2;
    const double* tb2;
    // batch source: explicit arrays, or the ring sampled with Philox
    const double* s;
    const uint8_t* a;
    const double* r;
    const double* s2;
    const double* c;
    const int64_t* ring_state;  // [1] = size (sampling mode)
    int32_t sampling;           // 1: indices drawn with Philox from [0, size)
    int64_t min_size;           // max(batch, warmup): skip the update below it
    uint64_t seed, counter;
    double discount;
    int32_t huber;
    double* partial;  // [nCTA][P + 1]: grads w1,b1,w2,b2 then loss
    int64_t* sample_idx;  // [B] (optional debug output)
    // be_train_iteration: Philox counter = (*iter_dev) * ups + uidx
    const int64_t* iter_dev;
    int32_t ups, uidx;
    const int64_t* gate;  // non-NULL: update iff *gate != 0 (DP learner, all-reduced readiness)
};

__device__ __forceinline__ double relu_d(double x) {
    const long long b = __double_as_longlong(x);
    return __longlong_as_double(b & ~(b >> 63));
}

// Forward of LROWS rows through (W1,b1,W2,b2) into h (smem [LROWS][H]) and q
// (smem [LROWS][M]); block-wide, fixed reduction order.
__device__ void forward_rows(const double* x, int D, int H, int M, const double* w1,
                             const double* b1, const double* w2, const double* b2, double* h,
                             double* q, double* red) {
    for (int j = threadIdx.x; j < H; j += blockDim.x) {
        const double bj = b1[j];
        double wcol[32];
        for (int d = 0; d < D; ++d) wcol[d] = w1[d * H + j];
        for (int row = 0; row < LROWS; ++row) {
            double acc = 0.0;
            for (int d = 0; d < D; ++d) acc = __fma_rn(x[row * D + d], wcol[d], acc);
            h[row * H + j] = relu_d(__dadd_rn(acc, bj));
        }
    }
    __syncthreads();
    // q[row][m] = sum_j h[row][j] w2[j][m]: warp w handles pairs w, w + 8, ...
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    for (int pair = warp; pair < LROWS * M; pair += nw) {
        const int row = pair / M, m = pair % M;
        double acc = 0.0;
        for (int j = lane; j < H; j += 32) acc = __fma_rn(h[row * H + j], w2[j * M + m], acc);
        for (int off = 16; off > 0; off >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
        if (lane == 0) q[pair] = __dadd_rn(acc, b2[m]);
    }
    __syncthreads();
    (void)red;
}

struct ApplyParams {
    int32_t nparam;
    double* params;   // online [nparam] (w1, b1, w2, b2 contiguous)
    double* target;   // [nparam]
    double* m;
    double* v;
    const double* grad;
    int64_t* counters;  // [0] adam t, [1] grad steps, [2] updates applied flag, [3] iteration
    double lr, beta1, beta2, eps;
    int32_t adam;
    int64_t sync_every;
    const int64_t* ring_state;
    int64_t min_size;
    int32_t sampling;
    double* loss;        // current loss
    double* last_loss;   // persisted "last_loss" for logs
    int32_t advance;     // 1: counters[3] += 1 afterwards (last update of a be_train_iteration)
    const int64_t* gate; // non-NULL: apply iff *gate != 0
};

// Adam (trainer.py:190-199) or SGD (:202-208), then the target sync
// (trainer.py:288-289) — all parameters, by one CTA.
__device__ void apply_update(const ApplyParams& p) {
    __shared__ double bc[2];
    __shared__ int do_sync;
    if (threadIdx.x == 0) {
        const int64_t t = p.counters[0] + 1;
        bc[0] = 1.0 - pow(p.beta1, (double)t);
        bc[1] = 1.0 - pow(p.beta2, (double)t);
        const int64_t gs = p.counters[1] + 1;  // step_index = grad_steps + 1
        do_sync = (gs % p.sync_every) == 0;
    }
    __syncthreads();
    for (int k = threadIdx.x; k < p.nparam; k += blockDim.x) {
        const double gk = p.grad[k];
        double w = p.params[k];
        if (p.adam) {
            double mk = __dadd_rn(__dmul_rn(p.m[k], p.beta1), __dmul_rn(1.0 - p.beta1, gk));
            double vk = __dadd_rn(__dmul_rn(p.v[k], p.beta2), __dmul_rn(__dmul_rn(1.0 - p.beta2, gk), gk));
            p.m[k] = mk;
            p.v[k] = vk;
            const double num = __dmul_rn(p.lr, __ddiv_rn(mk, bc[0]));
            const double den = __dadd_rn(__dsqrt_rn(__ddiv_rn(vk, bc[1])), p.eps);
            w = __dsub_rn(w, __ddiv_rn(num, den));
        } else {
            w = __dsub_rn(w, __dmul_rn(p.lr, gk));
        }
        p.params[k] = w;
        if (do_sync) p.target[k] = w;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        p.counters[0] += 1;
        p.counters[1] += 1;
        p.counters[2] = 1;
        *p.last_loss = *p.loss;
    }
}

__global__ void learner_apply_kernel(const ApplyParams p) {
    if (!(p.gate ? *p.gate == 0 : (p.sampling && p.ring_state[1] < p.min_size))) apply_update(p);
    if (p.advance && threadIdx.x == 0) p.counters[3] += 1;
}

// Fused update (be_train_iteration, single GPU): the CTA that finishes its
// row tile last sums every tile's partials in tile order (the same fixed order
// as learner_reduce_kernel) and applies the optimizer step — one launch per
// update: Double-Q targets, Huber backward, reduction, Adam, target sync.
struct FuseParams {
    int32_t fused;
    unsigned* done;  // arrival counter of the CTAs (reset by the last one)
    double* grad;
    double* loss;
    ApplyParams ap;
};

__global__ void __launch_bounds__(LTHREADS) learner_partial_kernel(const LearnParams p, const FuseParams f) {
    extern __shared__ __align__(16) double lsm[];
    const int D = p.D, H = p.H, M = p.M;
    double* xs = lsm;                    // [LROWS][D]
    double* xs2 = xs + LROWS * D;        // [LROWS][D]
    double* hh = xs2 + LROWS * D;        // [LROWS][H]  online h(s)
    double* ht = hh + LROWS * H;         // [LROWS][H]  scratch h(s')
    double* q = ht + LROWS * H;          // [LROWS][M]
    double* q2 = q + LROWS * M;          // [LROWS][M]
    double* q2t = q2 + LROWS * M;        // [LROWS][M]
    double* g = q2t + LROWS * M;         // [LROWS][M]  dL/dq
    double* rw = g + LROWS * M;          // [LROWS]
    double* cc = rw + LROWS;             // [LROWS]
    double* lrow = cc + LROWS;           // [LROWS] per-row loss
    int* act = reinterpret_cast<int*>(lrow + LROWS);  // [LROWS]
    const int row0 = blockIdx.x * LROWS;
    const int nparam = D * H + H + H * M + M;
    double* out = p.partial + (size_t)blockIdx.x * (nparam + 1);
    if (p.gate ? *p.gate == 0 : (p.sampling && p.ring_state[1] < p.min_size)) {  // warm-up: no update
        if (f.fused && f.ap.advance && blockIdx.x == 0 && threadIdx.x == 0) f.ap.counters[3] += 1;
        return;
    }
    const uint64_t counter = p.iter_dev ? (uint64_t)(*p.iter_dev) * (uint64_t)p.ups + (uint64_t)p.uidx
                                        : p.counter;

    // ---- gather the batch rows (ReplayBuffer.sample: rng.integers(0, size, B))
    for (int k = threadIdx.x; k < LROWS; k += blockDim.x) {
        const int b = row0 + k;
        int64_t src = b < p.B ? b : 0;
        if (p.sampling) {
            const uint64_t size = (uint64_t)p.ring_state[1];
            P4 rn = philox4x32_10(counter, (uint64_t)b, p.seed);
            const uint64_t r64 = ((uint64_t)rn.x[0] << 32) | rn.x[1];
            src = (int64_t)(((unsigned __int128)r64 * size) >> 64);
            if (p.sample_idx) p.sample_idx[b] = src;
        }
        act[k] = b < p.B ? (int)p.a[src] : 0;
        rw[k] = b < p.B ? p.r[src] : 0.0;
        cc[k] = b < p.B ? p.c[src] : 0.0;
        for (int d = 0; d < D; ++d) {
            xs[k * D + d] = b < p.B ? p.s[src * D + d] : 0.0;
            xs2[k * D + d] = b < p.B ? p.s2[src * D + d] : 0.0;
        }
    }
    __syncthreads();
    // ---- Double-Q targets (trainer.py:240-243)
    forward_rows(xs2, D, H, M, p.w1, p.b1, p.w2, p.b2, ht, q2, nullptr);
    forward_rows(xs2, D, H, M, p.tw1, p.tb1, p.tw2, p.tb2, ht, q2t, nullptr);
    forward_rows(xs, D, H, M, p.w1, p.b1, p.w2, p.b2, hh, q, nullptr);
    for (int k = threadIdx.x; k < LROWS; k += blockDim.x) {
        const bool valid = row0 + k < p.B;
        int best = 0;
        double bv = q2[k * M];
        for (int m = 1; m < M; ++m)
            if (q2[k * M + m] > bv) {
                bv = q2[k * M + m];
                best = m;
            }
        // y = r + cont * discount * q2t[best]  (left to right, trainer.py:243)
        const double y = __dadd_rn(rw[k], __dmul_rn(__dmul_rn(cc[k], p.discount), q2t[k * M + best]));
        const double res = __dsub_rn(q[k * M + act[k]], y);
        double l, dq;
        if (p.huber) {
            const double a = fabs(res);
            l = a <= 1.0 ? __dmul_rn(0.5, __dmul_rn(res, res)) : __dsub_rn(a, 0.5);
            dq = __ddiv_rn(fmin(fmax(res, -1.0), 1.0), (double)p.B);
        } else {
            l = __dmul_rn(0.5, __dmul_rn(res, res));
            dq = __ddiv_rn(res, (double)p.B);
        }
        lrow[k] = valid ? l : 0.0;
        for (int m = 0; m < M; ++m) g[k * M + m] = (valid && m == act[k]) ? dq : 0.0;
    }
    __syncthreads();
    // ---- backward over this tile's rows (trainer.py:256-263)
    for (int j = threadIdx.x; j < H; j += blockDim.x) {
        double dw2[8], db1 = 0.0, dw1[32];
        for (int m = 0; m < M; ++m) dw2[m] = 0.0;
        for (int d = 0; d < D; ++d) dw1[d] = 0.0;
        double w2j[8];
        for (int m = 0; m < M; ++m) w2j[m] = p.w2[j * M + m];
        for (int row = 0; row < LROWS; ++row) {
            const double hv = hh[row * H + j];
            double dh = 0.0;
            for (int m = 0; m < M; ++m) {
                const double gm = g[row * M + m];
                dw2[m] = __fma_rn(hv, gm, dw2[m]);
                dh = __fma_rn(gm, w2j[m], dh);
            }
            if (!(hv > 0.0)) dh = 0.0;  // dh[h <= 0] = 0
            db1 = __dadd_rn(db1, dh);
            for (int d = 0; d < D; ++d) dw1[d] = __fma_rn(xs[row * D + d], dh, dw1[d]);
        }
        for (int d = 0; d < D; ++d) out[d * H + j] = dw1[d];
        out[D * H + j] = db1;
        for (int m = 0; m < M; ++m) out[D * H + H + j * M + m] = dw2[m];
    }
    if (threadIdx.x < M) {
        double s = 0.0;
        for (int row = 0; row < LROWS; ++row) s = __dadd_rn(s, g[row * M + threadIdx.x]);
        out[D * H + H + H * M + threadIdx.x] = s;
    }
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int row = 0; row < LROWS; ++row) s = __dadd_rn(s, lrow[row]);
        out[nparam] = s;
    }
    if (!f.fused) return;
    __threadfence();  // publish this tile's partials
    __syncthreads();
    __shared__ int last;
    if (threadIdx.x == 0) last = atomicAdd(f.done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int k = threadIdx.x; k <= nparam; k += blockDim.x) {
        double s = 0.0;
        for (int t = 0; t < (int)gridDim.x; ++t) s = __dadd_rn(s, __ldcg(p.partial + (size_t)t * (nparam + 1) + k));
        if (k < nparam) f.grad[k] = s;
        else *f.loss = __ddiv_rn(s, (double)p.B);
    }
    __syncthreads();
    apply_update(f.ap);
    if (threadIdx.x == 0) {
        *f.done = 0u;
        if (f.ap.advance) f.ap.counters[3] += 1;
    }
}

// Sum the per-tile partials in tile order -> grad[nparam], loss.
__global__ void learner_reduce_kernel(int n_tiles, int nparam, int B, const double* partial,
                                      double* grad, double* loss, const int64_t* ring_state,
                                      int64_t min_size, int sampling, const int64_t* gate) {
    if (gate ? *gate == 0 : (sampling && ring_state[1] < min_size)) {
        // no update this iteration: a zero gradient keeps a DP all-reduce well defined
        for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nparam; k += gridDim.x * blockDim.x)
            grad[k] = 0.0;
        return;
    }
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k <= nparam; k += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int t = 0; t < n_tiles; ++t) s = __dadd_rn(s, partial[(size_t)t * (nparam + 1) + k]);
        if (k < nparam) grad[k] = s;
        else *loss = __ddiv_rn(s, (double)B);
    }
}

}  // namespace be

using namespace be;

// ------------------------------------------------------------------ C ABI
struct be_learner {
    be_learner_cfg cfg;
    int32_t device, D, nparam, n_tiles;
    double* params;   // online: w1 | b1 | w2 | b2
    double* target;
    double* m;
    double* v;
    double* grad;
    double* partial;
    double* loss;     // [0] loss of the last computed update, [1] last applied
    int64_t* counters;
    // replay
    double *rs, *rs2, *rr, *rc;
    uint8_t* ra;
    int64_t* ring_state;  // cursor, size, total, pending count
    // pending (deferred rewards)
    double* px;      // [P][E][D]
    uint8_t* pa;     // [P][E]
    uint8_t* pflags; // [E][P]
    double* preward; // [E][P]
    int64_t* low;
    int32_t* count;
    int64_t* offset;
    int32_t* status;
    double* wl_state;  // [E][3]
    // be_train_iteration: per-env arrival / task / true rate of the current iteration
    double* it_arrival;
    uint8_t* it_task;
    double* it_rate;
    unsigned* done;    // fused-update CTA arrival counter
    int64_t* gate;     // DP update gate (be_train_iteration use_gate)
};

static void learner_free(be_learner* L) {
    void* ptrs[] = {L->params, L->target, L->m, L->v, L->grad, L->partial, L->loss, L->counters,
                    L->rs, L->rs2, L->rr, L->rc, L->ra, L->ring_state, L->px, L->pa, L->pflags,
                    L->preward, L->low, L->count, L->offset, L->status, L->wl_state,
                    L->it_arrival, L->it_task, L->it_rate, L->done, L->gate};
    for (void* p : ptrs) cudaFree(p);
    delete L;
}

extern "C" {

int32_t be_learner_create(const be_learner_cfg* c, int32_t device, be_learner** out) {
    if (!c || !out) return set_error(BE_EINVAL, "NULL argument");
    *out = nullptr;
    if (c->n_tasks < 1 || c->n_tiers < 1 || c->n_tiers > 8 || c->n_tasks + c->n_tiers + 1 > 32)
        return set_error(BE_EINVAL, "bad dimensions");
    if (c->hidden < 1 || c->hidden > 1024) return set_error(BE_EINVAL, "hidden out of range");
    if (c->batch < 1 || c->batch > c->replay_capacity)
        return set_error(BE_EINVAL, "batch_size must be >= 1 and <= buffer capacity");
    if (!(c->discount > 0 && c->discount < 1)) return set_error(BE_EINVAL, "discount must lie in (0, 1)");
    if (c->n_envs < 1 || c->pending_capacity < 2) return set_error(BE_EINVAL, "bad env / pending sizes");
    if (c->target_sync_every < 1) return set_error(BE_EINVAL, "target_sync_every must be >= 1");
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaSetDevice");
    be_learner* L = new be_learner();
    memset(L, 0, sizeof(*L));
    L->cfg = *c;
    L->device = device;
    const int D = c->n_tasks + c->n_tiers + 1, H = c->hidden, M = c->n_tiers;
    L->D = D;
    L->nparam = D * H + H + H * M + M;
    L->n_tiles = (c->batch + LROWS - 1) / LROWS;
    const size_t np = (size_t)L->nparam, C = (size_t)c->replay_capacity, E = (size_t)c->n_envs,
                 P = (size_t)c->pending_capacity;
    struct A { void** p; size_t n; } allocs[] = {
        {(void**)&L->params, np * 8}, {(void**)&L->target, np * 8}, {(void**)&L->m, np * 8},
        {(void**)&L->v, np * 8}, {(void**)&L->grad, np * 8},
        {(void**)&L->partial, (size_t)L->n_tiles * (np + 1) * 8}, {(void**)&L->loss, 16},
        {(void**)&L->counters, 64}, {(void**)&L->rs, C * D * 8}, {(void**)&L->rs2, C * D * 8},
        {(void**)&L->rr, C * 8}, {(void**)&L->rc, C * 8}, {(void**)&L->ra, C},
        {(void**)&L->ring_state, 64}, {(void**)&L->px, P * E * D * 8}, {(void**)&L->pa, P * E},
        {(void**)&L->pflags, E * P}, {(void**)&L->preward, E * P * 8}, {(void**)&L->low, E * 8},
        {(void**)&L->count, E * 4}, {(void**)&L->offset, E * 8}, {(void**)&L->status, 64},
        {(void**)&L->wl_state, E * 3 * 8}, {(void**)&L->it_arrival, E * 8},
        {(void**)&L->it_task, E}, {(void**)&L->it_rate, E * 8}, {(void**)&L->done, 64}, {(void**)&L->gate, 64}};
    for (auto& a : allocs) {
        e = cudaMalloc(a.p, a.n);
        if (e != cudaSuccess) {
            learner_free(L);
            return set_cuda_error(e, "be_learner_create: cudaMalloc");
        }
        cudaMemset(*a.p, 0, a.n);
    }
    // configured here, not at launch time: launches may be captured in a CUDA graph
    cudaFuncSetAttribute(learner_partial_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        learner_free(L);
        return set_cuda_error(e, "be_learner_create");
    }
    *out = L;
    return BE_OK;
}

int32_t be_learner_destroy(be_learner* L) {
    if (L) learner_free(L);
    return BE_OK;
}

int32_t be_learner_set_params(be_learner* L, const double* w1, const double* b1, const double* w2,
                              const double* b2, void* stream) {
    if (!L || !w1 || !b1 || !w2 || !b2) return set_error(BE_EINVAL, "NULL argument");
    const int D = L->D, H = L->cfg.hidden, M = L->cfg.n_tiers;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t s[4] = {(size_t)D * H, (size_t)H, (size_t)H * M, (size_t)M};
    const double* src[4] = {w1, b1, w2, b2};
    size_t off = 0;
    for (int k = 0; k < 4; ++k) {
        cudaMemcpyAsync(L->params + off, src[k], s[k] * 8, cudaMemcpyDefault, st);
        cudaMemcpyAsync(L->target + off, src[k], s[k] * 8, cudaMemcpyDefault, st);
        off += s[k];
    }
    cudaMemsetAsync(L->m, 0, (size_t)L->nparam * 8, st);
    cudaMemsetAsync(L->v, 0, (size_t)L->nparam * 8, st);
    cudaMemsetAsync(L->counters, 0, 64, st);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "set_params");
}

int32_t be_learner_views(be_learner* L, be_learner_views_t* v) {
    if (!L || !v) return set_error(BE_EINVAL, "NULL argument");
    const int D = L->D, H = L->cfg.hidden, M = L->cfg.n_tiers;
    v->online.hidden = H;
    v->online.w1 = L->params;
    v->online.b1 = L->params + D * H;
    v->online.w2 = L->params + D * H + H;
    v->online.b2 = L->params + D * H + H + H * M;
    v->target.hidden = H;
    v->target.w1 = L->target;
    v->target.b1 = L->target + D * H;
    v->target.w2 = L->target + D * H + H;
    v->target.b2 = L->target + D * H + H + H * M;
    v->params = L->params;
    v->grad = L->grad;
    v->nparam = L->nparam;
    v->loss = L->loss;
    v->counters = L->counters;
    v->ring_states = L->rs;
    v->ring_next_states = L->rs2;
    v->ring_actions = L->ra;
    v->ring_rewards = L->rr;
    v->ring_cont = L->rc;
    v->ring_state = L->ring_state;
    v->pending_x = L->px;
    v->pending_action = L->pa;
    v->pending_flags = L->pflags;
    v->pending_reward = L->preward;
    v->workload_state = L->wl_state;
    v->gate = L->gate;
    return BE_OK;
}

int32_t be_learner_workload(be_learner* L, uint64_t seed, int64_t step, double* arrival_ms,
                            uint8_t* task, double* true_rate, void* stream) {
    if (!L || !arrival_ms || !task || !true_rate) return set_error(BE_EINVAL, "NULL argument");
    const be_learner_cfg& c = L->cfg;
    if (!(c.rate_low > 0) || c.rate_high < c.rate_low) return set_error(BE_EINVAL, "need 0 < rate_low <= rate_high");
    const int E = c.n_envs;
    train_workload_kernel<<<(E + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
        E, L->wl_state, log(c.rate_low), log(c.rate_high), c.regime_equal_time, c.regime_mean_seconds,
        c.regime_mean_requests, c.n_tasks, seed, (uint64_t)step, arrival_ms, task, true_rate, nullptr);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "workload launch");
}

static int commit_impl(be_learner* L, int64_t step, const int64_t* step_dev, cudaStream_t st) {
    CommitParams p{};
    p.step_dev = step_dev;
    p.E = L->cfg.n_envs;
    p.D = L->D;
    p.P = L->cfg.pending_capacity;
    p.step = step;
    p.px = L->px;
    p.pa = L->pa;
    p.pflags = L->pflags;
    p.preward = L->preward;
    p.low = L->low;
    p.count = L->count;
    p.offset = L->offset;
    p.ring_state = L->ring_state;
    p.capacity = L->cfg.replay_capacity;
    p.rs = L->rs;
    p.rs2 = L->rs2;
    p.ra = L->ra;
    p.rr = L->rr;
    p.rc = L->rc;
    p.status = L->status;
    const int blocks = (int)(((int64_t)p.E * 32 + 255) / 256);
    commit_kernel<false><<<blocks, 256, 0, st>>>(p);
    commit_scan_kernel<<<1, 1023, 0, st>>>(p.E, L->count, L->offset, L->ring_state, p.capacity);
    commit_kernel<true><<<blocks, 256, 0, st>>>(p);
    commit_finish_kernel<<<1, 1, 0, st>>>(L->ring_state, p.capacity);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "commit launch");
}

int32_t be_learner_commit(be_learner* L, int64_t step, void* stream) {
    if (!L || step < 0) return set_error(BE_EINVAL, "bad argument");
    return commit_impl(L, step, nullptr, (cudaStream_t)stream);
}

static ApplyParams apply_params(be_learner* L, int32_t explicit_batch, int32_t advance);

static int learner_backward_impl(be_learner* L, const double* s, const uint8_t* a, const double* r,
                                 const double* s2, const double* c, int32_t B, uint64_t seed,
                                 uint64_t counter, int64_t* sample_idx, cudaStream_t st,
                                 const int64_t* iter_dev = nullptr, int32_t ups = 1, int32_t uidx = 0,
                                 int32_t fused = 0, int32_t advance = 0,
                                 const int64_t* gate = nullptr) {
    const be_learner_cfg& cf = L->cfg;
    if (B != cf.batch) return set_error(BE_EINVAL, "batch size differs from the learner config");
    LearnParams p{};
    const int D = L->D, H = cf.hidden, M = cf.n_tiers;
    p.D = D;
    p.H = H;
    p.M = M;
    p.B = B;
    p.w1 = L->params;
    p.b1 = L->params + D * H;
    p.w2 = L->params + D * H + H;
    p.b2 = L->params + D * H + H + H * M;
    p.tw1 = L->target;
    p.tb1 = L->target + D * H;
    p.tw2 = L->target + D * H + H;
    p.tb2 = L->target + D * H + H + H * M;
    const bool sampling = s == nullptr;
    p.s = sampling ? L->rs : s;
    p.a = sampling ? L->ra : a;
    p.r = sampling ? L->rr : r;
    p.s2 = sampling ? L->rs2 : s2;
    p.c = sampling ? L->rc : c;
    p.sampling = sampling ? 1 : 0;
    p.ring_state = L->ring_state;
    p.min_size = cf.batch > cf.warmup ? cf.batch : cf.warmup;
    p.seed = seed;
    p.counter = counter;
    p.discount = cf.discount;
    p.huber = cf.huber;
    p.partial = L->partial;
    p.sample_idx = sample_idx;
    p.iter_dev = iter_dev;
    p.ups = ups;
    p.uidx = uidx;
    p.gate = gate;
    FuseParams f{};
    f.fused = fused;
    if (fused) {
        f.done = L->done;
        f.grad = L->grad;
        f.loss = L->loss;
        f.ap = apply_params(L, sampling ? 0 : 1, advance);
    }
    const size_t smem = sizeof(double) * (2 * LROWS * D + 2 * LROWS * H + 4 * LROWS * M + 3 * LROWS) +
                        sizeof(int) * LROWS;
    if (smem > 200 * 1024) return set_error(BE_EINVAL, "hidden too large for the learner tile");
    learner_partial_kernel<<<L->n_tiles, LTHREADS, smem, st>>>(p, f);
    if (!fused)
        learner_reduce_kernel<<<(L->nparam + 256) / 256, 256, 0, st>>>(
            L->n_tiles, L->nparam, B, L->partial, L->grad, L->loss, L->ring_state, p.min_size,
            sampling ? 1 : 0, p.gate);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "learner launch");
}

int32_t be_learner_backward(be_learner* L, uint64_t seed, uint64_t counter, int64_t* sample_idx,
                            void* stream) {
    if (!L) return set_error(BE_EINVAL, "NULL learner");
    return learner_backward_impl(L, nullptr, nullptr, nullptr, nullptr, nullptr, L->cfg.batch, seed,
                                 counter, sample_idx, (cudaStream_t)stream);
}

int32_t be_learner_backward_batch(be_learner* L, const double* states, const uint8_t* actions,
                                  const double* rewards, const double* next_states,
                                  const double* cont, int32_t batch, void* stream) {
    if (!L || !states || !actions || !rewards || !next_states || !cont)
        return set_error(BE_EINVAL, "NULL argument");
    return learner_backward_impl(L, states, actions, rewards, next_states, cont, batch, 0, 0, nullptr,
                                 (cudaStream_t)stream);
}

static ApplyParams apply_params(be_learner* L, int32_t explicit_batch, int32_t advance) {
    const be_learner_cfg& cf = L->cfg;
    ApplyParams p{};
    p.nparam = L->nparam;
    p.params = L->params;
    p.target = L->target;
    p.m = L->m;
    p.v = L->v;
    p.grad = L->grad;
    p.counters = L->counters;
    p.lr = cf.learning_rate;
    p.beta1 = 0.9;
    p.beta2 = 0.999;
    p.eps = 1e-8;
    p.adam = cf.adam;
    p.sync_every = cf.target_sync_every;
    p.ring_state = L->ring_state;
    p.min_size = cf.batch > cf.warmup ? cf.batch : cf.warmup;
    p.sampling = explicit_batch ? 0 : 1;
    p.loss = L->loss;
    p.last_loss = L->loss + 1;
    p.advance = advance;
    return p;
}

int32_t be_learner_apply(be_learner* L, int32_t explicit_batch, void* stream) {
    if (!L) return set_error(BE_EINVAL, "NULL learner");
    learner_apply_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(apply_params(L, explicit_batch, 0));
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "apply launch");
}

int32_t be_train_iteration(be_learner* L, be_env* env, const be_train_iter_cfg* c, void* stream) {
    if (!L || !env || !c) return set_error(BE_EINVAL, "NULL argument");
    const be_learner_cfg& cf = L->cfg;
    cudaStream_t st = (cudaStream_t)stream;
    if (env->E != cf.n_envs || env->cfg.n_tiers != cf.n_tiers || env->cfg.n_tasks != cf.n_tasks)
        return set_error(BE_EINVAL, "env and learner shapes differ");
    if (c->updates_per_step < 0 || c->phase < 0 || c->phase > 3 || c->update_index < 0 ||
        ((c->phase == 1 || c->phase == 2) && c->update_index >= c->updates_per_step))
        return set_error(BE_EINVAL, "bad phase / update index");
    if (!(cf.rate_low > 0) || cf.rate_high < cf.rate_low)
        return set_error(BE_EINVAL, "need 0 < rate_low <= rate_high");
    const int64_t* it = L->counters + 3;
    const int E = cf.n_envs, D = L->D, H = cf.hidden, M = cf.n_tiers;
    int rc;
    const int64_t* gate = c->use_gate ? L->gate : nullptr;
    if (c->phase == 0 || c->phase == 3) {
        // workload (trainer.py:375) -> env step (:376-395) -> commits (:143-156)
        train_workload_kernel<<<(E + 255) / 256, 256, 0, st>>>(
            E, L->wl_state, log(cf.rate_low), log(cf.rate_high), cf.regime_equal_time,
            cf.regime_mean_seconds, cf.regime_mean_requests, cf.n_tasks, c->workload_seed, 0,
            L->it_arrival, L->it_task, L->it_rate, it);
        be_qweights W;
        W.hidden = H;
        W.w1 = L->params;
        W.b1 = L->params + D * H;
        W.w2 = L->params + D * H + H;
        W.b2 = L->params + D * H + H + H * M;
        be_records rec{};
        rec.flags = L->pflags;
        rec.reward = L->preward;
        rc = launch_env_step_dev(env, L->it_arrival, L->it_task, L->it_rate, &W, c->policy_seed, it,
                                 c->epsilon_start, c->epsilon_end, c->epsilon_decay_steps,
                                 cf.pending_capacity, cf.pending_capacity, &rec, L->pa, L->px, st);
        if (rc) return rc;
        rc = commit_impl(L, 0, it, st);
        if (rc) return rc;
    }
    const int ups = c->updates_per_step;
    if (c->phase == 0) {
        for (int u = 0; u < ups; ++u) {
            rc = learner_backward_impl(L, nullptr, nullptr, nullptr, nullptr, nullptr, cf.batch,
                                       c->sample_seed, 0, nullptr, st, it, ups, u, 1, u == ups - 1);
            if (rc) return rc;
        }
        if (ups == 0) {  // no learner: still advance the iteration
            learner_apply_kernel<<<1, 32, 0, st>>>(apply_params(L, 2, 1));
        }
    } else if (c->phase == 1) {
        rc = learner_backward_impl(L, nullptr, nullptr, nullptr, nullptr, nullptr, cf.batch,
                                   c->sample_seed, 0, nullptr, st, it, ups, c->update_index, 0, 0,
                                   gate);
        if (rc) return rc;
    } else if (c->phase == 2) {
        ApplyParams ap = apply_params(L, 0, c->update_index == ups - 1);
        ap.gate = gate;
        learner_apply_kernel<<<1, 1024, 0, st>>>(ap);
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "train iteration launch");
}

int32_t be_learner_check(be_learner* L, void* stream) {
    if (!L) return set_error(BE_EINVAL, "NULL learner");
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e != cudaSuccess) return set_cuda_error(e, "be_learner_check: sync");
    int32_t st[2];
    cudaMemcpy(st, L->status, sizeof(st), cudaMemcpyDeviceToHost);
    if (st[0] == 0) return BE_OK;
    cudaMemset(L->status, 0, 64);
    return set_error(st[0], "pending-transition ring overflow: a request stayed in flight longer "
                            "than pending_capacity decisions; raise pending_capacity");
}

}  // extern "C"
