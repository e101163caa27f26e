// learner.cu — DQN training on the device (K3 replay + K4 learner).
//
//   TrainingWorkload.next_arrival    trainer.py:293-316   -> train_workload_kernel (host-driven),
//                                                             in the env step (be_train_iteration)
//   ReplayBuffer pending store       trainer.py:93-156    -> pending ring [P][E] + commit_fused_kernel
//                                                             (host-driven) / env_step_commit_kernel
//   ReplayBuffer ring / sample       trainer.py:101-163   -> ring [C] + Philox sampling
//   _StepKernel.compute              trainer.py:211-267   -> learner_partial_kernel
//   td_targets_double_q              trainer.py:166-174
//   Adam / SGD, target sync          trainer.py:177-208, :276-290 -> learner_tail (fused into
//                                                             learner_partial_kernel) / learner_update_kernel
//                                                             (reduce-only / apply-only: NCCL DP, host API)
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
#include <stdio.h>

#include "be200.h"
#include "be_internal.h"
#include "be_philox.cuh"
#include "be_workload.cuh"

namespace be {

constexpr int LROWS = 4;       // rows per learner CTA (B = 512 -> 128 CTAs: latency, not work, bounds an update)
constexpr int UTHREADS = 256;  // learner_update_kernel: 32 parameters x 8 tile slices per CTA
constexpr int LTHREADS = 256;  // one thread per hidden unit (looping for H > 256)

// --------------------------------------------------------------- workload
// TrainingWorkload.next_arrival per env: be_workload.cuh (shared with the fused
// weight-packing + workload launch of be_train_iteration, step.cu).
__global__ void train_workload_kernel(WorkloadArgs w) {
    pdl_trigger();  // the next kernel of the stream may be scheduled now
    pdl_wait();     // the previous one has completed and its writes are visible
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < w.E) train_workload_env(w, e);
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
    int64_t* ring_state;     // [0] cursor, [1] size, [2] total commits
    int64_t capacity;
    double* rs;              // ring states [C][D]
    double* rs2;             // ring next states [C][D]
    uint8_t* ra;             // ring actions [C]
    double* rr;              // ring rewards [C]
    double* rc;              // ring continue flags [C]
    int32_t* status;
    const int64_t* step_dev;  // be_train_iteration: `step` read from device memory
    // be_train_iteration: per env {lowest, highest id completed this step, oldest in flight}
    // from the env step — every completion of the step is committable now, and nothing
    // else is, so only that id range is scanned (nullable: scan from `low`)
    const int64_t* crange;
    // single-pass commit (commit_fused_kernel): decoupled look-back scan state
    unsigned long long* scan;  // [E / 8] (epoch << 40 | flag << 38 | value)
    unsigned* ticket;          // [0] virtual CTA ticket, [1] epoch (both advanced by the last CTA)
};

// A transition j is ready when its reward is known and j <= step - 1 (its next
// state x_{j+1} exists).
// The whole commit step in one launch (32 envs per CTA, one warp each): count the
// ready transitions, exclusive scan of the counts in env-id order across CTAs by
// decoupled look-back (virtual CTA ids from a ticket, so every predecessor has
// started; scan entries are tagged with a per-launch epoch instead of being
// cleared), write the transitions, and the last CTA advances the ring cursor.
// Slots follow env-id order, then request-id order within an env (never an atomic cursor).
constexpr int CENVS = 32;  // envs (warps) per commit CTA
constexpr unsigned FULL_MASK = 0xffffffffu;

__device__ __forceinline__ int commit_env(const CommitParams& p, int e, int lane, int64_t base, int64_t cursor,
                                          bool write, int64_t* window = nullptr) {
    const int64_t step = p.step_dev ? *p.step_dev : p.step;
    int64_t hi = step - 1;  // inclusive upper candidate
    int64_t lo = p.low[e];
    if (p.crange) {
        lo = p.crange[3 * (int64_t)e];
        const int64_t chi = p.crange[3 * (int64_t)e + 1];
        hi = chi < hi ? chi : hi;
    }
    int total = 0;
    int64_t new_low = lo;
    bool blocked = false;
    // pending slot of j0 (= j0 mod P) and ring slot of this env's first commit, kept
    // incrementally: no 64-bit division inside the loop
    int64_t r0 = lo <= hi ? lo % p.P : 0;
    const int64_t s0 = write ? (cursor + base) % p.capacity : 0;
    for (int64_t j0 = lo; j0 <= hi; j0 += 32) {
        const int64_t j = j0 + lane;
        int64_t sj = r0 + lane;
        while (sj >= p.P) sj -= p.P;
        bool ready = false, pend = false;
        if (j <= hi) {
            const uint8_t f = p.pflags[(int64_t)e * p.P + sj];
            ready = (f & 0x40) != 0;
            pend = (f & 0x60) == 0;
        }
        const unsigned rb = __ballot_sync(0xffffffffu, ready);
        const unsigned pb = __ballot_sync(0xffffffffu, pend);
        if (write && ready) {
            const int rank = __popc(rb & ((1u << lane) - 1u));
            int64_t slot = s0 + total + rank;
            while (slot >= p.capacity) slot -= p.capacity;
            const int64_t sj1 = sj + 1 == p.P ? 0 : sj + 1;
            for (int d = 0; d < p.D; ++d) {
                p.rs[slot * p.D + d] = p.px[(sj * p.E + e) * p.D + d];
                p.rs2[slot * p.D + d] = p.px[(sj1 * p.E + e) * p.D + d];
            }
            p.ra[slot] = p.pa[sj * p.E + e];
            p.rr[slot] = p.preward[(int64_t)e * p.P + sj];
            p.rc[slot] = 1.0;
            p.pflags[(int64_t)e * p.P + sj] = 0x20;
        }
        total += __popc(rb);
        r0 += 32;
        while (r0 >= p.P) r0 -= p.P;
        if (!blocked) {
            if (pb) {
                new_low = j0 + __ffs(pb) - 1;
                blocked = true;
            } else {
                new_low = (j0 + 32 <= hi + 1) ? j0 + 32 : hi + 1;
            }
        }
    }
    if (write && lane == 0) {
        if (p.crange) new_low = p.crange[3 * (int64_t)e + 2];  // the oldest request still in flight
        p.low[e] = new_low;
        if (step + 1 - new_low >= p.P && atomicCAS(&p.status[0], 0, BE_ECAPACITY) == 0) p.status[1] = e;
        if (window) *window = step + 1 - new_low;
    }
    return total;
}

__global__ void __launch_bounds__(CENVS * 32) commit_fused_kernel(const CommitParams p) {
    pdl_wait();     // the previous one has completed and its writes are visible
    __shared__ int vb_sh, cnt[CENVS];
    __shared__ long long wpre[CENVS];
    __shared__ long long excl_sh, cursor_sh;
    __shared__ unsigned epoch_sh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        // read the cursor and epoch before taking a ticket: the last CTA changes them
        cursor_sh = __ldcg(p.ring_state);
        epoch_sh = __ldcg(p.ticket + 1) & 0xffffffu;
        __threadfence();
        vb_sh = (int)atomicAdd(p.ticket, 1u);
    }
    __syncthreads();
    const int vb = vb_sh, nb = (p.E + CENVS - 1) / CENVS;
    const int e = vb * CENVS + warp;
    const unsigned long long ep = (unsigned long long)epoch_sh << 40;
    int c = 0;
    if (e < p.E) c = commit_env(p, e, lane, 0, 0, false);
    if (lane == 0) cnt[warp] = c;
    __syncthreads();
    if (warp == 0) {
        // exclusive prefix of the counts over this CTA's warps (inclusive scan - own)
        const long long own = lane < CENVS ? cnt[lane] : 0;
        long long inc = own;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const long long v = __shfl_up_sync(FULL_MASK, inc, off);
            if (lane >= off) inc += v;
        }
        if (lane < CENVS) wpre[lane] = inc - own;
        const long long agg = __shfl_sync(FULL_MASK, inc, 31);
        long long excl = 0;
        if (vb == 0) {
            if (lane == 0) atomicExch(&p.scan[0], ep | (2ull << 38) | (unsigned long long)agg);
        } else {
            if (lane == 0) atomicExch(&p.scan[vb], ep | (1ull << 38) | (unsigned long long)agg);
            // warp-wide look-back over windows of 32 predecessors (nearest first)
            for (int j = vb - 1;; j -= 32) {
                const int idx = j - lane;
                unsigned long long v = 2ull << 38;  // before the first CTA: prefix 0
                if (idx >= 0) {
                    do {
                        v = atomicAdd(&p.scan[idx], 0ull);
                    } while ((v >> 40) != (ep >> 40) || ((v >> 38) & 3ull) == 0);
                }
                const unsigned pb = __ballot_sync(FULL_MASK, ((v >> 38) & 3ull) == 2ull);
                const int stop = pb ? __ffs(pb) - 1 : 31;  // lanes 0..stop contribute
                long long val = lane <= stop ? (long long)(v & ((1ull << 38) - 1)) : 0;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) val += __shfl_xor_sync(FULL_MASK, val, off);
                excl += val;
                if (pb) break;
            }
            if (lane == 0) atomicExch(&p.scan[vb], ep | (2ull << 38) | (unsigned long long)(excl + agg));
        }
        if (lane == 0) {
            excl_sh = excl;
            if (vb == nb - 1) {  // commits this step: advance the ring
                const long long n = excl + agg;
                p.ring_state[3] = n;
                p.ring_state[0] = (cursor_sh + n) % p.capacity;
                p.ring_state[1] = p.ring_state[1] + n < p.capacity ? p.ring_state[1] + n : p.capacity;
                p.ring_state[2] += n;
                p.ticket[1] = p.ticket[1] + 1u;
                __threadfence();
                p.ticket[0] = 0u;
            }
        }
    }
    __shared__ unsigned long long wmax_sh;
    if (threadIdx.x == 0) wmax_sh = 0ull;
    __syncthreads();
    int64_t win = 0;
    if (e < p.E) commit_env(p, e, lane, excl_sh + wpre[warp], cursor_sh, true, &win);
    if (lane == 0 && e < p.E) atomicMax(&wmax_sh, (unsigned long long)win);
    __syncthreads();
    // high-water mark of in-flight decisions per env (ring_state[4]; diagnostics for
    // sizing pending_capacity)
    if (threadIdx.x == 0 && wmax_sh > (unsigned long long)__ldcg(p.ring_state + 4))
        atomicMax(reinterpret_cast<unsigned long long*>(p.ring_state + 4), wmax_sh);
    pdl_trigger();
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
    // fused update (learner_tail): the last TAIL_CTAS tiles to finish reduce the tile
    // partials of one hidden-unit slice each, apply the optimizer and repack the env
    // step's weights; no second launch
    int32_t tail;
    unsigned long long* tick;  // [0] tile arrivals, [1] slice completions (monotonic)
    double* qpack;             // the env step's packed weights (QLayout), or NULL
    int32_t T;                 // tasks (packing)
    int32_t stage_out;         // tile partials staged in shared memory, copied out coalesced
    int32_t tail_ns;           // tail CTAs: min(TAIL_CTAS, tiles, resident CTAs - 1) (waiting is safe)
};

__device__ __forceinline__ double relu_d(double x) {
    const long long b = __double_as_longlong(x);
    return __longlong_as_double(b & ~(b >> 63));
}

// The learner's three forwards in one pass (trainer.py:240-244): online(s'), target(s')
// and online(s) for the tile's LROWS rows — the hidden layers of all three in one loop
// over the hidden units (12 independent FMA chains per thread), then all 3 LROWS M
// outputs with several (row, tier) pairs per warp in flight.  Fixed arithmetic per
// output: h = relu((sum_d x_d W1[d][j], FMA chain in d order) + b1[j]); q = (lane-strided
// FMA chains over j, xor-butterfly tree) + b2[m] — identical on every execution path.
// w1 column j = threadIdx.x (wo, wt, bo, bt) arrives preloaded (the loads overlapped the
// batch gather); W2 / b2 of both networks are staged in shared memory (sw2 = [2][H][M],
// sb2 = [2][M]).
template <int DM>
__device__ __forceinline__ void load_w1_col(const double* w1, const double* b1, const double* tw1, const double* tb1,
                                            int D, int H, int j, double (&wo)[DM], double (&wt)[DM], double& bo,
                                            double& bt) {
    bo = b1[j];
    bt = tb1[j];
#pragma unroll
    for (int d = 0; d < DM; ++d) {
        wo[d] = d < D ? w1[d * H + j] : 0.0;
        wt[d] = d < D ? tw1[d * H + j] : 0.0;
    }
}

template <int DM>
__device__ void forward3_rows(const double* xs2, const double* xs, int D, int H, int M, const double* w1,
                              const double* b1, const double* tw1, const double* tb1, double (&wo)[DM],
                              double (&wt)[DM], double bo, double bt, const double* sw2, const double* sb2,
                              double* h2o, double* h2t, double* hs, double* q2, double* q2t, double* q) {
    for (int j = threadIdx.x; j < H; j += blockDim.x) {
        if (j != (int)threadIdx.x) load_w1_col<DM>(w1, b1, tw1, tb1, D, H, j, wo, wt, bo, bt);
#pragma unroll
        for (int row = 0; row < LROWS; ++row) {
            double a2o = 0.0, a2t = 0.0, ao = 0.0;
#pragma unroll
            for (int d = 0; d < DM; ++d)
                if (d < D) {
                    a2o = __fma_rn(xs2[row * D + d], wo[d], a2o);
                    a2t = __fma_rn(xs2[row * D + d], wt[d], a2t);
                    ao = __fma_rn(xs[row * D + d], wo[d], ao);
                }
            h2o[row * H + j] = relu_d(__dadd_rn(a2o, bo));
            h2t[row * H + j] = relu_d(__dadd_rn(a2t, bt));
            hs[row * H + j] = relu_d(__dadd_rn(ao, bo));
        }
    }
    __syncthreads();
    constexpr int PW = 4;  // pairs per warp in flight
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x >> 5;
    const int npair = LROWS * M;
    for (int pb = warp * PW; pb < 3 * npair; pb += nw * PW) {
        const double* hp[PW];
        const double* wp[PW];
        int mm[PW];
        double acc[PW];
#pragma unroll
        for (int i = 0; i < PW; ++i) {
            const int id = pb + i < 3 * npair ? pb + i : 3 * npair - 1;
            const int set = id / npair, pair = id % npair, row = pair / M;
            mm[i] = pair % M;
            hp[i] = (set == 0 ? h2o : set == 1 ? h2t : hs) + row * H;
            wp[i] = sw2 + (set == 1 ? H * M : 0);
            acc[i] = 0.0;
        }
        for (int j = lane; j < H; j += 32) {
#pragma unroll
            for (int i = 0; i < PW; ++i) acc[i] = __fma_rn(hp[i][j], wp[i][j * M + mm[i]], acc[i]);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
            for (int i = 0; i < PW; ++i) acc[i] = __dadd_rn(acc[i], __shfl_xor_sync(0xffffffffu, acc[i], off));
        }
        if (lane < PW && pb + lane < 3 * npair) {
            double v = acc[0];
#pragma unroll
            for (int i = 1; i < PW; ++i)
                if (lane == i) v = acc[i];
            const int id = pb + lane, set = id / npair, pair = id % npair;
            const double* bb = sb2 + (set == 1 ? M : 0);
            (set == 0 ? q2 : set == 1 ? q2t : q)[pair] = __dadd_rn(v, bb[pair % M]);
        }
    }
    __syncthreads();
}

struct ApplyParams {
    int32_t nparam;
    double* params;   // online [nparam] (w1, b1, w2, b2 contiguous)
    double* target;   // [nparam]
    double* m;
    double* v;
    double* grad;
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
// (trainer.py:288-289), one parameter per thread over many CTAs.  The
// bias corrections and the sync decision come from the step counters, which
// only the last CTA to finish advances (apply_finish), after every CTA read them.
struct AdamCoef {
    double bc0, bc1;
    bool sync;
};

__device__ __forceinline__ AdamCoef adam_coef(const ApplyParams& p) {
    AdamCoef a;
    const int64_t t = p.counters[0] + 1;
    a.bc0 = 1.0 - pow(p.beta1, (double)t);
    a.bc1 = 1.0 - pow(p.beta2, (double)t);
    const int64_t gs = p.counters[1] + 1;  // step_index = grad_steps + 1
    a.sync = (gs % p.sync_every) == 0;
    return a;
}

__device__ __forceinline__ void apply_elem(const ApplyParams& p, const AdamCoef& a, int k, double gk) {
    double w = p.params[k];
    if (p.adam) {
        double mk = __dadd_rn(__dmul_rn(p.m[k], p.beta1), __dmul_rn(1.0 - p.beta1, gk));
        double vk = __dadd_rn(__dmul_rn(p.v[k], p.beta2), __dmul_rn(__dmul_rn(1.0 - p.beta2, gk), gk));
        p.m[k] = mk;
        p.v[k] = vk;
        const double num = __dmul_rn(p.lr, __ddiv_rn(mk, a.bc0));
        const double den = __dadd_rn(__dsqrt_rn(__ddiv_rn(vk, a.bc1)), p.eps);
        w = __dsub_rn(w, __ddiv_rn(num, den));
    } else {
        w = __dsub_rn(w, __dmul_rn(p.lr, gk));
    }
    p.params[k] = w;
    if (a.sync) p.target[k] = w;
}

// apply_elem with w, m, v already loaded (the fused update prefetches them)
__device__ __forceinline__ void apply_elem_pre(const ApplyParams& p, const AdamCoef& a, int k, double gk, double w,
                                               double mk0, double vk0) {
    if (p.adam) {
        double mk = __dadd_rn(__dmul_rn(mk0, p.beta1), __dmul_rn(1.0 - p.beta1, gk));
        double vk = __dadd_rn(__dmul_rn(vk0, p.beta2), __dmul_rn(__dmul_rn(1.0 - p.beta2, gk), gk));
        p.m[k] = mk;
        p.v[k] = vk;
        const double num = __dmul_rn(p.lr, __ddiv_rn(mk, a.bc0));
        const double den = __dadd_rn(__dsqrt_rn(__ddiv_rn(vk, a.bc1)), p.eps);
        w = __dsub_rn(w, __ddiv_rn(num, den));
    } else {
        w = __dsub_rn(w, __dmul_rn(p.lr, gk));
    }
    p.params[k] = w;
    if (a.sync) p.target[k] = w;
}

__device__ __forceinline__ void apply_finish(const ApplyParams& p) {
    p.counters[0] += 1;
    p.counters[1] += 1;
    p.counters[2] = 1;
    *p.last_loss = *p.loss;
}

__device__ __forceinline__ bool update_gated(const ApplyParams& p) {
    return p.gate ? *p.gate == 0 : (p.sampling && p.ring_state[1] < p.min_size);
}

// Tile partial sums are stored hidden-unit-major: position j (D + 1 + M) + r holds
// hidden unit j's r-th parameter (r < D: W1[r][j]; r == D: b1[j]; else W2[j][r - D - 1]),
// then b2 and the loss — so the fused update's slice of hidden units reads one
// contiguous run.  pos_of / param_of convert between that and the parameter index
// (w1 | b1 | w2 | b2, the network's flat layout); the loss is nparam in both.
__device__ __forceinline__ int pos_of(int k, int D, int H, int M) {
    const int PU = D + 1 + M;
    if (k < D * H) return (k % H) * PU + k / H;
    if (k < D * H + H) return (k - D * H) * PU + D;
    if (k < D * H + H + H * M) {
        const int i = k - D * H - H;
        return (i / M) * PU + D + 1 + i % M;
    }
    return H * PU + (k - D * H - H - H * M);
}
__device__ __forceinline__ int param_of(int q, int D, int H, int M) {
    const int PU = D + 1 + M;
    if (q >= H * PU) return D * H + H + H * M + (q - H * PU);
    const int j = q / PU, r = q % PU;
    return r < D ? r * H + j : r == D ? D * H + j : D * H + H + j * M + (r - D - 1);
}

// Everything after the row tiles.  A CTA owns 32 consecutive parameters
// (k == nparam: the loss); warp w sums tiles [w n/8, (w + 1) n/8) in tile order
// and warp 0 adds the 8 slice sums in slice order — one fixed tree for every
// execution path, so host-driven, device-resident and graph runs agree bit for bit.
//   reduce: grad[k] = that sum, loss = sum / B;
//   apply:  the optimizer step from grad (reduce && apply: fused, one launch);
//   neither: only advance the iteration counter (updates_per_step == 0).
// Warm-up / DP gate closed: no update; a reduce-only launch zeroes grad (keeps a DP
// all-reduce well defined); the iteration counter still advances.
struct UpdateParams {
    int32_t n_tiles, B, reduce, apply;
    int32_t D, H, M;        // network shape (partial layout: pos_of)
    const double* partial;  // [n_tiles][nparam + 1]
    unsigned* done;         // CTA arrival counter (reset by the last CTA)
    ApplyParams ap;
};

__global__ void __launch_bounds__(UTHREADS) learner_update_kernel(const UpdateParams u) {
    pdl_wait();     // the previous one has completed and its writes are visible
    const ApplyParams& p = u.ap;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int k = blockIdx.x * 32 + lane;
    if (!u.reduce && !u.apply) {
        if (k == 0 && warp == 0 && p.advance) p.counters[3] += 1;
        return;
    }
    if (update_gated(p)) {
        if (warp == 0) {
            if (!u.apply && k < p.nparam) p.grad[k] = 0.0;
            if (u.apply && p.advance && k == 0) p.counters[3] += 1;
        }
        return;
    }
    __shared__ double slice[UTHREADS / 32][32];
    double gk = 0.0;
    if (u.reduce) {
        constexpr int NS = UTHREADS / 32;
        const int per = (u.n_tiles + NS - 1) / NS;
        const int t0 = warp * per, t1 = min(u.n_tiles, t0 + per);
        double s = 0.0;
        if (k <= p.nparam) {
            const size_t ld = (size_t)p.nparam + 1;
            const double* src = u.partial + pos_of(k, u.D, u.H, u.M);
#pragma unroll 8
            for (int t = t0; t < t1; ++t) s = __dadd_rn(s, __ldcg(src + (size_t)t * ld));
        }
        slice[warp][lane] = s;
        __syncthreads();
        if (warp != 0) return;
        s = slice[0][lane];
#pragma unroll
        for (int w = 1; w < NS; ++w) s = __dadd_rn(s, slice[w][lane]);
        if (k < p.nparam) p.grad[k] = gk = s;
        else if (k == p.nparam) *p.loss = __ddiv_rn(s, (double)u.B);
    } else {
        if (warp != 0) return;
        if (k < p.nparam) gk = p.grad[k];
    }
    if (!u.apply) return;
    // warp 0 only from here
    const AdamCoef a = adam_coef(p);
    if (k < p.nparam) apply_elem(p, a, k, gk);
    __threadfence();
    __syncwarp();
    if (lane == 0 && atomicAdd(u.done, 1u) == gridDim.x - 1) {
        __threadfence();
        apply_finish(p);
        if (p.advance) p.counters[3] += 1;
        *u.done = 0u;
    }
}

// ------------------------------------------- data-parallel update over peer memory
// The DP learner without a collective library: each rank's update kernel reduces
// its own row tiles into an exchange buffer, publishes it with a release store of
// the update's epoch, waits (acquire, system scope) until every rank published the
// same epoch, then sums all ranks' gradients in rank order straight out of their
// exchange buffers (NVLink peer memory, or the same GPU), scales by 1/W and applies
// Adam — the same arithmetic as "all-reduce (sum) then x 1/W" for every rank, so
// the replicas stay bit-identical, with no NCCL launch on the update path.
// Readiness ("replay holds max(batch, warmup)") travels in the same buffer: the
// update runs iff every rank is ready (the NCCL path's MIN all-reduce of the gate).
// Exchange buffers are double-buffered by epoch parity: a rank can be at most one
// epoch ahead of the slowest (it waits for everyone's flag), so it never overwrites
// a buffer a peer may still be reading.
constexpr int XMAX_RANKS = 16;
constexpr unsigned long long XWAIT_NS = 2000000000ull;  // 2 s without a peer: fail loudly, never hang

struct XParams {
    int32_t world, rank;
    double* xbuf_self;                            // [2][nparam + 2]
    unsigned long long* flag_self;                // [1] last published epoch
    const double* xbuf[XMAX_RANKS];               // every rank's exchange buffer (own included)
    const unsigned long long* flag[XMAX_RANKS];
    unsigned* done;                               // [2] CTA tickets (publish, finish)
    int32_t* status;
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ double ld_relaxed_sys(const double* p) {
    double v;
    asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(UTHREADS) learner_xupdate_kernel(const UpdateParams u, const XParams x) {
    pdl_wait();
    const ApplyParams& p = u.ap;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int k = blockIdx.x * 32 + lane;
    const int ld = p.nparam + 2;
    // epoch of this update: counters[4] advances only in the last CTA of the finish ticket
    const unsigned long long epoch = (unsigned long long)p.counters[4] + 1ull;
    const int par = (int)(epoch & 1ull);
    double* mine = x.xbuf_self + (size_t)par * ld;
    const bool ready = !(p.sampling && p.ring_state[1] < p.min_size);  // local replay readiness
    // ---- publish: this rank's tile sums (same fixed tree as learner_update_kernel)
    __shared__ double slice[UTHREADS / 32][32];
    __shared__ int all_ready;
    if (ready) {
        constexpr int NS = UTHREADS / 32;
        const int per = (u.n_tiles + NS - 1) / NS;
        const int t0 = warp * per, t1 = min(u.n_tiles, t0 + per);
        double sum = 0.0;
        if (k <= p.nparam) {
            const double* src = u.partial + pos_of(k, u.D, u.H, u.M);
            const size_t pld = (size_t)p.nparam + 1;
#pragma unroll 8
            for (int t = t0; t < t1; ++t) sum = __dadd_rn(sum, __ldcg(src + (size_t)t * pld));
        }
        slice[warp][lane] = sum;
        __syncthreads();
        if (warp == 0 && k <= p.nparam) {
            double s = slice[0][lane];
#pragma unroll
            for (int w = 1; w < NS; ++w) s = __dadd_rn(s, slice[w][lane]);
            mine[k] = s;  // k == nparam: the local loss sum
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) mine[p.nparam + 1] = ready ? 1.0 : 0.0;
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(&x.done[0], 1u) == gridDim.x - 1) {
        x.done[0] = 0u;
        __threadfence_system();
        st_release_sys(x.flag_self, epoch);
    }
    // ---- wait for every rank's epoch (bounded: a missing peer is an error, not a hang)
    if (threadIdx.x == 0) {
        int ok = 1;
        unsigned long long t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (int r = 0; r < x.world; ++r) {
            while (ld_acquire_sys(x.flag[r]) < epoch) {
                unsigned long long now;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                if (now - t0 > XWAIT_NS) {
                    ok = 0;
                    if (atomicCAS(&x.status[0], 0, BE_ECUDA) == 0) x.status[1] = r;
                    break;
                }
                __nanosleep(64);
            }
        }
        int rd = ok;
        for (int r = 0; r < x.world && rd; ++r) rd = ld_relaxed_sys(x.xbuf[r] + (size_t)par * ld + p.nparam + 1) != 0.0;
        all_ready = rd;
    }
    __syncthreads();
    if (all_ready && warp == 0) {
        if (k < p.nparam) {
            double s = 0.0;
            for (int r = 0; r < x.world; ++r) s = __dadd_rn(s, ld_relaxed_sys(x.xbuf[r] + (size_t)par * ld + k));
            const double g = __dmul_rn(s, __ddiv_rn(1.0, (double)x.world));
            p.grad[k] = g;
            apply_elem(p, adam_coef(p), k, g);
        } else if (k == p.nparam) {
            *p.loss = __ddiv_rn(mine[k], (double)u.B);  // local loss, as the NCCL path logs it
        }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(&x.done[1], 1u) == gridDim.x - 1) {
        __threadfence();
        if (all_ready) apply_finish(p);
        if (p.advance) p.counters[3] += 1;
        p.counters[4] = (long long)epoch;
        x.done[1] = 0u;
    }
}

// ------------------------------------------- fused update (learner_partial_kernel tail)
// The TD/Huber backward and the optimizer step in ONE launch: every tile CTA takes a
// ticket after writing its partial sums; the last tail_ns to arrive (at most TAIL_CTAS,
// and fewer than the GPU holds at once, so the tiles they wait for always find a slot)
// wait for the remaining tiles, then each reduces the partials of one slice of hidden units — w1[:, j],
// b1[j], w2[j, :] for j in the slice (slice 0 also b2 and the loss) — with exactly
// learner_update_kernel's fixed tree (8 tile slices summed in tile order, then in slice
// order), applies Adam / SGD (apply_elem) and repacks those units' entries of the env
// step's weight layout (QLayout, stage_qnet's values).  The last slice to finish advances
// the counters (apply_finish).  Bit-identical to partial + learner_update_kernel.
constexpr int TAIL_CTAS = 128;  // at most (measured: 128 > 64 > 32 at batch 512)

// fetch-add with release semantics at GPU scope: the CTA's writes this thread observed
// through the preceding barrier are ordered before the ticket (cumulativity)
__device__ __forceinline__ unsigned long long atom_add_release_gpu(unsigned long long* a, unsigned long long v) {
    unsigned long long old;
    asm volatile("atom.add.release.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(a), "l"(v) : "memory");
    return old;
}
__device__ __forceinline__ unsigned long long atom_add_acq_rel_gpu(unsigned long long* a, unsigned long long v) {
    unsigned long long old;
    asm volatile("atom.add.acq_rel.gpu.global.u64 %0, [%1], %2;" : "=l"(old) : "l"(a), "l"(v) : "memory");
    return old;
}

__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* a) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}

// partial-sum position (pos_of) of item i of a slice of hidden units [j0, j0 + nj):
// the slice's contiguous run, then (slice 0) b2 and the loss; -1 past the end
__device__ __forceinline__ int tail_pos(int i, int j0, int nj, int D, int H, int M, bool extras) {
    const int PU = D + 1 + M;
    if (i < nj * PU) return j0 * PU + i;
    i -= nj * PU;
    if (extras && i <= M) return H * PU + i;  // b2[i], i == M: the loss
    return -1;
}

__device__ void learner_tail(const LearnParams& p, const ApplyParams& ap, int nparam) {
    __shared__ unsigned long long rank_sh;
    __shared__ double part[2][UTHREADS / 32][32];
    __syncthreads();  // every thread's partial sums are written
    if (threadIdx.x == 0) rank_sh = atom_add_release_gpu(p.tick, 1ull);
    __syncthreads();
    const unsigned long long nt = gridDim.x, v = rank_sh;
    const int NS = p.tail_ns;
    const unsigned long long rank = v % nt;
    if (rank < nt - NS) return;
    const int slice = (int)(rank - (nt - NS));
    const AdamCoef a = adam_coef(ap);  // (overlaps the wait)
    if (threadIdx.x == 0) {
        const unsigned long long target = (v / nt + 1) * nt;
        while (ld_acquire_gpu(p.tick) < target) __nanosleep(32);
    }
    __syncthreads();
    const int D = p.D, H = p.H, M = p.M;
    const int U = (H + NS - 1) / NS;
    const int j0 = slice * U, nj = j0 < H ? min(U, H - j0) : 0;
    const bool extras = slice == 0;
    const int n_items = nj * (D + 1 + M) + (extras ? M + 1 : 0);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    constexpr int NSUB = UTHREADS / 32;
    const int n_tiles = (int)nt;
    const int per = (n_tiles + NSUB - 1) / NSUB;
    const int t0 = w * per, t1 = min(n_tiles, t0 + per);
    const size_t ld = (size_t)nparam + 1;
    for (int c0 = 0; c0 < n_items; c0 += 64) {  // two rounds of 32 items, loads of both in flight
        // the optimizer state of this thread's item (threads < 64), in flight with the sums
        const int qme = threadIdx.x < 64 ? tail_pos(c0 + threadIdx.x, j0, nj, D, H, M, extras) : -1;
        const int kme = qme >= 0 ? param_of(qme, D, H, M) : -1;
        double wme = 0.0, mme = 0.0, vme = 0.0;
        if (kme >= 0 && kme < nparam) {
            wme = ap.params[kme];
            if (ap.adam) {
                mme = ap.m[kme];
                vme = ap.v[kme];
            }
        }
        double sum[2] = {0.0, 0.0};
        int k2[2];
#pragma unroll
        for (int r = 0; r < 2; ++r) k2[r] = tail_pos(c0 + r * 32 + lane, j0, nj, D, H, M, extras);
        for (int tb = t0; tb < t1; tb += 16) {  // 16 tiles' loads in flight, then the in-order sum
            double x[2][16];
#pragma unroll
            for (int i = 0; i < 16; ++i)
#pragma unroll
                for (int r = 0; r < 2; ++r)
                    x[r][i] = (tb + i < t1 && k2[r] >= 0) ? __ldcg(p.partial + (size_t)(tb + i) * ld + k2[r]) : 0.0;
#pragma unroll
            for (int i = 0; i < 16; ++i)
#pragma unroll
                for (int r = 0; r < 2; ++r)
                    if (tb + i < t1) sum[r] = __dadd_rn(sum[r], x[r][i]);
        }
        part[0][w][lane] = sum[0];
        part[1][w][lane] = sum[1];
        __syncthreads();
        if (kme >= 0) {
            const int r = threadIdx.x >> 5;
            double g = part[r][0][lane];
#pragma unroll
            for (int q = 1; q < NSUB; ++q) g = __dadd_rn(g, part[r][q][lane]);
            if (kme < nparam) {
                ap.grad[kme] = g;
                apply_elem_pre(ap, a, kme, g, wme, mme, vme);
            } else {
                *ap.loss = __ddiv_rn(g, (double)p.B);
            }
        }
        __syncthreads();
    }
    // the env step's packed weights for this slice's hidden units (stage_qnet's values):
    // task rows W1[t][j] + b1[j], pairs / odd entries W1[T + v][j] (v <= M) and W2[j][v - M - 1]
    if (p.qpack) {
        const int T = p.T, NV = 2 * M + 1, NP = M;
        const double* w1 = ap.params;
        const double* b1 = ap.params + D * H;
        const double* w2 = ap.params + D * H + H;
        for (int i = threadIdx.x; i < nj * (T + NV); i += blockDim.x) {
            const int u = i / (T + NV), r = i % (T + NV), j = j0 + u;
            if (r < T) {
                p.qpack[(size_t)r * H + j] = __dadd_rn(w1[(size_t)r * H + j], b1[j]);
            } else {
                const int vv = r - T;
                const double x = vv <= M ? w1[(size_t)(T + vv) * H + j] : w2[(size_t)j * M + (vv - M - 1)];
                double* pairs = p.qpack + (size_t)T * H;
                if (vv < 2 * NP) pairs[((size_t)(vv >> 1) * H + j) * 2 + (vv & 1)] = x;
                else pairs[(size_t)2 * NP * H + j] = x;
            }
        }
        if (extras && threadIdx.x < M) p.qpack[(size_t)(T + NV) * H + threadIdx.x] = ap.params[D * H + H + H * M + threadIdx.x];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // acq_rel: this slice's counter reads are released before the ticket, and the
        // last slice acquires every other slice's (they read counters[0..1] first)
        if (atom_add_acq_rel_gpu(p.tick + 1, 1ull) % (unsigned long long)NS == (unsigned long long)(NS - 1)) {
            apply_finish(ap);
            if (ap.advance) ap.counters[3] += 1;
        }
    }
}

template <int DM>
__global__ void __launch_bounds__(LTHREADS) learner_partial_kernel(const LearnParams p, const ApplyParams ap) {
    extern __shared__ __align__(16) double lsm[];
    const int D = p.D, H = p.H, M = p.M;
    double* xs = lsm;                    // [LROWS][D]
    double* xs2 = xs + LROWS * D;        // [LROWS][D]
    double* hh = xs2 + LROWS * D;        // [LROWS][H]  online h(s)
    double* ht = hh + LROWS * H;         // [LROWS][H]  online h(s')
    double* ht2 = ht + LROWS * H;        // [LROWS][H]  target h(s')
    double* q = ht2 + LROWS * H;         // [LROWS][M]
    double* q2 = q + LROWS * M;          // [LROWS][M]
    double* q2t = q2 + LROWS * M;        // [LROWS][M]
    double* g = q2t + LROWS * M;         // [LROWS][M]  dL/dq
    double* rw = g + LROWS * M;          // [LROWS]
    double* cc = rw + LROWS;             // [LROWS]
    double* lrow = cc + LROWS;           // [LROWS] per-row loss
    double* sw2 = lrow + LROWS;          // [2][H][M] W2 online, target
    double* sb2 = sw2 + 2 * H * M;       // [2][M]    b2 online, target
    int* act = reinterpret_cast<int*>(sb2 + 2 * M);  // [LROWS]
    const int row0 = blockIdx.x * LROWS;
    const int nparam_ = D * H + H + H * M + M;
    // the tile's partial sums, staged for one coalesced copy out (when they fit)
    double* so = p.stage_out ? reinterpret_cast<double*>(act + ((LROWS + 1) & ~1)) : nullptr;
    const int nparam = D * H + H + H * M + M;
    double* out = p.partial + (size_t)blockIdx.x * (nparam + 1);
    // ---- the weights the forwards read (in flight during the batch gather), before the
    // wait: behind a programmatic launch the predecessor is the env step, and everything
    // this prologue reads was final before that step's own wait returned (measured: the
    // step triggering at its top instead of its end is slower — early CTAs compete)
    double wo[DM], wt[DM], bo = 0.0, bt = 0.0;
    if ((int)threadIdx.x < H) load_w1_col<DM>(p.w1, p.b1, p.tw1, p.tb1, D, H, threadIdx.x, wo, wt, bo, bt);
    for (int k = threadIdx.x; k < H * M; k += blockDim.x) {
        sw2[k] = p.w2[k];
        sw2[H * M + k] = p.tw2[k];
    }
    if ((int)threadIdx.x < M) {
        sb2[threadIdx.x] = p.b2[threadIdx.x];
        sb2[M + threadIdx.x] = p.tb2[threadIdx.x];
    }
    pdl_wait();  // the previous kernel has completed and its writes are visible
    if (p.gate ? *p.gate == 0 : (p.sampling && p.ring_state[1] < p.min_size)) {  // warm-up: no update
        // (fused update: the iteration still advances; nothing in this launch reads it)
        if (p.tail && ap.advance && blockIdx.x == 0 && threadIdx.x == 0) ap.counters[3] += 1;
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
    forward3_rows<DM>(xs2, xs, D, H, M, p.w1, p.b1, p.tw1, p.tb1, wo, wt, bo, bt, sw2, sb2, ht, ht2, hh, q2,
                      q2t, q);
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
        double dw2[BE_MAX_TIERS], db1 = 0.0, dw1[DM], w2j[BE_MAX_TIERS];
#pragma unroll
        for (int m = 0; m < BE_MAX_TIERS; ++m) {
            dw2[m] = 0.0;
            w2j[m] = m < M ? sw2[j * M + m] : 0.0;
        }
#pragma unroll
        for (int d = 0; d < DM; ++d) dw1[d] = 0.0;
#pragma unroll
        for (int row = 0; row < LROWS; ++row) {
            const double hv = hh[row * H + j];
            double dh = 0.0;
#pragma unroll
            for (int m = 0; m < BE_MAX_TIERS; ++m) {
                if (m < M) {
                    const double gm = g[row * M + m];
                    dw2[m] = __fma_rn(hv, gm, dw2[m]);
                    dh = __fma_rn(gm, w2j[m], dh);
                }
            }
            if (!(hv > 0.0)) dh = 0.0;  // dh[h <= 0] = 0
            db1 = __dadd_rn(db1, dh);
#pragma unroll
            for (int d = 0; d < DM; ++d)
                if (d < D) dw1[d] = __fma_rn(xs[row * D + d], dh, dw1[d]);
        }
        double* oj = (so ? so : out) + j * (D + 1 + M);  // hidden-unit-major (pos_of)
#pragma unroll
        for (int d = 0; d < DM; ++d)
            if (d < D) oj[d] = dw1[d];
        oj[D] = db1;
#pragma unroll
        for (int m = 0; m < BE_MAX_TIERS; ++m)
            if (m < M) oj[D + 1 + m] = dw2[m];
    }
    if (threadIdx.x < M) {
        double s = 0.0;
        for (int row = 0; row < LROWS; ++row) s = __dadd_rn(s, g[row * M + threadIdx.x]);
        (so ? so : out)[H * (D + 1 + M) + threadIdx.x] = s;
    }
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int row = 0; row < LROWS; ++row) s = __dadd_rn(s, lrow[row]);
        (so ? so : out)[nparam] = s;
    }
    if (so) {
        __syncthreads();
        for (int i = threadIdx.x; i <= nparam_; i += blockDim.x) out[i] = so[i];
    }
    if (p.tail) learner_tail(p, ap, nparam);
    pdl_trigger();
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
    int32_t* status;
    double* wl_state;  // [E][3]
    // be_train_iteration: per-env arrival / task / true rate of the current iteration
    double* it_arrival;
    uint8_t* it_task;
    double* it_rate;
    unsigned* done;    // fused-update CTA arrival counter
    unsigned long long* scan;  // commit look-back state [(E + 7) / 8]
    unsigned* ticket;          // commit ticket / epoch; [2] the fused step+commit's scan epoch
    unsigned long long* scan16;  // fused step+commit look-back state [(E + 15) / 16]
    unsigned long long* tick;    // fused learner update tickets (learner_tail)
    // the env whose packed step weights (d_qpack) hold the current parameters: the fused
    // update (learner_tail) repacks them, every other parameter write clears this
    const be_env* qpack_env;
    // peer exchange (phase 4): one allocation = [2][nparam + 2] doubles + the epoch flag
    void* xmem;
    int32_t x_world, x_rank;
    const double* x_buf[XMAX_RANKS];
    const unsigned long long* x_flag[XMAX_RANKS];
    void* x_opened[XMAX_RANKS];  // peer allocations opened through CUDA IPC (closed at destroy)
    int64_t* gate;     // DP update gate (be_train_iteration use_gate)
    // tensor-core router (be_train_iteration router = BE_ROUTER_TC): packed weight image
    // (rebuilt every iteration: the weights change with every update) and statistics
    int64_t* crange;    // [E][3] completion id range of the step + oldest in flight (commits)
    void* tc_img;       // NULL when the network shape is outside route_tc's support
    int64_t* tc_stats;  // [2] states routed, fp64 re-evaluations
};

static void learner_free(be_learner* L) {
    void* ptrs[] = {L->params, L->target, L->m, L->v, L->grad, L->partial, L->loss, L->counters,
                    L->rs, L->rs2, L->rr, L->rc, L->ra, L->ring_state, L->px, L->pa, L->pflags,
                    L->preward, L->low, L->status, L->wl_state,
                    L->it_arrival, L->it_task, L->it_rate, L->done, L->gate, L->scan, L->ticket,
                    L->tc_img, L->tc_stats, L->crange, L->scan16, L->tick};
    for (void* p : ptrs) cudaFree(p);
    for (int r = 0; r < XMAX_RANKS; ++r)
        if (L->x_opened[r]) cudaIpcCloseMemHandle(L->x_opened[r]);
    cudaFree(L->xmem);
    delete L;
}

static size_t xmem_bytes(const be_learner* L) { return (size_t)2 * (L->nparam + 2) * sizeof(double) + 64; }
static double* x_buf_self(const be_learner* L) { return reinterpret_cast<double*>(L->xmem); }
static unsigned long long* x_flag_self(const be_learner* L) {
    return reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(L->xmem) +
                                                 (size_t)2 * (L->nparam + 2) * sizeof(double));
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
        {(void**)&L->status, 64},
        {(void**)&L->wl_state, E * 3 * 8}, {(void**)&L->it_arrival, E * 8},
        {(void**)&L->it_task, E}, {(void**)&L->it_rate, E * 8}, {(void**)&L->done, 64}, {(void**)&L->gate, 64},
        {(void**)&L->scan, ((E + CENVS - 1) / CENVS) * 8}, {(void**)&L->ticket, 64},
        {(void**)&L->crange, E * 3 * 8}, {(void**)&L->scan16, ((E + 15) / 16) * 8},
        {(void**)&L->tick, 64}};
    for (auto& a : allocs) {
        e = cudaMalloc(a.p, a.n);
        if (e != cudaSuccess) {
            learner_free(L);
            return set_cuda_error(e, "be_learner_create: cudaMalloc");
        }
        cudaMemset(*a.p, 0, a.n);
    }
    e = cudaMalloc(&L->xmem, xmem_bytes(L));
    if (e != cudaSuccess) {
        learner_free(L);
        return set_cuda_error(e, "be_learner_create: exchange buffer");
    }
    cudaMemset(L->xmem, 0, xmem_bytes(L));
    if (route_tc_supported(c->n_tasks, c->n_tiers, c->hidden)) {
        if ((e = cudaMalloc(&L->tc_img, route_tc_workspace_bytes(c->hidden))) != cudaSuccess ||
            (e = cudaMalloc((void**)&L->tc_stats, 16)) != cudaSuccess) {
            learner_free(L);
            return set_cuda_error(e, "be_learner_create: tensor-core router workspace");
        }
        cudaMemset(L->tc_stats, 0, 16);
        route_tc_prepare(c->n_tasks, c->n_tiers, c->hidden);
        step_tc_prepare(c->n_tiers, c->hidden);
    }
    // configured here, not at launch time: launches may be captured in a CUDA graph
    cudaFuncSetAttribute(learner_partial_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(learner_partial_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(learner_partial_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
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
    cudaMemsetAsync(L->xmem, 0, xmem_bytes(L), st);  // peer-exchange epochs restart with the counters
    L->qpack_env = nullptr;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "set_params");
}

int32_t be_learner_views(be_learner* L, be_learner_views_t* v) {
    if (!L || !v) return set_error(BE_EINVAL, "NULL argument");
    const int D = L->D, H = L->cfg.hidden, M = L->cfg.n_tiers;
    v->online.hidden = H;
    v->online.n_tasks = (int16_t)L->cfg.n_tasks;
    v->online.n_tiers = (int16_t)M;
    v->online.w1 = L->params;
    v->online.b1 = L->params + D * H;
    v->online.w2 = L->params + D * H + H;
    v->online.b2 = L->params + D * H + H + H * M;
    v->target.hidden = H;
    v->target.n_tasks = (int16_t)L->cfg.n_tasks;
    v->target.n_tiers = (int16_t)M;
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
    WorkloadArgs w{E, L->wl_state, log(c.rate_low), log(c.rate_high), c.regime_equal_time, c.regime_mean_seconds,
                   c.regime_mean_requests, c.n_tasks, seed, (uint64_t)step, arrival_ms, task, true_rate, nullptr};
    cudaError_t e = launch_pdl(train_workload_kernel, dim3((E + 255) / 256), dim3(256), 0, (cudaStream_t)stream, w);
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "workload launch");
}

static int commit_impl(be_learner* L, int64_t step, const int64_t* step_dev, cudaStream_t st,
                       const int64_t* crange = nullptr) {
    CommitParams p{};
    p.step_dev = step_dev;
    p.crange = crange;
    p.E = L->cfg.n_envs;
    p.D = L->D;
    p.P = L->cfg.pending_capacity;
    p.step = step;
    p.px = L->px;
    p.pa = L->pa;
    p.pflags = L->pflags;
    p.preward = L->preward;
    p.low = L->low;
    p.ring_state = L->ring_state;
    p.capacity = L->cfg.replay_capacity;
    p.rs = L->rs;
    p.rs2 = L->rs2;
    p.ra = L->ra;
    p.rr = L->rr;
    p.rc = L->rc;
    p.status = L->status;
    p.scan = L->scan;
    p.ticket = L->ticket;
    cudaError_t e = launch_pdl(commit_fused_kernel, dim3((p.E + CENVS - 1) / CENVS), dim3(CENVS * 32), 0, st, p);
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "commit launch");
}

int32_t be_learner_commit(be_learner* L, int64_t step, void* stream) {
    if (!L || step < 0) return set_error(BE_EINVAL, "bad argument");
    return commit_impl(L, step, nullptr, (cudaStream_t)stream);
}

static ApplyParams apply_params(be_learner* L, int32_t explicit_batch, int32_t advance);

static int launch_update(be_learner* L, int reduce, int apply, ApplyParams ap, const int64_t* gate,
                         cudaStream_t st) {
    UpdateParams u{};
    u.n_tiles = L->n_tiles;
    u.B = L->cfg.batch;
    u.D = L->D;
    u.H = L->cfg.hidden;
    u.M = L->cfg.n_tiers;
    u.reduce = reduce;
    u.apply = apply;
    u.partial = L->partial;
    u.done = L->done;
    ap.gate = gate;
    u.ap = ap;
    const int blocks = (reduce || apply) ? (L->nparam + 32) / 32 : 1;  // 32 parameters (+ the loss) per CTA
    if (apply) L->qpack_env = nullptr;
    cudaError_t e = launch_pdl(learner_update_kernel, dim3(blocks), dim3(UTHREADS), 0, st, u);
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "learner update launch");
}

static int launch_xupdate(be_learner* L, int32_t advance, cudaStream_t st) {
    UpdateParams u{};
    u.n_tiles = L->n_tiles;
    u.B = L->cfg.batch;
    u.D = L->D;
    u.H = L->cfg.hidden;
    u.M = L->cfg.n_tiers;
    u.reduce = 1;
    u.apply = 1;
    u.partial = L->partial;
    u.done = L->done;
    u.ap = apply_params(L, 0, advance);
    L->qpack_env = nullptr;
    XParams x{};
    x.world = L->x_world;
    x.rank = L->x_rank;
    x.xbuf_self = x_buf_self(L);
    x.flag_self = x_flag_self(L);
    for (int r = 0; r < L->x_world; ++r) {
        x.xbuf[r] = L->x_buf[r];
        x.flag[r] = L->x_flag[r];
    }
    x.done = L->done + 1;
    x.status = L->status;
    const int blocks = (L->nparam + 32) / 32;
    cudaError_t e = launch_pdl(learner_xupdate_kernel, dim3(blocks), dim3(UTHREADS), 0, st, u, x);
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "learner peer-exchange update launch");
}

static int learner_backward_impl(be_learner* L, const double* s, const uint8_t* a, const double* r,
                                 const double* s2, const double* c, int32_t B, uint64_t seed,
                                 uint64_t counter, int64_t* sample_idx, cudaStream_t st,
                                 const int64_t* iter_dev = nullptr, int32_t ups = 1, int32_t uidx = 0,
                                 int32_t fused = 0, int32_t advance = 0,
                                 const int64_t* gate = nullptr, int32_t partials_only = 0,
                                 int32_t tail = 0, double* qpack = nullptr) {
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
    size_t smem = sizeof(double) * (2 * LROWS * D + 3 * LROWS * H + 4 * LROWS * M + 3 * LROWS + 2 * H * M + 2 * M) +
                  sizeof(int) * ((LROWS + 1) & ~1);
    const size_t stage = sizeof(double) * ((size_t)L->nparam + 1);
    if (smem + stage <= 200 * 1024) {
        p.stage_out = 1;
        smem += stage;
    }
    if (smem > 200 * 1024) return set_error(BE_EINVAL, "hidden too large for the learner tile");
    ApplyParams ap{};
    auto kern = D <= 8 ? learner_partial_kernel<8> : D <= 16 ? learner_partial_kernel<16> : learner_partial_kernel<32>;
    if (tail) {  // backward + optimizer in this one launch (learner_tail)
        // the tail CTAs spin until every tile has arrived: fewer of them than the
        // GPU holds at once, so the tiles they wait for always find a slot
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, LTHREADS, smem);
        int ns = TAIL_CTAS < L->n_tiles ? TAIL_CTAS : L->n_tiles;
        if (ns > sms * per_sm - 1) ns = sms * per_sm - 1;
        if (ns < 1) return set_error(BE_EINVAL, "learner tile does not fit the GPU");
        p.tail_ns = ns;
        ap = apply_params(L, sampling ? 0 : 1, advance);
        ap.gate = gate;
        p.tail = 1;
        p.tick = L->tick;
        p.qpack = qpack;
        p.T = cf.n_tasks;
    }
    if (tail && uidx == 0) {
        // be_train_iteration's first update follows the env step, which triggers at its
        // end: a programmatic launch hides this launch's latency (the weight prologue
        // reads only what the step itself waited for; +0.5%)
        cudaError_t e2 = launch_pdl(kern, dim3(L->n_tiles), dim3(LTHREADS), smem, st, p, ap);
        if (e2 != cudaSuccess) return set_cuda_error(e2, "learner launch");
        return BE_OK;
    }
    kern<<<L->n_tiles, LTHREADS, smem, st>>>(p, ap);
    // fused: tile reduction + optimizer step in one launch; else tile reduction -> grad
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e, "learner launch");
    if (partials_only || tail) return BE_OK;
    return launch_update(L, 1, fused, apply_params(L, sampling ? 0 : 1, fused ? advance : 0), gate, st);
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
    return launch_update(L, 0, 1, apply_params(L, explicit_batch, 0), nullptr, (cudaStream_t)stream);
}

int32_t be_learner_exchange_buffer(be_learner* L, void** xmem, size_t* bytes) {
    if (!L || !xmem) return set_error(BE_EINVAL, "NULL argument");
    *xmem = L->xmem;
    if (bytes) *bytes = xmem_bytes(L);
    return BE_OK;
}

int32_t be_learner_ipc_handle(be_learner* L, void* handle_out) {
    if (!L || !handle_out) return set_error(BE_EINVAL, "NULL argument");
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, L->xmem);
    if (e != cudaSuccess) return set_cuda_error(e, "be_learner_ipc_handle");
    memcpy(handle_out, &h, sizeof(h));
    return BE_OK;
}

int32_t be_learner_set_peers(be_learner* L, int32_t world, int32_t rank, const uint64_t* xmems) {
    if (!L || !xmems) return set_error(BE_EINVAL, "NULL argument");
    if (world < 1 || world > XMAX_RANKS || rank < 0 || rank >= world)
        return set_error(BE_EINVAL, "world must be in [1, 16] and 0 <= rank < world");
    if ((void*)(uintptr_t)xmems[rank] != L->xmem) return set_error(BE_EINVAL, "xmems[rank] is not this learner's buffer");
    const size_t off = (size_t)2 * (L->nparam + 2) * sizeof(double);
    for (int r = 0; r < world; ++r) {
        if (!xmems[r]) return set_error(BE_EINVAL, "missing peer buffer");
        L->x_buf[r] = reinterpret_cast<const double*>((uintptr_t)xmems[r]);
        L->x_flag[r] = reinterpret_cast<const unsigned long long*>((uintptr_t)xmems[r] + off);
    }
    L->x_world = world;
    L->x_rank = rank;
    return BE_OK;
}

int32_t be_learner_open_peers_ipc(be_learner* L, int32_t world, int32_t rank, const void* handles) {
    if (!L || !handles) return set_error(BE_EINVAL, "NULL argument");
    if (world < 1 || world > XMAX_RANKS || rank < 0 || rank >= world)
        return set_error(BE_EINVAL, "world must be in [1, 16] and 0 <= rank < world");
    uint64_t ptrs[XMAX_RANKS] = {0};
    for (int r = 0; r < world; ++r) {
        if (r == rank) {
            ptrs[r] = (uint64_t)(uintptr_t)L->xmem;
            continue;
        }
        if (L->x_opened[r]) {
            cudaIpcCloseMemHandle(L->x_opened[r]);
            L->x_opened[r] = nullptr;
        }
        cudaIpcMemHandle_t h;
        memcpy(&h, reinterpret_cast<const char*>(handles) + (size_t)r * sizeof(h), sizeof(h));
        void* ptr = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return set_cuda_error(e, "be_learner_open_peers_ipc");
        L->x_opened[r] = ptr;
        ptrs[r] = (uint64_t)(uintptr_t)ptr;
    }
    return be_learner_set_peers(L, world, rank, ptrs);
}

int32_t be_train_iteration(be_learner* L, be_env* env, const be_train_iter_cfg* c, void* stream) {
    if (!L || !env || !c) return set_error(BE_EINVAL, "NULL argument");
    const be_learner_cfg& cf = L->cfg;
    cudaStream_t st = (cudaStream_t)stream;
    if (env->E != cf.n_envs || env->cfg.n_tiers != cf.n_tiers || env->cfg.n_tasks != cf.n_tasks)
        return set_error(BE_EINVAL, "env and learner shapes differ");
    if (c->phase == 4 && L->x_world < 1) return set_error(BE_EINVAL, "phase 4 needs be_learner_set_peers first");
    if (c->updates_per_step < 0 || c->phase < 0 || c->phase > 4 || c->update_index < 0 ||
        ((c->phase == 1 || c->phase == 2) && c->update_index >= c->updates_per_step))
        return set_error(BE_EINVAL, "bad phase / update index");
    if (!(cf.rate_low > 0) || cf.rate_high < cf.rate_low)
        return set_error(BE_EINVAL, "need 0 < rate_low <= rate_high");
    if (c->router != BE_ROUTER_FP64 && c->router != BE_ROUTER_TC) return set_error(BE_EINVAL, "unknown router");
    if (c->router == BE_ROUTER_TC && !L->tc_img)
        return set_error(BE_EINVAL, "the tensor-core router needs n_tiers <= 4, n_tasks + n_tiers + 2 <= 16 and "
                                    "hidden a multiple of 32 in [32, 256]");
    const int64_t* it = L->counters + 3;
    const int E = cf.n_envs, D = L->D, H = cf.hidden, M = cf.n_tiers;
    int rc;
    const int64_t* gate = c->use_gate ? L->gate : nullptr;
    if (c->phase == 0 || c->phase == 3 || c->phase == 4) {
        // workload (trainer.py:375) -> env step (:376-395) -> commits (:143-156); the
        // workload rides in the env step's weight-packing launch
        const WorkloadArgs wl{E, L->wl_state, log(cf.rate_low), log(cf.rate_high), cf.regime_equal_time,
                              cf.regime_mean_seconds, cf.regime_mean_requests, cf.n_tasks, c->workload_seed, 0,
                              L->it_arrival, L->it_task, L->it_rate, it};
        be_qweights W;
        W.hidden = H;
        W.n_tasks = (int16_t)cf.n_tasks;
        W.n_tiers = (int16_t)M;
        W.w1 = L->params;
        W.b1 = L->params + D * H;
        W.w2 = L->params + D * H + H;
        W.b2 = L->params + D * H + H + H * M;
        be_records rec{};
        rec.flags = L->pflags;
        rec.reward = L->preward;
        bool fused_commit = false;
        const bool fuse = env_step_commit_supported(env) && (c->router != BE_ROUTER_TC || env->R <= 16);
        StepCommitArgs cm{cf.replay_capacity, L->rs, L->rs2, L->rr, L->rc, L->ra, L->low,
                          L->ring_state, L->status, L->scan16, L->ticket + 2, 0, L->ticket + 4, 0};
        if (fuse && L->qpack_env != env) {
            // the step reads the packed fp64 weights the learner's fused update keeps
            // current; pack them here once if anything else wrote the parameters
            rc = launch_stage_qpack(env, &W, st);
            if (rc) return rc;
            L->qpack_env = env;
        }
        if (c->router == BE_ROUTER_TC && env->R <= 16) {
            // the decision on the tensor cores inside the env step (+ arrivals + replay
            // commit): the router image is repacked, then env_step_commit_kernel<M, true>
            // runs layer 1 of 16 envs per CTA as one tcgen05 tile (certified, fp64
            // fallback: the fp64 step's decisions)
            rc = launch_env_step_dev(env, L->it_arrival, L->it_task, L->it_rate, &W, c->policy_seed, it,
                                     c->epsilon_start, c->epsilon_end, c->epsilon_decay_steps,
                                     cf.pending_capacity, cf.pending_capacity, &rec, L->pa, L->px, st, &wl, 0,
                                     reinterpret_cast<float*>(L->tc_img), nullptr, fuse ? &cm : nullptr);
            fused_commit = fuse;
        } else if (c->router == BE_ROUTER_TC) {
            // > 16 replicas per env: observe + encode (pending slot) -> the batched
            // tcgen05 router on the E states -> submit
            rc = launch_env_step_dev(env, L->it_arrival, L->it_task, L->it_rate, &W, c->policy_seed, it,
                                     c->epsilon_start, c->epsilon_end, c->epsilon_decay_steps,
                                     cf.pending_capacity, cf.pending_capacity, &rec, L->pa, L->px, st, &wl, 1,
                                     nullptr, L->crange);
            if (rc) return rc;
            rc = launch_route_tc_dev(&W, cf.n_tasks, M, L->px, E, c->policy_seed, it, c->epsilon_start,
                                     c->epsilon_end, c->epsilon_decay_steps, cf.pending_capacity, L->pa,
                                     L->tc_img, L->tc_stats, st);
            if (rc) return rc;
            rc = launch_env_step_dev(env, L->it_arrival, L->it_task, L->it_rate, &W, c->policy_seed, it,
                                     c->epsilon_start, c->epsilon_end, c->epsilon_decay_steps,
                                     cf.pending_capacity, cf.pending_capacity, &rec, L->pa, L->px, st, nullptr, 2,
                                     nullptr, L->crange);
        } else if (fuse) {
            // the replay commit fused into the env step: one launch, no flag scan; the
            // step generates the arrivals itself
            rc = launch_env_step_dev(env, L->it_arrival, L->it_task, L->it_rate, &W, c->policy_seed, it,
                                     c->epsilon_start, c->epsilon_end, c->epsilon_decay_steps,
                                     cf.pending_capacity, cf.pending_capacity, &rec, L->pa, L->px, st, &wl, 0,
                                     nullptr, nullptr, &cm);
            if (rc) return rc;
            fused_commit = true;
        } else {
            rc = launch_env_step_dev(env, L->it_arrival, L->it_task, L->it_rate, &W, c->policy_seed, it,
                                     c->epsilon_start, c->epsilon_end, c->epsilon_decay_steps,
                                     cf.pending_capacity, cf.pending_capacity, &rec, L->pa, L->px, st, &wl, 0,
                                     nullptr, L->crange);
        }
        if (rc) return rc;
        if (!fused_commit) {
            rc = commit_impl(L, 0, it, st, L->crange);
            if (rc) return rc;
        }
    }
    const int ups = c->updates_per_step;
    if (c->phase == 0) {
        for (int u = 0; u < ups; ++u) {
            rc = learner_backward_impl(L, nullptr, nullptr, nullptr, nullptr, nullptr, cf.batch,
                                       c->sample_seed, 0, nullptr, st, it, ups, u, 1, u == ups - 1, nullptr, 0,
                                       /*tail=*/1, env->d_qpack);
            if (rc) return rc;
        }
        if (ups == 0) {  // no learner: still advance the iteration
            rc = launch_update(L, 0, 0, apply_params(L, 1, 1), nullptr, st);
            if (rc) return rc;
        }
    } else if (c->phase == 1) {
        rc = learner_backward_impl(L, nullptr, nullptr, nullptr, nullptr, nullptr, cf.batch,
                                   c->sample_seed, 0, nullptr, st, it, ups, c->update_index, 0, 0,
                                   gate);
        if (rc) return rc;
    } else if (c->phase == 4) {
        // updates with the peer-memory gradient exchange (no collective library)
        for (int u = 0; u < ups; ++u) {
            rc = learner_backward_impl(L, nullptr, nullptr, nullptr, nullptr, nullptr, cf.batch, c->sample_seed,
                                       0, nullptr, st, it, ups, u, 0, 0, nullptr, /*partials_only=*/1);
            if (rc) return rc;
            rc = launch_xupdate(L, u == ups - 1, st);
            if (rc) return rc;
        }
        if (ups == 0) {
            rc = launch_update(L, 0, 0, apply_params(L, 1, 1), nullptr, st);
            if (rc) return rc;
        }
    } else if (c->phase == 2) {
        rc = launch_update(L, 0, 1, apply_params(L, 0, c->update_index == ups - 1), gate, st);
        if (rc) return rc;
    } else if (c->phase == 3 && ups == 0) {  // no phase 2 follows: advance the iteration here
        rc = launch_update(L, 0, 0, apply_params(L, 1, 1), nullptr, st);
        if (rc) return rc;
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
    if (st[0] == BE_ECUDA) {
        char msg[160];
        snprintf(msg, sizeof(msg), "peer gradient exchange: rank %d never published its update (timed out)", st[1]);
        return set_error(BE_ECUDA, msg);
    }
    return set_error(st[0], "pending-transition ring overflow: a request stayed in flight longer "
                            "than pending_capacity decisions; raise pending_capacity");
}

}  // extern "C"

