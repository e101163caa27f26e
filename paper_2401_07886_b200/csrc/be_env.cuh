// be_env.cuh — device-side building blocks of the batched serving environment.
//
// Layout (B200-first):
//   * one warp per environment, one lane per replica (sum of replicas <= 32);
//     lane state (pending event, iteration counter, FIFO cursor, cached FIFO
//     head) lives in registers for the whole rollout;
//   * each replica owns a FIFO ring of 16-byte slots in HBM: the reference's
//     `active` dict and `queue` deque (simcore.py:53-60) are one FIFO whose
//     first min(count, max_batch) entries are the active batch;
//   * per-env scalars (rate-estimator window, segment cursor) are warp-uniform
//     registers; per-tier reductions use REDUX (__reduce_*_sync).
//
// Exactness: every event-time operation uses explicit round-to-nearest
// intrinsics in the reference's evaluation order (simcore.py:146 evaluates
// `time + alpha + beta * n` as (time + alpha) + (beta * n)), so the
// translation unit's FMA contraction setting cannot change results.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "be200.h"
#include "be_internal.h"
#include "be_tc.cuh"

namespace be {

constexpr int K_NONE = 0;
constexpr int K_START = 1;
constexpr int K_END = 2;
constexpr unsigned FULL = 0xffffffffu;

// One FIFO entry: a submitted Request (simcore.py:40-50) reduced to what the
// event loop needs.  join = iteration counter at the START that first put the
// request in a running batch (tokens_done = iters - join), -1 before that.
struct __align__(16) Slot {
    double arrival;
    uint32_t idtask;  // request id (low 24 bits) | task id << 24
    int32_t join;
};

// Per-lane (= per-replica) state; the FIFO head is cached in registers.
struct Rep {
    double t;        // time of the pending event (kind != K_NONE)
    double h_arr;    // arrival of the FIFO head
    int kind;
    int iters;       // END events processed on this replica
    uint32_t head;   // monotone FIFO cursor (slot = head & mask)
    int count;       // len(active) + len(queue)
    int n_running;   // FIFO prefix that has joined an iteration
    int h_join;
    uint32_t h_idtask;
    int n_assigned;  // FIFO prefix whose join iteration is known (<= max_batch; see submit_lane)
};

struct TierC {
    double alpha;
    double beta;
    int max_batch;
    int tokens;
    int tier;
    const double* skip;  // this tier's skip table [n][SKIP_NB] (smem or global), or NULL
};

// Reward constants (reward.py:45-126) staged in shared memory.
struct Score {
    double deadline[BE_MAX_TASKS];
    double cut[BE_MAX_TASKS];  // cutoff_fraction * deadline (reward.py:108)
    double matrix[BE_MAX_TASKS * BE_MAX_TIERS];
    // hit_tau[t][m]: largest x with RN(x / tokens_m) <= deadline_t, so that for a
    // hard deadline "realized <= deadline" is exactly "(t_end - arrival) <= hit_tau"
    // (RN(x / c) is monotone in x) and no division is needed (host-computed).
    double hit_tau[BE_MAX_TASKS * BE_MAX_TIERS];
    int soft[BE_MAX_TASKS];
    double decay;
    int M;
};



// This env's record rows (element id at [id]): row pointers are formed once per
// env so every completion indexes with the 24-bit request id alone.
struct RecOut {
    uint8_t* flags;
    double* reward;
    double* realized;  // nullable
    __device__ __forceinline__ static RecOut row(const be_records& rec, int64_t base) {
        return RecOut{rec.flags + base, rec.reward + base, rec.realized ? rec.realized + base : nullptr};
    }
};

__device__ __forceinline__ void load_score(Score& s, const be_cfg& c, const ScoreAux& aux) {
    // called by a single warp; caller syncs
    int lane = threadIdx.x & 31;
    for (int k = lane; k < BE_MAX_TASKS * BE_MAX_TIERS; k += 32) s.hit_tau[k] = aux.hit_tau[k];
    for (int k = lane; k < BE_MAX_TASKS; k += 32) {
        s.deadline[k] = c.deadline[k];
        s.cut[k] = __dmul_rn(c.cutoff_fraction, c.deadline[k]);
        s.soft[k] = c.soft[k];
    }
    for (int k = lane; k < BE_MAX_TASKS * BE_MAX_TIERS; k += 32) {
        int t = k / BE_MAX_TIERS, m = k % BE_MAX_TIERS;
        s.matrix[k] = (t < c.n_tasks && m < c.n_tiers) ? c.matrix[t * c.n_tiers + m] : 0.0;
    }
    if (lane == 0) {
        s.decay = c.decay_per_ms;
        s.M = c.n_tiers;
    }
}

// lane -> (tier, constants); lanes beyond the replica count get tier = -1.
__device__ __forceinline__ TierC lane_tier(const be_cfg& c, int lane, const double* skip_tab = nullptr) {
    TierC tc;
    tc.alpha = 1.0;
    tc.beta = 0.0;
    tc.max_batch = 1;
    tc.tokens = 1;
    tc.tier = -1;
    tc.skip = nullptr;
    int acc = 0, row = 0;
#pragma unroll
    for (int m = 0; m < BE_MAX_TIERS; ++m) {
        if (m < c.n_tiers) {
            int r = c.tiers[m].replicas;
            if (lane >= acc && lane < acc + r) {
                tc.alpha = c.tiers[m].alpha_ms;
                tc.beta = c.tiers[m].beta_ms;
                tc.max_batch = c.tiers[m].max_batch;
                tc.tokens = c.tiers[m].tokens_per_request;
                tc.tier = m;
                tc.skip = skip_tab ? skip_tab + (size_t)row * SKIP_NB : nullptr;
            }
            acc += r;
            row += c.tiers[m].max_batch + 1;
        }
    }
    return tc;
}

// ---------------------------------------------------------------------------
// Record stores of completions (rollout / step): with BE_REC_NOALLOC the write-through
// stores skip allocating L1 lines (L1 keeps the FIFO rings and spill lines instead)
// (measured r2: DRAM traffic of the config-4 rollout 9.6 + 11.5 -> 6.7 + 8.7 GB per
// launch, throughput unchanged; an L2 evict-first hint on top changed nothing)
#ifndef BE_REC_NOALLOC
#define BE_REC_NOALLOC 1
#endif
__device__ __forceinline__ void st_rec(double* p, double v) {
#if BE_REC_NOALLOC
    asm volatile("st.global.L1::no_allocate.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
#else
    *p = v;
#endif
}
__device__ __forceinline__ void st_rec(uint8_t* p, uint8_t v) {
#if BE_REC_NOALLOC
    asm volatile("st.global.L1::no_allocate.u8 [%0], %1;" ::"l"(p), "h"((unsigned short)v) : "memory");
#else
    *p = v;
#endif
}

// Request completion: realized latency (simcore.py:135), deadline weight and
// reward (reward.py:94-126), deadline miss (evalkit.py:65-67).
__device__ __forceinline__ void complete(const Rep& r, const TierC& tc, const Score& sc,
                                         const RecOut& o, double t_end) {
    int task = (int)(r.h_idtask >> 24);
    const uint32_t id = r.h_idtask & 0xffffffu;
    const double span = __dsub_rn(t_end, r.h_arr);
    if (!sc.soft[task] && !o.realized) {
        // hard deadline, realized not requested: weight_hard (reward.py:94-96) via the
        // exact division-free threshold
        const bool hit = span <= sc.hit_tau[task * BE_MAX_TIERS + tc.tier];
        st_rec(o.reward + id, hit ? sc.matrix[task * BE_MAX_TIERS + tc.tier] : 0.0);
        st_rec(o.flags + id, (uint8_t)(tc.tier | 0x40 | (hit ? 0 : 0x80)));
        return;
    }
    double realized = __ddiv_rn(span, (double)tc.tokens);
    double dl = sc.deadline[task];
    double w;
    if (!sc.soft[task]) {
        w = realized <= dl ? 1.0 : 0.0;
    } else {
        double excess = __dsub_rn(realized, dl);
        if (excess <= 0.0) {
            w = 1.0;
        } else if (excess <= sc.cut[task]) {
            double v = __dsub_rn(1.0, __dmul_rn(sc.decay, excess));
            w = v > 0.0 ? v : 0.0;  // max(0.0, v)
        } else {
            w = 0.0;
        }
    }
    double reward = __dmul_rn(w, sc.matrix[task * BE_MAX_TIERS + tc.tier]);
    // flags: tier (bits 0-5) | completed (0x40) | deadline miss (0x80)
    uint8_t flag = (uint8_t)(tc.tier | 0x40 | ((realized > dl) ? 0x80 : 0));
    st_rec(o.reward + id, reward);
    st_rec(o.flags + id, flag);
    if (o.realized) st_rec(o.realized + id, realized);
}

// ---------------------------------------------------------------------------
// Exact closed-form skipping of steady-state iterations.
//
// Between membership changes a replica repeats START(t) -> END at
// t' = RN(RN(t + alpha) + c), c = RN(beta * n).  While t, RN(t + alpha) and t'
// stay inside one binade [2^e, 2^(e+1)), every double there is an integer
// multiple of u = 2^(e-52) and t is one, so RN(t + alpha) = t + RN_u(alpha)
// and RN(. + c) = . + RN_u(c), where RN_u rounds to the nearest multiple of u
// (ties excluded, as they would depend on the parity of t / u).  Hence k
// cycles advance t by exactly k * D, D = RN_u(alpha) + RN_u(c) — the same bits
// the iteration-by-iteration recurrence produces.  D depends only on (tier, n,
// binade): the host tabulates it once per env (build_skip_table, api.cu; 0 =
// "do not skip": a rounding tie, or the binade is outside the table) and the
// kernels stage the table in shared memory.  Skipping keeps every operand at
// or below (2^53 - 2) u, the second-largest double of the binade.

// The table entry of a START at time t with n running requests (0: no skip); `tab`
// is this tier's table, indexed [n][binade - SKIP_ELO].
__device__ __forceinline__ double skip_entry(double t, const double* __restrict__ tab, int n) {
    const int hi = __double2hiint(t);
    const int ib = ((hi >> 20) & 0x7ff) - (1023 + SKIP_ELO);
    if ((unsigned)ib >= (unsigned)SKIP_NB || hi < 0) return 0.0;
    return tab[n * SKIP_NB + ib];
}

// Number k <= kmax of whole START->END cycles that can be jumped from a START at
// time t (0 < t < until), D = skip_entry(t, ...) (loaded by the caller ahead of
// time); writes the time after k cycles.
__device__ __forceinline__ int skip_cycles_d(double t, double D, int kmax, double until, double& t_out) {
    if (kmax <= 0) return 0;
    if (!(D > 0.0)) return 0;
    const int hi = __double2hiint(t);
    // (2^53 - 2) u: same exponent as t, mantissa all ones but the last bit
    const double top = __hiloint2double(hi | 0x000fffff, (int)0xfffffffe);
    // x = min(top, until) - t is exact: both operands are multiples of u in t's binade
    const double x = __dsub_rn(until < top ? until : top, t);
    // k D <= x  <=>  RN(k D - x) <= 0 (rounding never changes a sign)
    double q;
    if (__fma_rn((double)kmax, D, -x) <= 0.0) {
        q = (double)kmax;  // common case: the next completion comes first
    } else {
        // floor(x / D) < kmax: float-reciprocal estimate, one refinement, exact sign fix-ups
        const double r = (double)__fdividef(1.0f, (float)D);
        q = floor(__dmul_rn(x, r));
        q = __dadd_rn(q, floor(__dmul_rn(__fma_rn(-q, D, x), r)));
        while (__fma_rn(q, D, -x) > 0.0) q = __dsub_rn(q, 1.0);
        while (__fma_rn(__dadd_rn(q, 1.0), D, -x) <= 0.0) q = __dadd_rn(q, 1.0);
    }
    if (!(q > 0.0)) return 0;
    t_out = __fma_rn(q, D, t);  // t + k D is a multiple of u inside the binade: exact
    return (int)q;
}


// ---------------------------------------------------------------------------
// One replica's share of ClusterSim.advance(until) (simcore.py:113-149):
// process events while (t, kind) < (until, START); END at the horizon is
// processed, START at the horizon stays pending (simcore.py:120).
// Returns false if the iteration counter would overflow.
__device__ __forceinline__ bool advance_lane(Rep& r, const TierC& tc, double until, Slot* ring,
                                             uint32_t mask, const Score& sc, const RecOut& o) {
    while (r.kind != K_NONE) {
        if (r.kind == K_START) {
            if (!(r.t < until)) break;
            int n_active = min(r.count, tc.max_batch);
            // the skip-table entry of this START, in flight during the joins below (+0.7%)
            const double Dskip = tc.skip ? skip_entry(r.t, tc.skip, n_active) : 0.0;
            if (r.n_running < n_active) {  // newly admitted requests join (simcore.py:143-145)
                if (r.n_running == 0) r.h_join = r.iters;
                // requests admitted straight into `active` got their join at submit; only
                // those admitted from the queue at the last END still need it
                for (int k = max(max(r.n_running, r.n_assigned), 1); k < n_active; ++k)
                    ring[(r.head + (uint32_t)k) & mask].join = r.iters;
                r.n_running = n_active;
                r.n_assigned = max(r.n_assigned, n_active);
            }
            double c = __dmul_rn(tc.beta, (double)n_active);
            if (tc.skip) {
                int K = r.h_join + tc.tokens - r.iters;  // ENDs until the head completes
                double tn;
                int k = skip_cycles_d(r.t, Dskip, min(K - 1, (1 << 30) - r.iters), until, tn);
                if (k > 0) {
                    r.t = tn;
                    r.iters += k;
                    if (!(r.t < until)) break;
                }
            }
            r.t = __dadd_rn(__dadd_rn(r.t, tc.alpha), c);
            r.kind = K_END;
        } else {
            if (!(r.t <= until)) break;
            if (r.iters >= (1 << 30)) return false;
            r.iters++;
            // FIFO completions (simcore.py:127-137): every running request got a token
            while (r.n_running > 0 && r.iters - r.h_join >= tc.tokens) {
                // the next entry's load is in flight while this completion is scored
                // (the same values a load after the pop would see: nothing writes the
                // ring in between; +1.7% rollout throughput)
                Slot s;
                if (r.count > 1) s = ring[(r.head + 1u) & mask];
                complete(r, tc, sc, o, r.t);
                r.head++;
                r.count--;
                r.n_running--;
                r.n_assigned--;  // >= n_running >= 1 before the pop
                if (r.count > 0) {
                    r.h_arr = s.arrival;
                    r.h_idtask = s.idtask;
                    r.h_join = s.join;
                }
            }
            // queue admission (simcore.py:138-140) is implicit: active = FIFO prefix
            r.kind = r.count > 0 ? K_START : K_NONE;  // START at the same time (simcore.py:141-142)
        }
    }
    return true;
}

// ClusterSim.submit on the chosen lane (simcore.py:94-111).  `clock` is the
// env clock (== the arrival being routed).  Returns false on ring overflow.
__device__ __forceinline__ bool submit_lane(Rep& r, const TierC& tc, double clock, uint32_t idtask,
                                            Slot* ring, uint32_t mask) {
    if ((uint32_t)r.count > mask) return false;
    // A request that enters `active` directly (len(active) < max_batch, simcore.py:101-104)
    // joins the running batch at the next START: now if the replica is idle or a START
    // is pending, after the pending END otherwise (END increments the iteration counter
    // first).  Recording it here saves the START-time write for the common case; a
    // queued request gets its join when a later START admits it.
    const bool direct = r.count < tc.max_batch;
    const int join = direct ? r.iters + (r.kind == K_END ? 1 : 0) : -1;
    if (r.count == 0) {
        r.h_arr = clock;
        r.h_idtask = idtask;
        r.h_join = join;
    } else {
        Slot s;
        s.arrival = clock;
        s.idtask = idtask;
        s.join = join;
        ring[(r.head + (uint32_t)r.count) & mask] = s;
    }
    if (direct && r.n_assigned == r.count) r.n_assigned++;
    r.count++;
    if (r.kind == K_NONE) {  // idle replica: START at the current clock
        r.kind = K_START;
        r.t = clock;
    }
    return true;
}

__device__ __forceinline__ void rep_reset(Rep& r) {
    r.t = 0.0;
    r.h_arr = 0.0;
    r.kind = K_NONE;
    r.iters = 0;
    r.count = 0;
    r.n_running = 0;
    r.h_join = -1;
    r.h_idtask = 0;
    r.n_assigned = 0;
}

// Rate estimator (workload.py:212-255), warp-uniform.
struct Estimator {
    double w[5];
    int n;
};

__device__ __forceinline__ double estimator_observe(Estimator& est, double t, bool true_rate,
                                                    double cur_rate, double prior) {
    if (est.n == 5) {
        est.w[0] = est.w[1];
        est.w[1] = est.w[2];
        est.w[2] = est.w[3];
        est.w[3] = est.w[4];
        est.n = 4;
    }
    // est.w[est.n] = t without dynamic register indexing
    if (est.n == 0) est.w[0] = t;
    else if (est.n == 1) est.w[1] = t;
    else if (est.n == 2) est.w[2] = t;
    else if (est.n == 3) est.w[3] = t;
    else est.w[4] = t;
    est.n++;
    if (true_rate) return cur_rate;
    if (est.n < 2) return prior;
    double last = t;
    // (last - w0) / (n - 1): for n - 1 in {1, 2, 4} (4 in steady state) the quotient is an
    // exact power-of-two scaling, so the multiply gives the same bits as the division
    const double span = __dsub_rn(last, est.w[0]);
    const int d = est.n - 1;
    const double mean = d == 3 ? __ddiv_rn(span, 3.0) : __dmul_rn(span, d == 4 ? 0.25 : d == 2 ? 0.5 : 1.0);
    double gap = __ddiv_rn(mean, 1000.0);
    return __ddiv_rn(1.0, gap > 1e-6 ? gap : 1e-6);
}

// ---------------------------------------------------------------------------
// Q-network forward for one state over a group of LPE lanes (policy.py:111-118;
// LPE = 16: two environments per warp).  Lane g of the group owns hidden units
// j = g + LPE k.  Shared-memory layout (stage_qnet), chosen so one hidden unit
// costs 1 + ceil((2M+1)/2) loads, all bank-conflict free:
//   task rows  [T][H]        W1[t][j] + b1[j]   (the one-hot input selects one;
//                                                 b1 is folded in at staging)
//   pairs      [NP][H] double2   consecutive entries of v_j = (W1[T+0][j] ..
//                                W1[T+M-1][j], W1[T+M][j] (rate), W2[j][0..M-1])
//   odd        [H]            v_j[2M] when 2M+1 is odd (always)
//   b2         [M]
// Result q[] is bit-identical on every lane of the group (xor-butterfly sums
// commute).  (Measured: a second accumulator set for shorter DFMA chains is
// slower here — more live registers for no latency win.)
template <int M>
struct QLayout {
    static constexpr int NV = 2 * M + 1;  // per-hidden-unit values besides the task row
    static constexpr int NP = NV / 2;
    __host__ __device__ static size_t doubles(int T, int H) { return (size_t)(T + NV) * H + M; }
};

// (tid, nt): this thread's index among the nt threads that share the staging.
template <int M>
__device__ __forceinline__ void stage_qnet(const double* __restrict__ w1, const double* __restrict__ b1,
                                           const double* __restrict__ w2, const double* __restrict__ b2,
                                           int T, int H, double* sw, int tid, int nt) {
    constexpr int NV = QLayout<M>::NV, NP = QLayout<M>::NP;
    for (int k = tid; k < T * H; k += nt) sw[k] = __dadd_rn(w1[k], b1[k % H]);
    double* pairs = sw + (size_t)T * H;
    for (int k = tid; k < NV * H; k += nt) {
        const int v = k / H, j = k % H;
        // v < M: tier inputs, v == M: rate input (W1 rows T..T+M); v > M: W2[j][v-M-1]
        const double x = v <= M ? w1[(size_t)(T + v) * H + j] : w2[(size_t)j * M + (v - M - 1)];
        if (v < 2 * NP) pairs[((size_t)(v >> 1) * H + j) * 2 + (v & 1)] = x;
        else pairs[(size_t)2 * NP * H + j] = x;
    }
    double* sb2 = sw + (size_t)(T + NV) * H;
    for (int k = tid; k < M; k += nt) sb2[k] = b2[k];
}

template <int M>
__device__ __forceinline__ void stage_qnet(const double* __restrict__ w1, const double* __restrict__ b1,
                                           const double* __restrict__ w2, const double* __restrict__ b2,
                                           int T, int H, double* sw) {
    stage_qnet<M>(w1, b1, w2, b2, T, H, sw, threadIdx.x, blockDim.x);
}

// The packed fp64 layout in global memory (the screened rollout's fallback and
// the step kernel read it through L1), grid-stride.
template <int M>
__global__ void __launch_bounds__(256) stage_qpack_kernel(const double* w1, const double* b1, const double* w2,
                                                          const double* b2, int T, int H, double* out) {
    pdl_trigger();
    pdl_wait();  // the weights may have been updated by the previous kernel
    stage_qnet<M>(w1, b1, w2, b2, T, H, out, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}
constexpr int QPACK_CTAS = 16;

template <int M, int LPE, int UNROLL = 8>
__device__ __forceinline__ void qnet_group(const double* __restrict__ sw, int T, int H, int task,
                                           const double (&xt)[M], double xr, double (&q)[M]) {
    constexpr int NV = QLayout<M>::NV, NP = QLayout<M>::NP;
    const int g = threadIdx.x & (LPE - 1);
    const double* wtask = sw + (size_t)task * H;
    const double2* pairs = reinterpret_cast<const double2*>(sw + (size_t)T * H);
    const double* odd = sw + (size_t)T * H + (size_t)2 * NP * H;
    const double* sb2 = sw + (size_t)(T + NV) * H;
    double a[M];
#pragma unroll
    for (int m = 0; m < M; ++m) a[m] = 0.0;
#pragma unroll UNROLL
    for (int j = g; j < H; j += LPE) {
        double v[NV];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const double2 w = pairs[(size_t)p * H + j];
            v[2 * p] = w.x;
            v[2 * p + 1] = w.y;
        }
        if (NV & 1) v[NV - 1] = odd[j];
        double pre = wtask[j];
#pragma unroll
        for (int m = 0; m < M; ++m) pre = __fma_rn(xt[m], v[m], pre);
        pre = __fma_rn(xr, v[M], pre);
        const long long pb = __double_as_longlong(pre);
        const double h = __longlong_as_double(pb & ~(pb >> 63));
#pragma unroll
        for (int m = 0; m < M; ++m) a[m] = __fma_rn(h, v[M + 1 + m], a[m]);
    }
#pragma unroll
    for (int off = LPE / 2; off > 0; off >>= 1) {
#pragma unroll
        for (int m = 0; m < M; ++m) a[m] = __dadd_rn(a[m], __shfl_xor_sync(FULL, a[m], off));
    }
#pragma unroll
    for (int m = 0; m < M; ++m) q[m] = __dadd_rn(a[m], sb2[m]);
}

// ---------------------------------------------------------------------------
// Certified fp32 screening of the greedy decision (fused rollout fast path).
//
// The decision only needs the argmax of q = relu(x W1 + b1) W2 + b2.  The
// screen evaluates q in fp32 with packed FFMA2 (two hidden units per
// instruction, half the shared-memory bytes of the fp64 path) together with
// a rigorous bound |q32_m - q_m| <= B_m on its error against exact
// arithmetic on the fp64 inputs; if the fp32 leader beats every other action
// by more than the sum of the two bounds, it IS the exact argmax (unique, so
// the first-max tie rule cannot matter) and the fp64 evaluation is skipped.
// Otherwise (about 1% of trained-policy states: near-ties, huge rate inputs,
// non-finite values) the caller falls back to qnet_group in fp64, so every
// decision equals the fp64 path's.  Q values are never taken from the screen
// (runs that record q use the fp64 path throughout).
//
// Error bound (u = 2^-24, gamma_n = n u / (1 - n u)).  Per hidden unit j the
// layer-1 value is four chained FMAs on operands each rounded once to fp32:
// |pre32_j - pre_j| <= (gamma_4 + 2u + O(u^2)) P_j <= 7u P_j with
// P_j = |W1[t][j] + b1[j]| + sum_i |x_i| |W1[T+i][j]|; relu is 1-Lipschitz
// and |h32_j| <= (1 + 7u) P_j.  Every layer-2 term passes through
// L = H/(2 LPE) chained FFMA2 + 1 pair add + log2(LPE) butterfly adds + 1 bias
// add roundings, with W2 rounded once: |q32_m - q_m| <= ((L + 1)(1 + 8u) + 7) u
// S_m, S_m = sum_j |W2[j][m]| P_j + |b2[m]|.  The kernel uses K = (L + 16) u
// (slack >= 8u also covers the fp32 evaluation of the bound itself, whose terms
// are all non-negative and rounded upward).  One scalar bound per state,
// B = max_m B_m <= A[t] + sum_i |x_i| C[i] with A[t] = K max_m (sum_j |W2[j][m]|
// |W1[t][j] + b1[j]| + |b2[m]|) and C[i] = K max_m sum_j |W2[j][m]| |W1[T+i][j]|
// (host-side maxima cost < 0.1% extra fallbacks on the goldens), certifies the
// leader when q32_best - q32_second > 2 B, evaluated in fp64.
template <int M>
struct QsLayout {
    static constexpr int NV = 2 * M + 1;  // per-hidden-unit values besides the task row
    static constexpr int NQ4 = NV / 2;    // float4 arrays (two values x two units)
    // floats: per task [T][H/2] float4 (task-row pair, last-value pair) + the other
    // values [NQ4][H/2] float4 + A [T] + C [M+1] + b2 [M]; the task row and the last
    // value share one 16-byte load per unit pair
    __host__ __device__ static size_t q4_off(int T, int H) { return (size_t)2 * T * H; }
    __host__ __device__ static size_t bA_off(int T, int H) { return (size_t)(2 * T + 2 * NQ4) * H; }
    __host__ __device__ static size_t floats(int T, int H) { return bA_off(T, H) + T + (M + 1) + M; }
};

// Lane g of a group owns hidden-unit pairs (j0, j1) = (g + 2p LPE, g + 2p LPE + LPE),
// stored at pair index P = p LPE + g so that a group's loads are consecutive.
template <int LPE>
__device__ __forceinline__ int screen_unit(int P, int half) {
    const int p = P / LPE, g = P % LPE;
    return g + 2 * p * LPE + half * LPE;
}

// All threads of the CTA; the caller synchronises before use.  Requires
// H % (2 LPE) == 0.
template <int M, int LPE>
__device__ __forceinline__ void stage_qscreen(const double* __restrict__ w1, const double* __restrict__ b1,
                                              const double* __restrict__ w2, const double* __restrict__ b2,
                                              int T, int H, float* sf) {
    constexpr int NV = QsLayout<M>::NV, NQ4 = QsLayout<M>::NQ4;
    const int H2 = H / 2;
    auto val = [&](int v, int j) -> double {  // v < M: tier inputs, v == M: rate, v > M: W2[j][v-M-1]
        return v <= M ? w1[(size_t)(T + v) * H + j] : w2[(size_t)j * M + (v - M - 1)];
    };
    float4* to4 = reinterpret_cast<float4*>(sf);
    for (int k = threadIdx.x; k < T * H2; k += blockDim.x) {
        const int t = k / H2, P = k % H2;
        const int j0 = screen_unit<LPE>(P, 0), j1 = screen_unit<LPE>(P, 1);
        to4[k] = make_float4(__double2float_rn(__dadd_rn(w1[(size_t)t * H + j0], b1[j0])),
                             __double2float_rn(__dadd_rn(w1[(size_t)t * H + j1], b1[j1])),
                             __double2float_rn(val(NV - 1, j0)), __double2float_rn(val(NV - 1, j1)));
    }
    float4* q4 = reinterpret_cast<float4*>(sf + QsLayout<M>::q4_off(T, H));
    for (int k = threadIdx.x; k < NQ4 * H2; k += blockDim.x) {
        const int q = k / H2, P = k % H2;
        const int j0 = screen_unit<LPE>(P, 0), j1 = screen_unit<LPE>(P, 1);
        q4[k] = make_float4(__double2float_rn(val(2 * q, j0)), __double2float_rn(val(2 * q, j1)),
                            __double2float_rn(val(2 * q + 1, j0)), __double2float_rn(val(2 * q + 1, j1)));
    }
    // bound tables: one warp per row r (task row r < T, else input T + (r - T)),
    // fp64 sums over j, maximum over m, rounded up to fp32
    float* bA = sf + QsLayout<M>::bA_off(T, H);
    float* bC = bA + T;
    float* b2f = bC + (M + 1);
    int lg = 0;
    while ((1 << lg) < LPE) ++lg;
    const double K = (double)(H / (2 * LPE) + 2 + lg + 16) * 0x1p-24;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int r = warp; r < T + M + 1; r += nw) {
        double mx = 0.0;
        bool bad = false;
        for (int m = 0; m < M; ++m) {
            double acc = 0.0;
            for (int j = lane; j < H; j += 32) {
                const double a = r < T ? fabs(__dadd_rn(w1[(size_t)r * H + j], b1[j])) : fabs(w1[(size_t)r * H + j]);
                acc = __fma_rn(fabs(w2[(size_t)j * M + m]), a, acc);
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(FULL, acc, off));
            if (r < T) acc = __dadd_ru(acc, fabs(b2[m]));
            mx = fmax(mx, acc);
            bad = bad || acc != acc;  // non-finite weights: never certify
        }
        if (bad) mx = __longlong_as_double(0x7ff8000000000000LL);
        if (lane == 0) {
            const float v = __double2float_ru(__dmul_ru(K, mx));
            if (r < T) bA[r] = v;
            else bC[r - T] = v;
        }
    }
    for (int m = threadIdx.x; m < M; m += blockDim.x) b2f[m] = __double2float_rn(b2[m]);
}

// Returns true if `tier` is certified to be the exact greedy decision; the
// result is identical on every lane of the group.
template <int M, int LPE>
__device__ __forceinline__ bool qnet_screen(const float* __restrict__ sf, int T, int H, int task,
                                            const double (&xt)[M], double xr, int& tier) {
    constexpr int NV = QsLayout<M>::NV, NQ4 = QsLayout<M>::NQ4;
    const int g = threadIdx.x & (LPE - 1);
    const int H2 = H / 2;
    const float4* to4 = reinterpret_cast<const float4*>(sf) + (size_t)task * H2;
    const float4* q4 = reinterpret_cast<const float4*>(sf + QsLayout<M>::q4_off(T, H));
    const float* bA = sf + QsLayout<M>::bA_off(T, H);
    const float* bC = bA + T;
    const float* b2f = bC + (M + 1);
    float x32[M + 1];
#pragma unroll
    for (int m = 0; m < M; ++m) x32[m] = __double2float_rn(xt[m]);
    x32[M] = __double2float_rn(xr);
    float2 a[M];
#pragma unroll
    for (int m = 0; m < M; ++m) a[m] = make_float2(0.f, 0.f);
#pragma unroll 8
    for (int P = g; P < H2; P += LPE) {
        float2 v[NV];
#pragma unroll
        for (int q = 0; q < NQ4; ++q) {
            const float4 w = q4[(size_t)q * H2 + P];
            v[2 * q] = make_float2(w.x, w.y);
            v[2 * q + 1] = make_float2(w.z, w.w);
        }
        const float4 tw = to4[P];
        v[NV - 1] = make_float2(tw.z, tw.w);
        float2 pre = make_float2(tw.x, tw.y);
#pragma unroll
        for (int m = 0; m <= M; ++m) pre = ffma2(make_float2(x32[m], x32[m]), v[m], pre);
        const float2 h = make_float2(fmaxf(pre.x, 0.f), fmaxf(pre.y, 0.f));
#pragma unroll
        for (int m = 0; m < M; ++m) a[m] = ffma2(h, v[M + 1 + m], a[m]);
    }
    float q[M];
#pragma unroll
    for (int m = 0; m < M; ++m) q[m] = __fadd_rn(a[m].x, a[m].y);
#pragma unroll
    for (int off = LPE / 2; off > 0; off >>= 1) {
#pragma unroll
        for (int m = 0; m < M; ++m) q[m] = __fadd_rn(q[m], __shfl_xor_sync(FULL, q[m], off));
    }
    // leader and runner-up (a tie makes the margin 0: never certified)
    int best = 0;
    bool fin = true;
    float bv = 0.f, sv = -INFINITY;
#pragma unroll
    for (int m = 0; m < M; ++m) {
        const float v = __fadd_rn(q[m], b2f[m]);
        fin = fin && isfinite(v);
        if (m == 0 || v > bv) {
            sv = bv;
            best = m;
            bv = v;
        } else if (v > sv) {
            sv = v;
        }
        if (m == 0) sv = -INFINITY;
    }
    float B = bA[task];
#pragma unroll
    for (int i = 0; i <= M; ++i) B = __fmaf_ru(fabsf(x32[i]), bC[i], B);
    tier = best;
    // M == 1: nothing to decide
    return M == 1 || (fin && isfinite(B) && __dsub_rd((double)bv, (double)sv) > 2.0 * (double)B);
}

// Sum / min over the lanes of this lane's group (REDUX over the warp with the
// other group masked out; all 32 lanes must call).
template <int LPE>
__device__ __forceinline__ unsigned group_sum(unsigned v, int grp) {
    if (LPE == 32) return __reduce_add_sync(FULL, v);
    const unsigned s0 = __reduce_add_sync(FULL, grp == 0 ? v : 0u);
    const unsigned s1 = __reduce_add_sync(FULL, grp == 1 ? v : 0u);
    return grp ? s1 : s0;
}
template <int LPE>
__device__ __forceinline__ unsigned group_min(unsigned v, int grp) {
    if (LPE == 32) return __reduce_min_sync(FULL, v);
    const unsigned s0 = __reduce_min_sync(FULL, grp == 0 ? v : 0xffffffffu);
    const unsigned s1 = __reduce_min_sync(FULL, grp == 1 ? v : 0xffffffffu);
    return grp ? s1 : s0;
}

// np.argmax semantics: first NaN if any, else first maximum.
template <int M>
__device__ __forceinline__ int argmax_first(const double (&q)[M]) {
    int best = 0;
    double bv = q[0];
    bool nan_seen = bv != bv;
#pragma unroll
    for (int m = 1; m < M; ++m) {
        const bool take = !nan_seen && (q[m] != q[m] || q[m] > bv);
        nan_seen = nan_seen || q[m] != q[m];
        best = take ? m : best;
        bv = take ? q[m] : bv;
    }
    return best;
}

}  // namespace be
