// step.cu — step-synchronous environment API: be_env_reset / be_env_step /
// be_env_drain.  Same device building blocks as the fused rollout
// (be_env.cuh); the per-replica registers are loaded from and stored back to
// HBM around every step, so the host can interleave its own logic (the
// training loop, a custom router) between steps.  One or two envs per warp.
// Also the training iteration's env step (be_train_iteration): arrivals, step and
// replay commit in one launch (env_step_commit_kernel), fp64 or tcgen05 decisions.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "be_env.cuh"
#include "be_internal.h"
#include "be_philox.cuh"
#include "be_route_tc.cuh"
#include "be_workload.cuh"

namespace be {

// Development probe points (compiled out unless BE_PROBE_T is defined): thread 0 of
// CTA b records %globaltimer into be_probe_t[b][k]; read back with be_debug_probe.
#ifdef BE_PROBE_T
__device__ unsigned long long be_probe_t[1024 * 16];
#define BE_PROBE(k)                                                                   \
    if (threadIdx.x == 0 && blockIdx.x < 1024) {                                      \
        unsigned long long t_;                                                        \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                        \
        be_probe_t[blockIdx.x * 16 + (k)] = t_;                                       \
    }
#else
#define BE_PROBE(k)
#endif

struct EnvState {
    double w[5];
    int32_t n;
    int32_t _pad;
    int64_t next_id;  // request id of the next submitted request
};

size_t env_state_bytes_per_env(int R) { return (size_t)R * sizeof(Rep) + sizeof(EnvState); }

static __device__ __forceinline__ Rep* reps_of(void* base, int e, int R) {
    return reinterpret_cast<Rep*>(base) + (size_t)e * R;
}
static __device__ __forceinline__ EnvState* state_of(void* base, int e, int E, int R) {
    return reinterpret_cast<EnvState*>(reinterpret_cast<Rep*>(base) + (size_t)E * R) + e;
}

__global__ void env_reset_kernel(void* base, int E, int R, const uint8_t* mask) {
    int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (gw >= E) return;
    if (mask && !mask[gw]) return;
    if (lane < R) {
        Rep r;
        rep_reset(r);
        r.head = 0;
        reps_of(base, gw, R)[lane] = r;
    }
    if (lane == 0) {
        EnvState s;
        for (int k = 0; k < 5; ++k) s.w[k] = 0.0;
        s.n = 0;
        s._pad = 0;
        s.next_id = 0;
        *state_of(base, gw, E, R) = s;
    }
}

struct StepParams {
    be_cfg cfg;
    ScoreAux aux;
    int32_t E, R, cap_log2;
    void* state;
    Slot* rings;
    const double* arrival;
    const uint8_t* task;
    const double* true_rate;
    const uint8_t* forced;
    int32_t static_tier;
    int32_t H;
    const double *w1, *b1, *w2, *b2;
    double epsilon;
    uint64_t seed, counter;
    int64_t rec_ld;
    be_records rec;
    int32_t* obs_out;
    double* rate_out;
    uint8_t* action_out;
    double* q_out;
    double* x_out;
    int32_t* status;
    int32_t drain;
    // split step (a router between): 1 = observe (advance, estimator, observe, encode
    // into x_out; no decision, no submit), 2 = submit the decision read from action_out
    int32_t phase;
    int32_t new_segment;      // drain + reset replicas and estimator (be_env_new_segment)
    const uint8_t* seg_mask;  // drain / new_segment: only envs with mask[e] != 0 (NULL = all)
    const double* skip;  // skip table (global), NULL = skipping off
    // device-step mode (be_train_iteration): epsilon, Philox counter and the
    // pending slot of x_out / action_out come from the iteration index *iter_dev
    const int64_t* iter_dev;
    double eps_start, eps_end;
    int64_t eps_decay;
    int32_t pending_P;
    const double* qpack;  // packed fp64 weights (QLayout) in global memory, read through L1
    // decision on the tensor cores (env_step_commit_kernel<M, true>): the router's packed image
    // (TcLayout, rebuilt by prep_kernel every iteration) and the TMEM columns to allocate
    const float* tc_img;
    int32_t tc_ncols;
    // training commits (be_train_iteration): per env {lowest, highest request id completed
    // in this step's advance, oldest request still in flight after the submit} (nullable)
    int64_t* crange;
    // fused replay commit (env_step_commit_kernel; fuse_commit = 1)
    StepCommitArgs cm;
    int32_t fuse_commit;
    // env_step_commit_kernel generates the iteration's arrivals itself (TrainingWorkload)
    int32_t gen_workload;
    WorkloadArgs wl;
};

// dynamic shared memory of the step kernels starts with the reward tables (Score)
__host__ __device__ constexpr size_t step_score_bytes() { return (sizeof(Score) + 15) & ~size_t(15); }

// Shared state of one env_step_commit_kernel CTA round.
constexpr int SC_ENVS = 16;  // envs per CTA round (8 warps x 2)
constexpr int SC_CW = 2;    // doubles per load batch of a transition copy (register-bound: 2 spills least)
constexpr int SC_MINB = 2;  // 2 CTAs per SM: one resident wave of 296 CTAs (4736 envs)
constexpr int SC_QU = 4;    // Q-forward unroll of the fused step (weights in shared memory: 2 / 4 / 8 measure alike)
constexpr int SC_LIST = 4096;  // block-wide transition list (ring-slot order); overflow: per env
struct CommitShared {
    long long cursor, agg, excl;
    int vb;                  // this round's virtual block (ticket mode)
    int cnt[SC_ENVS];        // commit counts of the block's envs
    unsigned long long ep;   // scan epoch << 40
    unsigned long long wmax;
    // the block's committable transitions in ring-slot order (env order, then request-id
    // order): pending slot and env of entry i, whose ring slot is the block's base + i
    uint32_t sj[SC_LIST];
    uint8_t le[SC_LIST];
};

// What one env's step hands the fused commit: the id range this step's advance
// completed (every request in it is committable now: its next state x_{j+1}
// exists) and the oldest request still in flight after the submit.  The step also
// publishes the block's commit count as soon as the advance is done (commit_publish),
// so the cross-block scan overlaps the Q forward and the submit.
struct StepOut {
    int64_t jlo, jhi, oldest;
    CommitShared* cs;
    int vb, le;
    bool live;
    bool has_wl;  // arrival / task / true rate below instead of p.arrival / p.task / p.true_rate
    int task;
    double U, rate;
};

// An env's committable transitions into the block list: its completed id range
// [jlo, jlo + L) is scanned 256 ids per pass (16 per lane, independent flag loads);
// the ready ones (reward written: flag 0x40) take list entries base, base + 1, ... in
// id order.  Entries past the list capacity are left to commit_copy_overflow.  Group-wide.
__device__ __forceinline__ void commit_list(const StepParams& p, CommitShared& cs, int e, int le, int P, int64_t jlo,
                                            int64_t L, long long base, int gl, unsigned gmask) {
    const int cap = p.cm.list_cap;
    const int64_t r0 = jlo % P;
    for (int64_t b0 = 0; b0 < L; b0 += 256) {
        const int64_t sbase = (r0 + b0 + gl * 16) % P;
        unsigned bits = 0;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            int64_t sj = sbase + k;
            if (sj >= P) sj = P >= 16 ? sj - P : sj % P;
            if (b0 + gl * 16 + k < L && (p.rec.flags[(int64_t)e * P + sj] & 0x40)) bits |= 1u << k;
        }
        const int cnt = __popc(bits);
        int inc = cnt;
#pragma unroll
        for (int off = 1; off < 16; off <<= 1) {
            const int v = __shfl_up_sync(gmask, inc, off, 16);
            if (gl >= off) inc += v;
        }
        long long r = base + inc - cnt;
        while (bits) {
            int64_t sj = sbase + __ffs(bits) - 1;
            if (sj >= P) sj = P >= 16 ? sj - P : sj % P;
            if (r < cap) {
                cs.sj[r] = (uint32_t)sj;
                cs.le[r] = (uint8_t)le;
            }
            ++r;
            bits &= bits - 1;
        }
        base += __shfl_sync(gmask, inc, 15, 16);
    }
}

// One transition (x_j, a_j, r_j, x_{j+1}) of env e, pending slot sj, into ring slot
// `slot` (ReplayBuffer.push, trainer.py:123-133): every load issued before any store.
template <int CW>
__device__ __forceinline__ void commit_copy(const StepParams& p, const StepCommitArgs& c, int e, int D, int P,
                                            int64_t sj, int64_t slot) {
    const int64_t sj1 = sj + 1 == P ? 0 : sj + 1;
    const double* pa = p.x_out + (sj * p.E + e) * D;
    const double* pb = p.x_out + (sj1 * p.E + e) * D;
    const uint8_t a = p.action_out[sj * p.E + e];
    const double r = p.rec.reward[(int64_t)e * P + sj];
    for (int d0 = 0; d0 < D; d0 += CW) {
        double xa[CW], xb[CW];
#pragma unroll
        for (int k = 0; k < CW; ++k)
            if (d0 + k < D) {
                xa[k] = pa[d0 + k];
                xb[k] = pb[d0 + k];
            }
#pragma unroll
        for (int k = 0; k < CW; ++k)
            if (d0 + k < D) {
                c.rs[slot * D + d0 + k] = xa[k];
                c.rs2[slot * D + d0 + k] = xb[k];
            }
    }
    c.ra[slot] = a;
    c.rr[slot] = r;
    c.rc[slot] = 1.0;
    p.rec.flags[(int64_t)e * P + sj] = 0x20;
}

// The block list overflowed (more transitions in one block and step than its capacity):
// the owning env group rescans its range and copies its entries at list index >= cap.
__device__ __forceinline__ void commit_copy_overflow(const StepParams& p, const StepCommitArgs& c, int e, int D, int P,
                                                     int64_t jlo, int64_t L, long long base, int64_t s0, int gl,
                                                     unsigned gmask) {
    const int64_t r0 = jlo % P;
    for (int64_t b0 = 0; b0 < L; b0 += 16) {
        int64_t sj = (r0 + b0 + gl) % P;
        const bool ready = b0 + gl < L && (p.rec.flags[(int64_t)e * P + sj] & 0x40);
        const unsigned rb = __ballot_sync(gmask, ready);
        const long long idx = base + __popc(rb & ((1u << (threadIdx.x & 31)) - 1u));
        if (ready && idx >= p.cm.list_cap) {
            int64_t slot = s0 + idx;
            while (slot >= c.capacity) slot -= c.capacity;
            commit_copy<4>(p, c, e, D, P, sj, slot);
        }
        base += __popc(rb);
    }
}


// scan words: epoch << 40 | flag << 38 | value (flag 1 = block aggregate, 2 = inclusive prefix)
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* a) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
    return v;
}
// release: this thread's earlier reads of the ring cursor / scan epoch are ordered
// before the publication the last block waits for before it changes them
__device__ __forceinline__ void st_release_u64(unsigned long long* a, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}

// Block-wide (every thread of the CTA calls it once per round): the counts of the
// block's 16 envs into shared memory, and their sum published to the look-back array
// (block 0: directly as its inclusive prefix).
__device__ __forceinline__ void commit_publish(const StepParams& p, const StepOut& so, int count) {
    CommitShared& cs = *so.cs;
    if ((threadIdx.x & 15) == 0) cs.cnt[so.le] = so.live ? count : 0;
    __syncthreads();
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const long long own = lane < SC_ENVS ? cs.cnt[lane] : 0;
        long long inc = own;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const long long v = __shfl_up_sync(FULL, inc, off);
            if (lane >= off) inc += v;
        }
        const long long agg = __shfl_sync(FULL, inc, 31);
        if (lane == 0) {
            cs.agg = agg;
            st_release_u64(&p.cm.scan[so.vb], cs.ep | ((so.vb == 0 ? 2ull : 1ull) << 38) | (unsigned long long)agg);
        }
    }
}

// request id of pending slot s (= id mod P) among the ids <= t
__device__ __forceinline__ int64_t id_of_slot(int64_t t, uint32_t s, int32_t P) {
    int64_t d = t % P - (int64_t)s;
    if (d < 0) d += P;
    return t - d;
}
template <int LPE>
__device__ __forceinline__ int64_t group_min64(int64_t v) {
#pragma unroll
    for (int off = LPE / 2; off > 0; off >>= 1) {
        const int64_t o = __shfl_xor_sync(FULL, v, off);
        v = o < v ? o : v;
    }
    return v;
}
template <int LPE>
__device__ __forceinline__ int64_t group_max64(int64_t v) {
#pragma unroll
    for (int off = LPE / 2; off > 0; off >>= 1) {
        const int64_t o = __shfl_xor_sync(FULL, v, off);
        v = o > v ? o : v;
    }
    return v;
}

// Per-CTA tensor-core decision context of env_step_commit_kernel<M, true> (shared memory + TMEM).
struct TcStepCtx {
    const float* img;  // TcLayout image in shared memory
    float* Ah;         // A operand, tf32 hi: [128 rows][TC_K] UMMA K-major (rows >= 16 stay 0)
    float* Al;         // tf32 lo
    float2* part;      // [2 column halves][16 rows][2 sets][TC_MP] layer-2 partial sums
    uint64_t* bar;     // MMA completion
    uint64_t* img_bar; // the image's bulk copy (waited for once, before the first MMA)
    uint32_t tmem;
    uint32_t phase;
    bool img_ready;
};

template <int M, int LPE, bool TCQ = false, int QU = 8>
__device__ __forceinline__ void step_env(const StepParams& p, int e, bool live, const Score& sc, const double* sw,
                                         bool policy, int T, int H, int D, TcStepCtx* tcx = nullptr,
                                         StepOut* so = nullptr);

// LPE lanes per env: 16 (two envs per warp) when the cluster has <= 16 replicas and
// the encoded state fits 16 lanes, else 32
template <int M, int LPE>
__global__ void __launch_bounds__(256) env_step_kernel(const StepParams p) {
    pdl_wait();  // the previous kernel has completed and its writes are visible
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Score& sc = *reinterpret_cast<Score*>(smem_raw);
    const int T = p.cfg.n_tasks;
    const int H = p.H, D = T + M + 1;
    const bool policy = !p.drain && p.phase == 0 && p.forced == nullptr && p.static_tier < 0;
    if (threadIdx.x < 32) load_score(sc, p.cfg, p.aux);
    __syncthreads();
    // persistent grid (one wave): the weights are staged once per CTA, then every
    // warp steps envs warp_id, warp_id + n_warps, ...
    constexpr int G = 32 / LPE;  // envs per warp
    const int n_warps = (gridDim.x * blockDim.x) >> 5;
    const int grp = (threadIdx.x & 31) / LPE;
    for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w * G < p.E; w += n_warps) {
        const int e = w * G + grp;
        step_env<M, LPE>(p, e < p.E ? e : p.E - 1, e < p.E, sc, p.qpack, policy, T, H, D);
    }
    pdl_trigger();  // this CTA is done: the next kernel may start filling the SM
}

// Shared-memory layout of the tensor-core step kernels: Score, the packed router image,
// the A operand (hi, lo), layer-2 partial sums, mbarriers.
struct TcStepSmem {
    size_t img, ah, al, part, bars, bytes;
    __host__ __device__ static size_t up(size_t x, size_t a) { return (x + a - 1) / a * a; }
    __host__ __device__ explicit TcStepSmem(int H) {
        img = up(sizeof(Score), 128);
        ah = up(img + (size_t)TcLayout{H}.bytes(), 128);
        al = ah + sizeof(float) * 128 * TC_K;
        part = al + sizeof(float) * 128 * TC_K;
        bars = up(part + sizeof(float2) * 2 * 16 * 2 * TC_MP, 16);
        bytes = bars + 2 * sizeof(uint64_t) + 16;
    }
};

// The training iteration's env step (be_train_iteration; TCQ: the greedy decision on
// the tensor cores, tc_decide, else the fp64 group forward) with the
// arrivals and the replay commit fused in — one launch where the reference runs
// TrainingWorkload.next_arrival, ClusterSim.advance / observe / submit, select_action and
// ReplayBuffer.resolve_* / push per env (trainer.py:374-395, :143-156).  Each CTA
// round steps 16 envs (two per warp):
//   * every lane of an env's group draws the env's next arrival (one lane stores the
//     workload state), then the step runs (step_env);
//   * every request the advance completed is committable at once (its reward was just
//     written, its next state x_{j+1} exists: j <= it - 1), so an env's commit count is
//     the number of FIFO entries its replicas popped; right after the advance the block
//     publishes its total (commit_publish), so the cross-block scan — decoupled
//     look-back over virtual blocks (round x grid + CTA; the grid is one resident wave,
//     so every predecessor is running or done) — overlaps the Q forward and the submit;
//   * each env lists its committable pending slots in shared memory (request-id order,
//     after the block's earlier envs), then every thread copies one transition: ring
//     slot = the block's prefix + list index — commit_fused_kernel's slots (env-id
//     order, request-id order within an env), so the host-driven loop and this one
//     fill the ring identically.
template <int M, bool TCQ>
__global__ void __launch_bounds__(256, SC_MINB) env_step_commit_kernel(const StepParams p) {
    pdl_wait();  // the previous kernel has completed and its writes are visible
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    Score& sc = *reinterpret_cast<Score*>(smem_raw);
    __shared__ CommitShared cs;
    // TCQ: one TMEM allocation (H columns; two CTAs per SM) and one bulk copy of the
    // packed router image per CTA, for all rounds
    TcStepCtx cx;
    uint64_t* bars = nullptr;
    if constexpr (TCQ) {
        const TcStepSmem S(p.H);
        cx.img = reinterpret_cast<const float*>(smem_raw + S.img);
        cx.Ah = reinterpret_cast<float*>(smem_raw + S.ah);
        cx.Al = reinterpret_cast<float*>(smem_raw + S.al);
        cx.part = reinterpret_cast<float2*>(smem_raw + S.part);
        bars = reinterpret_cast<uint64_t*>(smem_raw + S.bars);
        cx.bar = &bars[1];
        cx.img_bar = &bars[0];
        cx.phase = 0;
        cx.img_ready = false;
        for (int k = threadIdx.x; k < 2 * 128 * TC_K; k += blockDim.x) cx.Ah[k] = 0.f;  // rows >= 16 stay 0
        if (threadIdx.x == 0) {
            tc::mbar_init(&bars[0], 1);
            tc::mbar_init(&bars[1], 1);
            tc::fence_mbar_init();
        }
        if ((threadIdx.x >> 5) == 0) tc::tmem_alloc(reinterpret_cast<uint32_t*>(bars + 2), (uint32_t)p.tc_ncols);
        tc::fence_before_sync();
    }
    const StepCommitArgs& c = p.cm;
    const int T = p.cfg.n_tasks, H = p.H, D = T + M + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, grp = lane >> 4, gl = lane & 15;
    const unsigned gmask = 0xffffu << (grp * 16);
    if (threadIdx.x == 0) {
        // cursor and scan epoch before this step's commits: read before this CTA
        // publishes anything (the last block changes both only after every block has)
        cs.cursor = __ldcg(c.ring_state);
        cs.ep = (unsigned long long)(__ldcg(c.epoch) & 0xffffffu) << 40;
        cs.wmax = 0ull;
    }
    // fp64 decisions: the packed weights into shared memory (asynchronous copies,
    // landing during the arrivals and the advance; read by every round's Q forward)
    const double* sw = p.qpack;
    if constexpr (!TCQ) {
        double* swm = reinterpret_cast<double*>(smem_raw + step_score_bytes());
        const int nd = (int)QLayout<M>::doubles(p.cfg.n_tasks, p.H);
        for (int k = threadIdx.x; 2 * k < nd; k += blockDim.x) {
            const uint32_t d = (uint32_t)__cvta_generic_to_shared(swm + 2 * k);
            if (2 * k + 1 < nd) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(p.qpack + 2 * k));
            else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(p.qpack + 2 * k));
        }
        asm volatile("cp.async.commit_group;\n" ::);
        sw = swm;
    }
    if (threadIdx.x < 32) load_score(sc, p.cfg, p.aux);
    __syncthreads();
    if constexpr (TCQ) {
        tc::fence_after_sync();
        cx.tmem = *reinterpret_cast<uint32_t*>(bars + 2);
        if (threadIdx.x == 0) {
            const uint32_t nb = (uint32_t)TcLayout{p.H}.bytes();
            tc::mbar_expect_tx(&bars[0], nb);
            tc::bulk_g2s(const_cast<float*>(cx.img), p.tc_img, nb, &bars[0]);
        }
    }
    const int64_t it = *p.iter_dev;
    const int P = p.pending_P;
    const int nvb = (p.E + SC_ENVS - 1) / SC_ENVS;
    // CTA-uniform rounds.  Virtual blocks: blockIdx.x, + gridDim.x, ... when the whole grid
    // is resident at once (every look-back predecessor is running or done); else taken
    // from a ticket in start order, so a block only ever waits on blocks already handed
    // to running CTAs
    const unsigned ep_par = (unsigned)(cs.ep >> 40) & 1u;
    for (int vb = blockIdx.x;; vb += gridDim.x) {
        if (c.use_ticket) {
            __syncthreads();  // the previous round's reads of cs.vb are done
            if (threadIdx.x == 0) cs.vb = (int)atomicAdd(&c.vticket[ep_par], 1u);
            __syncthreads();
            vb = cs.vb;
        }
        if (vb >= nvb) break;
        const int le = warp * 2 + grp;
        const int e = vb * SC_ENVS + le;
        const bool live = e < p.E;
        StepOut so;
        so.cs = &cs;
        so.vb = vb;
        so.le = le;
        so.live = live;
        so.has_wl = false;
        BE_PROBE(0)
        if (p.gen_workload) {  // TrainingWorkload.next_arrival (trainer.py:304-316), lane 0 stores
            train_workload_next(p.wl, live ? e : p.E - 1, live && gl == 0, so.U, so.task, so.rate);
            so.has_wl = true;
        }
        BE_PROBE(1)
        if constexpr (!TCQ) asm volatile("cp.async.wait_all;\n" ::);  // visible to all after step_env's barrier
        step_env<M, 16, TCQ, SC_QU>(p, live ? e : p.E - 1, live, sc, sw, true, T, H, D, TCQ ? &cx : nullptr, &so);
        // ---- this env's transitions into the block list (independent of the cross-block
        // prefix, so it overlaps warp 0's look-back)
        BE_PROBE(3)
        const int64_t L = (live && so.jlo <= so.jhi) ? so.jhi - so.jlo + 1 : 0;
        // this env's first list entry: the counts of the block's earlier envs (cs.cnt is
        // complete since commit_publish's barrier)
        long long pre = 0;
        for (int l = 0; l < le; ++l) pre += cs.cnt[l];
        if (L) commit_list(p, cs, e, le, P, so.jlo, L, pre, gl, gmask);
        BE_PROBE(4)
        if (warp == 0 && vb > 0) {
            // the block's exclusive prefix: look back over windows of 256 predecessors
            // (8 per lane, nearest first), summing aggregates up to the nearest
            // inclusive prefix; the aggregates were published right after each
            // block's advance, so one window usually completes the scan
            long long excl = 0;
            for (int j = vb - 1;; j -= 256) {
                unsigned long long v[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int idx = j - lane * 8 - k;
                    v[k] = idx >= 0 ? ld_relaxed_u64(&c.scan[idx]) : (2ull << 38);
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int idx = j - lane * 8 - k;
                    while (idx >= 0 && ((v[k] >> 40) != (cs.ep >> 40) || ((v[k] >> 38) & 3ull) == 0))
                        v[k] = ld_relaxed_u64(&c.scan[idx]);
                }
                int kstop = 8;  // this lane's nearest inclusive prefix
#pragma unroll
                for (int k = 7; k >= 0; --k)
                    if (((v[k] >> 38) & 3ull) == 2ull) kstop = k;
                const unsigned pb = __ballot_sync(FULL, kstop < 8);
                const int stop = pb ? __ffs(pb) - 1 : 32;  // lanes < stop: all 8; lane stop: k <= kstop
                long long val = 0;
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (lane < stop || (lane == stop && k <= kstop)) val += (long long)(v[k] & ((1ull << 38) - 1));
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) val += __shfl_xor_sync(FULL, val, off);
                excl += val;
                if (pb) break;
            }
            if (lane == 0) {
                cs.excl = excl;
                // acquire what the observed publications released (their cursor reads)
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                st_release_u64(&c.scan[vb], cs.ep | (2ull << 38) | (unsigned long long)(excl + cs.agg));
            }
        } else if (warp == 0 && lane == 0) {
            cs.excl = 0;
        }
        if (warp == 0 && lane == 0 && vb == nvb - 1) {  // commits this step: advance the ring
            const long long n = cs.excl + cs.agg;
            c.ring_state[3] = n;
            c.ring_state[0] = (cs.cursor + n) % c.capacity;
            c.ring_state[1] = c.ring_state[1] + n < c.capacity ? c.ring_state[1] + n : c.capacity;
            c.ring_state[2] += n;
            *c.epoch = *c.epoch + 1u;
            if (c.use_ticket) c.vticket[ep_par ^ 1u] = 0u;  // the next launch's counter
        }
        BE_PROBE(5)
        __syncthreads();
        BE_PROBE(6)
        // ---- the block's transitions, one per thread: ring slot = block base + list index
        const long long n_blk = cs.agg;
        const int64_t s0 = (cs.cursor + cs.excl) % c.capacity;
        const long long n_list = n_blk < c.list_cap ? n_blk : c.list_cap;
        if (n_blk > c.list_cap) {  // (block-uniform) the list overflowed
            // entries past the list, found by rescanning the ready flags — before any
            // listed entry's flag is cleared below, so the ranks match the list's
            if (live && L) commit_copy_overflow(p, c, e, D, P, so.jlo, L, pre, s0, gl, gmask);
            __syncthreads();
        }
        for (long long i = threadIdx.x; i < n_list; i += blockDim.x) {
            const int lei = cs.le[i];
            int64_t slot = s0 + i;
            while (slot >= c.capacity) slot -= c.capacity;
            commit_copy<SC_CW>(p, c, vb * SC_ENVS + lei, D, P, cs.sj[i], slot);
        }
        if (live) {
            if (gl == 0) {
                c.low[e] = so.oldest;
                const int64_t win = it + 1 - so.oldest;
                if (win >= P && atomicCAS(&c.status[0], 0, BE_ECAPACITY) == 0) c.status[1] = e;
                if (win > 0) atomicMax(&cs.wmax, (unsigned long long)win);
            }
        }
        BE_PROBE(7)
        __syncthreads();  // cs is reused by the next round
        BE_PROBE(8)
    }
    // high-water mark of in-flight decisions per env (ring_state[4])
    if (threadIdx.x == 0 && cs.wmax > (unsigned long long)__ldcg(c.ring_state + 4))
        atomicMax(reinterpret_cast<unsigned long long*>(c.ring_state + 4), cs.wmax);
    if constexpr (TCQ) {
        tc::fence_before_sync();
        __syncthreads();
        if ((threadIdx.x >> 5) == 0) tc::tmem_dealloc(cx.tmem, (uint32_t)p.tc_ncols);
    }
    pdl_trigger();
}

// The tensor-core router image for the fused training step (the weights change every
// update; the fp64 packed weights are kept current by the learner's fused update).
template <int M>
__global__ void __launch_bounds__(256) tc_image_kernel(const double* w1, const double* b1, const double* w2,
                                                       const double* b2, int D, int H, float* img) {
    pdl_wait();
    if constexpr (M <= TC_MP) tc_pack_image<M>(w1, b1, w2, b2, D, H, img, blockIdx.x * blockDim.x + threadIdx.x,
                                                 gridDim.x * blockDim.x);
    pdl_trigger();
}

// The greedy decision of one env on the tensor cores, inside the env step (every
// thread of the CTA calls it once per round: two CTA barriers).  Layer 1 of the 16
// envs of the CTA as one tcgen05.mma.kind::tf32 tile (3xTF32 split, M = 128 rows of
// which 16 are envs, N = H, accumulators in TMEM); relu + layer 2 by warps 0 and 4
// (TMEM lanes 0-31) on FFMA2 with the same summation structure as route_tc, so the
// router's pairwise error bounds certify the leader; a decision the bound cannot
// certify is re-evaluated by the group in fp64 (qnet_group, the fused step's own
// arithmetic).  Returns the greedy tier (identical to the fp64 step's).
template <int M>
__device__ __forceinline__ int tc_decide(TcStepCtx& cx, bool live, bool explore, int task, const double (&xt)[M],
                                         double xr, const double* sw, int T, int H, int D, int le, int gl) {
    const TcLayout L{H};
    const float* B1h = cx.img + L.b1h() / 4;
    const float* B1l = cx.img + L.b1l() / 4;
    const float4* W2q = reinterpret_cast<const float4*>(cx.img + L.w2p() / 4);
    const float* fb2 = cx.img + L.b2() / 4;
    const float* C = cx.img + L.bound() / 4;
    const float* Dp = cx.img + L.pairs() / 4;
    // ---- A row le: input gl (fp32-rounded, then tf32 hi + lo), the bias input = 1
    float xk = 0.f;
    if (gl < T) xk = gl == task ? 1.f : 0.f;
#pragma unroll
    for (int m = 0; m < M; ++m)
        if (gl == T + m) xk = __double2float_rn(xt[m]);
    if (gl == T + M) xk = __double2float_rn(xr);
    if (gl == D) xk = 1.f;
    if (!live) xk = 0.f;
    if (gl < TC_K) {
        const float hi = tc::to_tf32(xk);
        cx.Ah[umma_off(le, gl)] = hi;
        cx.Al[umma_off(le, gl)] = tc::to_tf32(__fsub_rn(xk, hi));
    }
    tc::fence_proxy_async_smem();
    if (!cx.img_ready) {  // issued at kernel start: the copy overlapped the first round's advance
        tc::mbar_wait(cx.img_bar, 0);
        cx.img_ready = true;
    }
    tc::fence_before_sync();
    __syncthreads();
    if (threadIdx.x == 0) {
        tc::fence_after_sync();
        const uint32_t idesc = tc::idesc_tf32(128, H);
#pragma unroll
        for (int s = 0; s < TC_K / 8; ++s) {  // K-step s reads K-groups 2s, 2s + 1
            const uint64_t ah = tc::smem_desc(cx.Ah + s * 64, 128, 512), al = tc::smem_desc(cx.Al + s * 64, 128, 512);
            const uint64_t bh = tc::smem_desc(B1h + s * 64, 128, 512), bl = tc::smem_desc(B1l + s * 64, 128, 512);
            tc::mma_tf32(cx.tmem, ah, bh, idesc, s > 0);
            tc::mma_tf32(cx.tmem, ah, bl, idesc, true);
            tc::mma_tf32(cx.tmem, al, bh, idesc, true);
        }
        tc::mma_commit(cx.bar);
    }
    tc::mbar_wait(cx.bar, cx.phase);
    cx.phase ^= 1u;
    tc::fence_after_sync();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if ((warp & 3) == 0) {  // warps 0 and 4: TMEM lanes 0-31 = rows 0-31 (rows 0-15 are envs)
        const int half = warp >> 2, HP = H / 2;
        float2 a[2][M];
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
            for (int m = 0; m < M; ++m) a[s2][m] = make_float2(0.f, 0.f);
        const int nch = HP / TC_CW;
        auto consume = [&](const float(&u)[TC_CW], int jb) {
#pragma unroll
            for (int i = 0; i < TC_CW / 2; i += 2) {
                const float2 h0 = make_float2(fmaxf(u[2 * i], 0.f), fmaxf(u[2 * i + 1], 0.f));
                const float2 h1 = make_float2(fmaxf(u[2 * i + 2], 0.f), fmaxf(u[2 * i + 3], 0.f));
                const float4* g = W2q + (size_t)((jb + 2 * i) >> 2) * 4;
                const float4 g0 = g[0], g1 = g[1];
                a[0][0] = ffma2(h0, make_float2(g0.x, g0.y), a[0][0]);
                a[1][0] = ffma2(h1, make_float2(g1.x, g1.y), a[1][0]);
                if (M > 1) {
                    constexpr int m1 = M > 1 ? 1 : 0;
                    a[0][m1] = ffma2(h0, make_float2(g0.z, g0.w), a[0][m1]);
                    a[1][m1] = ffma2(h1, make_float2(g1.z, g1.w), a[1][m1]);
                }
                if (M > 2) {
                    constexpr int m2 = M > 2 ? 2 : 0;
                    const float4 g2 = g[2];
                    a[0][m2] = ffma2(h0, make_float2(g2.x, g2.y), a[0][m2]);
                    a[1][m2] = ffma2(h1, make_float2(g2.z, g2.w), a[1][m2]);
                }
                if (M > 3) {
                    constexpr int m3 = M > 3 ? 3 : 0;
                    const float4 g3 = g[3];
                    a[0][m3] = ffma2(h0, make_float2(g3.x, g3.y), a[0][m3]);
                    a[1][m3] = ffma2(h1, make_float2(g3.z, g3.w), a[1][m3]);
                }
            }
        };
        // double-buffered TMEM loads (two named buffers: no local-memory indexing)
        float u0[TC_CW], u1[TC_CW];
        const uint32_t col0 = cx.tmem + (uint32_t)(half * HP);
        tc::tmem_ld_issue(col0, u0);
        for (int c = 0; c < nch; c += 2) {
            tc::tmem_ld_wait(u0);
            if (c + 1 < nch) tc::tmem_ld_issue(col0 + (uint32_t)((c + 1) * TC_CW), u1);
            consume(u0, half * HP + c * TC_CW);
            if (c + 1 < nch) {
                tc::tmem_ld_wait(u1);
                if (c + 2 < nch) tc::tmem_ld_issue(col0 + (uint32_t)((c + 2) * TC_CW), u0);
                consume(u1, half * HP + (c + 1) * TC_CW);
            }
        }
        if (lane < 16) {
#pragma unroll
            for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
                for (int m = 0; m < M; ++m) cx.part[((half * 16 + lane) * 2 + s2) * TC_MP + m] = a[s2][m];
        }
    }
    tc::fence_before_sync();  // this round's TMEM loads complete before the next round's MMA
    __syncthreads();
    // ---- q (fp32) of row le: the two column halves merged as route_tc merges them
    float q[M];
    int best = 0;
    float bv = 0.f;
    bool fin = true;
#pragma unroll
    for (int m = 0; m < M; ++m) {
        float2 t[2];
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
            const float2 own = cx.part[((0 * 16 + le) * 2 + s2) * TC_MP + m];
            const float2 oth = cx.part[((1 * 16 + le) * 2 + s2) * TC_MP + m];
            t[s2] = make_float2(__fadd_rn(own.x, oth.x), __fadd_rn(own.y, oth.y));
        }
        const float t0 = __fadd_rn(t[0].x, t[0].y), t1 = __fadd_rn(t[1].x, t[1].y);
        q[m] = __fadd_rn(__fadd_rn(t0, t1), fb2[m]);
        fin = fin && isfinite(q[m]);
        if (m == 0 || q[m] > bv) {  // first maximum (a tie is never certified)
            best = m;
            bv = q[m];
        }
    }
    // ---- certification: the leader beats every other action by more than the pair's bound
    float xf[TC_K];
#pragma unroll
    for (int k = 0; k < TC_K; ++k) xf[k] = 0.f;
#pragma unroll
    for (int k = 0; k < TC_K; ++k) {
        if (k < T) xf[k] = k == task ? 1.f : 0.f;
#pragma unroll
        for (int m = 0; m < M; ++m)
            if (k == T + m) xf[k] = __double2float_rn(xt[m]);
        if (k == T + M) xf[k] = __double2float_rn(xr);
    }
    float Bd = C[D];
#pragma unroll
    for (int k = 0; k < TC_K; ++k)
        if (k < D) Bd = __fmaf_ru(fabsf(xf[k]), C[k], Bd);
    bool sure = fin;
#pragma unroll
    for (int b = 0; b < M; ++b)
#pragma unroll
        for (int sx = b + 1; sx < M; ++sx) {
            if (best == b || best == sx) {
                const float* dp = Dp + tc_pair(b, sx) * TC_K;
                float v = dp[D];
#pragma unroll
                for (int k = 0; k < TC_K; ++k)
                    if (k < D) v = __fmaf_ru(fabsf(xf[k]), dp[k], v);
                const float Bp = __fadd_ru(v, Bd);
                const float other = best == b ? q[sx] : q[b];
                sure = sure && isfinite(Bp) && __dsub_rd((double)bv, (double)other) > (double)Bp;
            }
        }
    sure = M == 1 || sure;
    int tier = best;
    // fp64 re-evaluation where the bound cannot certify (group-wide shuffles: both
    // groups of the warp run it when either needs it)
    if (__ballot_sync(FULL, live && !explore && !sure)) {
        double q64[M];
        qnet_group<M, 16>(sw, T, H, task, xt, xr, q64);
        if (!sure) tier = argmax_first<M>(q64);
    }
    return tier;
}

size_t step_tc_smem_bytes(int H) { return TcStepSmem(H).bytes; }

void step_tc_prepare(int M, int H) {
    const int smem = (int)TcStepSmem(H).bytes;
    switch (M) {
#define BE_TCP(MM)                                                                                          \
    case MM:                                                                                                \
        cudaFuncSetAttribute(env_step_commit_kernel<MM, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
        cudaFuncSetAttribute(env_step_commit_kernel<MM, true>, cudaFuncAttributePreferredSharedMemoryCarveout,   \
                             (int)cudaSharedmemCarveoutMaxShared); /* two CTAs per SM (shared TMEM) */       \
        break;
        BE_TCP(1) BE_TCP(2) BE_TCP(3) BE_TCP(4)
#undef BE_TCP
        default: break;
    }
}

// One env per LPE-lane group (all 32 lanes of the warp call it: the group
// reductions are warp-wide); `live` = false for a padding group past the last env.
template <int M, int LPE, bool TCQ, int QU>
__device__ __forceinline__ void step_env(const StepParams& p, int e, bool live, const Score& sc, const double* sw,
                                         bool policy, int T, int H, int D, TcStepCtx* tcx, StepOut* so) {
    const int lane = threadIdx.x & 31;
    const int gl = lane & (LPE - 1), grp = LPE == 32 ? 0 : lane / LPE;
    const unsigned gmask = LPE == 32 ? FULL : (0xffffu << (grp * LPE));
    const TierC tc = lane_tier(p.cfg, gl, p.skip);  // skip table read through L1
    const bool al = live && tc.tier >= 0;
    const uint32_t mask = (1u << p.cap_log2) - 1u;
    Slot* ring = p.rings + ((size_t)e * p.R + (al ? gl : 0)) * ((size_t)mask + 1);
    Rep r;
    if (al) r = reps_of(p.state, e, p.R)[gl];
    else rep_reset(r);
    EnvState* es = state_of(p.state, e, p.E, p.R);
    // records are indexed by request id modulo rec_ld (a ring for long runs)
    // complete() writes at base + id; id is the 24-bit slot id.
    const RecOut out = RecOut::row(p.rec, (int64_t)e * p.rec_ld);
    bool ok = true;
    if (p.drain) {
        // drain (simcore.py:151-153); new_segment: the stable-segment reset of run_eval
        // (evalkit.py:186-192) — drain, then a fresh ClusterSim and estimator for the
        // selected envs; request ids keep counting (they are trace indices)
        const bool sel = live && (!p.seg_mask || p.seg_mask[e]);
        if (al && sel) ok = advance_lane(r, tc, __longlong_as_double(0x7ff0000000000000LL), ring, mask, sc, out);
        if (sel && p.new_segment) rep_reset(r);  // the FIFO is empty: its cursor may stay
        if (al && sel) reps_of(p.state, e, p.R)[gl] = r;
        if (sel && p.new_segment && gl == 0) {
#pragma unroll
            for (int k = 0; k < 5; ++k) es->w[k] = 0.0;
            es->n = 0;
        }
        const bool all_ok = (__ballot_sync(FULL, !ok) & gmask) == 0;
        if (sel && !all_ok && gl == 0 && atomicCAS(&p.status[0], 0, BE_ECAPACITY) == 0) p.status[1] = e;
        return;
    }
    if (p.phase == 2) {
        // submit (simcore.py:94-111) of the decision the router left in action_out
        const double U2 = p.arrival[e];
        const int task2 = live ? p.task[e] : 0;
        const int64_t id2 = es->next_id;
        const uint8_t* act = p.action_out;
        if (p.iter_dev) act += (size_t)(*p.iter_dev % p.pending_P) * (size_t)p.E;
        const int tier2 = live ? (int)act[e] : 0;
        const unsigned key2 = (al && tc.tier == tier2) ? (((unsigned)r.count << 5) | (unsigned)gl) : 0xffffffffu;
        const unsigned best2 = group_min<LPE>(key2, grp);
        const bool bad2 = best2 == 0xffffffffu || task2 >= T;
        if (live && !bad2 && (int)(best2 & 31u) == gl) {
            const uint32_t rid = (uint32_t)(id2 % p.rec_ld);
            p.rec.flags[(int64_t)e * p.rec_ld + rid] = 0;  // record slot now "in flight"
            ok &= submit_lane(r, tc, U2, rid | ((uint32_t)task2 << 24), ring, mask);
        }
        if (al) reps_of(p.state, e, p.R)[gl] = r;
        if (live && gl == 0) es->next_id = id2 + 1;
        if (p.crange) {  // oldest request in flight (FIFO heads), for the commit's overflow check
            const int64_t oh = group_min64<LPE>((al && r.count > 0) ? id_of_slot(id2, r.h_idtask & 0xffffffu, p.pending_P)
                                                                   : INT64_MAX);
            if (live && gl == 0) p.crange[3 * (int64_t)e + 2] = oh;
        }
        const bool all_ok2 = (__ballot_sync(FULL, !ok) & gmask) == 0;
        if (live && gl == 0 && (bad2 || !all_ok2)) {
            if (atomicCAS(&p.status[0], 0, bad2 ? BE_EINVAL : BE_ECAPACITY) == 0) p.status[1] = e;
        }
        return;
    }
    const bool wl_in = so != nullptr && so->has_wl;
    const double U = wl_in ? so->U : p.arrival[e];
    int task = live ? (wl_in ? so->task : (int)p.task[e]) : 0;
    const bool bad_task = live && task >= T;  // encode raises (policy.py:57-58)
    if (task >= T) task = 0;
    const uint32_t cr_h0 = r.head, cr_idt0 = r.h_idtask;
    const int cr_c0 = r.count;
    if (al) ok = advance_lane(r, tc, U, ring, mask, sc, out);
    if (p.crange || so) {
        // the requests this advance completed are the popped FIFO prefix of every replica
        // (ids increase along a FIFO): the env's lowest / highest completed id of this
        // step bound the commit scan (be_train_iteration), instead of the whole window of
        // unresolved decisions
        const int popped = al ? cr_c0 - r.count : 0;
        const int64_t t1 = es->next_id - 1;
        int64_t jlo = INT64_MAX, jhi = -1;
        if (popped > 0) {
            const uint32_t s_first = cr_idt0 & 0xffffffu;
            const uint32_t s_last = popped == 1 ? s_first : ring[(cr_h0 + popped - 1) & mask].idtask & 0xffffffu;
            jlo = id_of_slot(t1, s_first, p.pending_P);
            jhi = id_of_slot(t1, s_last, p.pending_P);
        }
        jlo = group_min64<LPE>(jlo);
        jhi = group_max64<LPE>(jhi);
        if (so) {
            so->jlo = jlo;
            so->jhi = jhi;
            commit_publish(p, *so, (int)group_sum<LPE>((unsigned)popped, grp));
            BE_PROBE(2)
        } else if (live && gl == 0) {
            p.crange[3 * (int64_t)e] = jlo;
            p.crange[3 * (int64_t)e + 1] = jhi;
        }
    }
    Estimator est;
#pragma unroll
    for (int k = 0; k < 5; ++k) est.w[k] = es->w[k];
    est.n = es->n;
    const int64_t id = es->next_id;
    const double cur = wl_in ? so->rate : p.true_rate ? p.true_rate[e] : 0.0;
    const double rate = estimator_observe(est, U, p.cfg.estimator_true_rate != 0, cur, p.cfg.prior_rate);
    int obs[M];
#pragma unroll
    for (int m = 0; m < M; ++m) obs[m] = (int)group_sum<LPE>((al && tc.tier == m) ? (unsigned)r.count : 0u, grp);
    double xt[M], q[M];
#pragma unroll
    for (int m = 0; m < M; ++m) {
        xt[m] = __ddiv_rn((double)obs[m], p.cfg.batch_scales[m]);
        q[m] = 0.0;
    }
    const double xr = __ddiv_rn(rate, p.cfg.rate_scale);
    int tier = 0;
    bool explore = false;
    if (p.phase == 1) {
        // observe only: the decision comes from a separate router launch
    } else if (p.forced) {
        tier = p.forced[e];
    } else if (p.static_tier >= 0) {
        tier = p.static_tier;
    } else {
        // select_action (policy.py:125-132): explore with probability epsilon
        double epsilon = p.epsilon;
        uint64_t counter = p.counter;
        if (p.iter_dev) {
            const int64_t it = *p.iter_dev;
            epsilon = epsilon_at(it, p.eps_start, p.eps_end, p.eps_decay);
            counter = (uint64_t)it;
        }
        if (epsilon > 0.0) {
            P4 rnd = philox4x32_10(counter, (uint64_t)e, p.seed);
            if (u01(rnd.x[0], rnd.x[1]) < epsilon) {
                explore = true;
                tier = (int)below(rnd.x[2], (uint32_t)M);
            }
        }
        if constexpr (TCQ) {
            const int dec = tc_decide<M>(*tcx, live, explore, task, xt, xr, sw, T, H, D,
                                         (threadIdx.x >> 5) * 2 + grp, gl);
            if (!explore) tier = dec;
        } else {
            qnet_group<M, LPE, QU>(sw, T, H, task, xt, xr, q);
            if (!explore) tier = argmax_first<M>(q);
        }
    }
    if (live && gl < M) {
#pragma unroll
        for (int m = 0; m < M; ++m) {
            if (gl == m) {
                if (p.obs_out) p.obs_out[(size_t)e * M + m] = obs[m];
                if (p.q_out) p.q_out[(size_t)e * M + m] = q[m];
            }
        }
    }
    double* x_out = p.x_out;
    uint8_t* action_out = p.action_out;
    if (p.iter_dev) {  // pending slot it % P of the learner's deferred-reward store
        const size_t slot = (size_t)(*p.iter_dev % p.pending_P);
        if (x_out) x_out += slot * (size_t)p.E * D;
        if (action_out) action_out += slot * (size_t)p.E;
    }
    if (live && x_out && gl < D) {
        // encode (policy.py:52-65): [onehot(task), obs/scale, rate/rate_scale]
        double v = 0.0;
        if (gl < T) v = gl == task ? 1.0 : 0.0;
#pragma unroll
        for (int m = 0; m < M; ++m)
            if (gl == T + m) v = xt[m];
        if (gl == T + M) v = xr;
        x_out[(size_t)e * D + gl] = v;
    }
    unsigned key = (al && tc.tier == tier) ? (((unsigned)r.count << 5) | (unsigned)gl) : 0xffffffffu;
    unsigned best = p.phase == 1 ? 0u : group_min<LPE>(key, grp);
    bool bad = best == 0xffffffffu;
    if (p.phase == 0 && live && !bad && (int)(best & 31u) == gl) {
        uint32_t rid = (uint32_t)(id % p.rec_ld);
        p.rec.flags[(int64_t)e * p.rec_ld + rid] = 0;  // record slot now "in flight"
        ok &= submit_lane(r, tc, U, rid | ((uint32_t)task << 24), ring, mask);
    }
    if (al) reps_of(p.state, e, p.R)[gl] = r;
    if ((p.crange || so) && p.phase == 0) {  // oldest request in flight after the submit
        const int64_t oh = group_min64<LPE>((al && r.count > 0) ? id_of_slot(id, r.h_idtask & 0xffffffu, p.pending_P)
                                                               : INT64_MAX);
        if (so) so->oldest = oh;
        else if (live && gl == 0) p.crange[3 * (int64_t)e + 2] = oh;
    }
    if (live && gl == 0) {
        if (p.rate_out) p.rate_out[e] = rate;
        if (action_out && p.phase == 0) action_out[e] = (uint8_t)tier;
#pragma unroll
        for (int k = 0; k < 5; ++k) es->w[k] = est.w[k];
        es->n = est.n;
        if (p.phase == 0) es->next_id = id + 1;
    }
    const bool all_ok = (__ballot_sync(FULL, !ok) & gmask) == 0;
    if (live && gl == 0 && (bad || bad_task || !all_ok)) {
        if (atomicCAS(&p.status[0], 0, (bad || bad_task) ? BE_EINVAL : BE_ECAPACITY) == 0) p.status[1] = e;
    }
}

int launch_env_reset(be_env* env, const uint8_t* mask, cudaStream_t st) {
    int threads = 256;
    int blocks = (int)(((long long)env->E * 32 + threads - 1) / threads);
    env_reset_kernel<<<blocks, threads, 0, st>>>(env->reps, env->E, env->R, mask);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "env reset");
}

// Weight packing for the env step, fused with the next training arrival of every env
// (be_train_iteration): CTAs [0, QPACK_CTAS) pack, the rest run the workload.
// With a tensor-core image requested (tc_img), CTAs [QPACK_CTAS, + TCPACK_CTAS) pack it.
constexpr int TCPACK_CTAS = 8;
template <int M>
__global__ void __launch_bounds__(256) prep_kernel(const double* w1, const double* b1, const double* w2,
                                                   const double* b2, int T, int H, double* out, WorkloadArgs wl,
                                                   float* tc_img) {
    pdl_wait();  // the weights were updated by the previous kernel
    const int ntc = tc_img ? TCPACK_CTAS : 0;
    if (blockIdx.x < QPACK_CTAS) {
        stage_qnet<M>(w1, b1, w2, b2, T, H, out, blockIdx.x * blockDim.x + threadIdx.x, QPACK_CTAS * blockDim.x);
    } else if ((int)blockIdx.x < QPACK_CTAS + ntc) {
        if constexpr (M <= TC_MP)
            tc_pack_image<M>(w1, b1, w2, b2, T + M + 1, H, tc_img,
                             (blockIdx.x - QPACK_CTAS) * blockDim.x + threadIdx.x, TCPACK_CTAS * blockDim.x);
    } else {
        const int e = (blockIdx.x - QPACK_CTAS - ntc) * blockDim.x + threadIdx.x;
        if (e < wl.E) train_workload_env(wl, e);
    }
    pdl_trigger();
}

template <int M>
static int launch_step_m(const StepParams& p, size_t smem, cudaStream_t st, const WorkloadArgs* wl) {
    const bool two = p.R <= 16 && p.cfg.n_tasks + M + 1 <= 16;
    auto kern = two ? env_step_kernel<M, 16> : env_step_kernel<M, 32>;
    float* tc_img = const_cast<float*>(p.tc_img);
    if (p.fuse_commit && p.gen_workload) {  // the step generates the workload; the learner keeps qpack packed
    } else if (p.qpack && wl) {  // pack the weights (+ the tensor-core image) + the training workload, one launch
        const int ntc = tc_img ? TCPACK_CTAS : 0;
        cudaError_t e = launch_pdl(prep_kernel<M>, dim3(QPACK_CTAS + ntc + (wl->E + 255) / 256), dim3(256), 0, st,
                                   p.w1, p.b1, p.w2, p.b2, p.cfg.n_tasks, p.H, const_cast<double*>(p.qpack), *wl,
                                   tc_img);
        if (e != cudaSuccess) return set_cuda_error(e, "prep launch");
    } else if (p.qpack) {  // pack the (possibly just updated) weights for this step
        cudaError_t e = launch_pdl(stage_qpack_kernel<M>, dim3(QPACK_CTAS), dim3(256), 0, st, p.w1, p.b1, p.w2, p.b2,
                                   p.cfg.n_tasks, p.H, const_cast<double*>(p.qpack));
        if (e != cudaSuccess) return set_cuda_error(e, "stage_qpack launch");
    }
    if constexpr (M <= TC_MP) {
        if (tc_img && p.fuse_commit) {  // image, then step + arrivals + commit with tcgen05 decisions
            cudaError_t e = launch_pdl(tc_image_kernel<M>, dim3(TCPACK_CTAS), dim3(256), 0, st, p.w1, p.b1, p.w2,
                                       p.b2, p.cfg.n_tasks + M + 1, p.H, tc_img);
            if (e != cudaSuccess) return set_cuda_error(e, "router image launch");
            int dev = 0, sms = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            // two CTAs per SM (they share its TMEM); when the occupancy calculator does not
            // vouch for all of them being resident at once, virtual blocks come from a ticket
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, env_step_commit_kernel<M, true>, 256,
                                                          step_tc_smem_bytes(p.H));
            if (per_sm < 1) return set_error(BE_EINVAL, "tensor-core step does not fit an SM");
            long long blocks = ((long long)p.E + SC_ENVS - 1) / SC_ENVS;
            if (blocks > 2LL * sms) blocks = 2LL * sms;
            StepParams q = p;
            q.cm.use_ticket = blocks > (long long)per_sm * sms ? 1 : 0;
            e = launch_pdl(env_step_commit_kernel<M, true>, dim3((unsigned)blocks), dim3(256), step_tc_smem_bytes(p.H),
                           st, q);
            return e == cudaSuccess ? BE_OK : set_cuda_error(e, "env step + commit (tensor cores) launch");
        }
        if (tc_img) return set_error(BE_EINVAL, "the tensor-core env step runs fused with the replay commit");
    }
    if (p.fuse_commit) {  // the training step + replay commit (two envs per warp)
        if (!two) return set_error(BE_EINVAL, "fused commit needs <= 16 replicas and input dim <= 16");
        int per_sm = 0, dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        smem = step_score_bytes() + QLayout<M>::doubles(p.cfg.n_tasks, p.H) * sizeof(double);  // + the weights
        if (smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(env_step_commit_kernel<M, false>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute");
        }
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, env_step_commit_kernel<M, false>, 256, smem);
        if (per_sm < 1) per_sm = 1;
        // one resident wave (the look-back needs every predecessor running or done)
        long long blocks = ((long long)p.E + SC_ENVS - 1) / SC_ENVS;
        if (blocks > (long long)sms * per_sm) blocks = (long long)sms * per_sm;
        cudaError_t e = launch_pdl(env_step_commit_kernel<M, false>, dim3((unsigned)blocks), dim3(256), smem, st, p);
        return e == cudaSuccess ? BE_OK : set_cuda_error(e, "env step + commit launch");
    }
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute");
    }
    int threads = 256;
    const long long warps = two ? ((long long)p.E + 1) / 2 : (long long)p.E;
    long long blocks = (warps * 32 + threads - 1) / threads;
    int per_sm = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    if (per_sm < 1) per_sm = 1;
    if (blocks > (long long)sms * per_sm) blocks = (long long)sms * per_sm;
    cudaError_t e = launch_pdl(kern, dim3((unsigned)blocks), dim3(threads), smem, st, p);
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "env step launch");
}

static size_t step_smem_bytes() { return step_score_bytes(); }

static int dispatch_step(const StepParams& p, size_t smem, cudaStream_t st, const WorkloadArgs* wl = nullptr) {
    switch (p.cfg.n_tiers) {
        case 1: return launch_step_m<1>(p, smem, st, wl);
        case 2: return launch_step_m<2>(p, smem, st, wl);
        case 3: return launch_step_m<3>(p, smem, st, wl);
        case 4: return launch_step_m<4>(p, smem, st, wl);
        case 5: return launch_step_m<5>(p, smem, st, wl);
        case 6: return launch_step_m<6>(p, smem, st, wl);
        case 7: return launch_step_m<7>(p, smem, st, wl);
        case 8: return launch_step_m<8>(p, smem, st, wl);
        default: return set_error(BE_EINVAL, "n_tiers out of range");
    }
}

static StepParams base_params(be_env* env, int64_t rec_ld, const be_records* rec) {
    StepParams p{};
    p.cfg = env->cfg;
    make_score_aux(env->cfg, &p.aux);
    p.E = env->E;
    p.R = env->R;
    p.cap_log2 = env->cap_log2;
    p.state = env->reps;
    p.rings = reinterpret_cast<Slot*>(env->rings);
    p.rec_ld = rec_ld;
    p.rec = *rec;
    p.status = env->d_status;
    p.static_tier = -1;
    p.skip = env->d_skip;
    return p;
}

int launch_env_step(be_env* env, const double* arrival, const uint8_t* task,
                    const double* true_rate, const uint8_t* forced, const be_qweights* W,
                    int static_tier, double epsilon, uint64_t seed, uint64_t counter,
                    int64_t rec_ld, const be_records* rec, int32_t* obs_out, double* rate_out,
                    uint8_t* action_out, double* q_out, double* x_out, cudaStream_t st) {
    StepParams p = base_params(env, rec_ld, rec);
    p.arrival = arrival;
    p.task = task;
    p.true_rate = true_rate;
    p.forced = forced;
    p.static_tier = static_tier;
    p.epsilon = epsilon;
    p.seed = seed;
    p.counter = counter;
    p.obs_out = obs_out;
    p.rate_out = rate_out;
    p.action_out = action_out;
    p.q_out = q_out;
    p.x_out = x_out;
    bool policy = forced == nullptr && static_tier < 0;
    if (policy) {
        p.H = W->hidden;
        p.w1 = W->w1;
        p.b1 = W->b1;
        p.w2 = W->w2;
        p.b2 = W->b2;
    }
    if (policy) p.qpack = env->d_qpack;
    return dispatch_step(p, step_smem_bytes(), st);
}

int launch_env_step_split(be_env* env, int phase, const double* arrival, const uint8_t* task,
                          const double* true_rate, uint8_t* action, double* x_out, int32_t* obs_out,
                          double* rate_out, int64_t rec_ld, const be_records* rec, cudaStream_t st) {
    StepParams p = base_params(env, rec_ld, rec);
    p.phase = phase;
    p.arrival = arrival;
    p.task = task;
    p.true_rate = true_rate;
    p.action_out = action;
    p.x_out = x_out;
    p.obs_out = obs_out;
    p.rate_out = rate_out;
    return dispatch_step(p, step_smem_bytes(), st);
}

int launch_env_step_dev(be_env* env, const double* arrival, const uint8_t* task,
                        const double* true_rate, const be_qweights* W, uint64_t seed,
                        const int64_t* iter_dev, double eps_start, double eps_end, int64_t eps_decay,
                        int32_t pending_P, int64_t rec_ld, const be_records* rec, uint8_t* action_base,
                        double* x_base, cudaStream_t st, const WorkloadArgs* wl, int phase, float* tc_img,
                        int64_t* crange, const StepCommitArgs* commit) {
    StepParams p = base_params(env, rec_ld, rec);
    p.phase = phase;
    p.crange = crange;
    if (commit) {
        if (phase != 0 || rec_ld != pending_P) return set_error(BE_EINVAL, "the fused commit is the training step");
        p.cm = *commit;
        // BE_COMMIT_LIST_CAP (tests only): a smaller block list, to exercise the overflow path
        p.cm.list_cap = SC_LIST;
        if (const char* lc = getenv("BE_COMMIT_LIST_CAP")) {
            const int v = atoi(lc);
            if (v >= 0 && v < SC_LIST) p.cm.list_cap = v;
        }
        p.fuse_commit = 1;
        p.crange = nullptr;
        if (wl) {
            p.gen_workload = 1;
            p.wl = *wl;
        }
    }
    p.tc_img = tc_img;
    p.tc_ncols = W->hidden <= 32 ? 32 : W->hidden <= 64 ? 64 : W->hidden <= 128 ? 128 : 256;
    p.arrival = arrival;
    p.task = task;
    p.true_rate = true_rate;
    p.seed = seed;
    p.action_out = action_base;
    p.x_out = x_base;
    p.iter_dev = iter_dev;
    p.eps_start = eps_start;
    p.eps_end = eps_end;
    p.eps_decay = eps_decay;
    p.pending_P = pending_P;
    p.H = W->hidden;
    p.w1 = W->w1;
    p.b1 = W->b1;
    p.w2 = W->w2;
    p.b2 = W->b2;
    p.qpack = phase == 2 ? nullptr : env->d_qpack;  // submit: no weights needed
    return dispatch_step(p, step_smem_bytes(), st, wl);
}

int launch_stage_qpack(be_env* env, const be_qweights* W, cudaStream_t st) {
    const int T = env->cfg.n_tasks;
    cudaError_t e = cudaSuccess;
    switch (env->cfg.n_tiers) {
#define BE_QP(MM)                                                                                             \
    case MM:                                                                                                  \
        e = launch_pdl(stage_qpack_kernel<MM>, dim3(QPACK_CTAS), dim3(256), 0, st, W->w1, W->b1, W->w2, W->b2, T, \
                       W->hidden, env->d_qpack);                                                              \
        break;
        BE_QP(1) BE_QP(2) BE_QP(3) BE_QP(4) BE_QP(5) BE_QP(6) BE_QP(7) BE_QP(8)
#undef BE_QP
        default: return set_error(BE_EINVAL, "n_tiers out of range");
    }
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "stage_qpack launch");
}

bool env_step_commit_supported(const be_env* env) {
    return env->R <= 16 && env->cfg.n_tasks + env->cfg.n_tiers + 1 <= 16;
}

int launch_env_drain(be_env* env, int64_t rec_ld, const be_records* rec, cudaStream_t st,
                     const uint8_t* mask, int new_segment) {
    StepParams p = base_params(env, rec_ld, rec);
    p.drain = 1;
    p.seg_mask = mask;
    p.new_segment = new_segment;
    return dispatch_step(p, step_smem_bytes(), st);
}

}  // namespace be


#ifdef BE_PROBE_T
extern "C" int be_debug_probe(unsigned long long* out, int n) {
    return (int)cudaMemcpyFromSymbol(out, be::be_probe_t, (size_t)n * sizeof(unsigned long long));
}
#endif
