// reduce.cu — on-device evaluation reducer (K5).
//
//   windowed(rewards, 20) + threshold_counts   evalkit.py:217-241
//   miss fraction by segment rate              evalkit.py:61-68
//   mean reward by segment rate                evalkit.py:70-74
//
// One thread per environment owns the strictly sequential fp64 prefix sum
// c_{k+1} = c_k + r_k (np.cumsum order — any parallel scan would change the
// rounding and therefore the threshold counts).  Rewards
// are env-major in HBM, so each warp streams a 32-env x CH-request tile per
// stage with cp.async (16-byte LDGSTS, every env row a CH x 8-byte burst) into
// padded shared memory, two stages deep, while the lanes scan the other; big
// batches give every warp two 32-env groups in turn with 256-byte bursts (half
// the concurrent row streams — DRAM row locality, not latency, bounds this kernel).
// The trailing-window quotient (c[k+w] - c[k]) / w is never formed: RN(x / w) is
// monotone in x, so `RN(x/w) >= theta` is exactly `x >= tau(theta)` for a
// host-precomputed double tau (and `== 1.0` an interval) — bit-identical counts,
// no DDIV.  HBM-bound: 9 algorithmic bytes per request (8 B reward + 1 B flags).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "be200.h"
#include "be_internal.h"

namespace be {

// Build-time tunables (measured on B200 at 65,536 envs x 10k, bench r1c): 2 warps x
// 2 stages x 8 CTAs/SM 1.20 ms; 4 x 3 x 4 1.26 ms; 2 x 3 x 8 1.24 ms; 4 x 2 x 4 1.22 ms.
// Measured and dropped (r2d, tools/probe_reduce.py): a cp.async.bulk.prefetch.L2 of
// each env's own row 4-16 chunks ahead (512 B-1 KB bursts) — 1.60-2.00 ms vs 1.21 ms.
constexpr int MAX_THETA = BE_MAX_THETA;
constexpr int NST = 2;       // pipeline stages (3 measured slower: shared memory, not latency)
constexpr int W = 20;        // evalkit.WINDOW
// Tile shapes (measured on B200 at 65,536 envs x 10k, tools/probe_reduce.py, r2):
//   CH = requests per stage (row burst CH x 8 bytes), NE = 32-env groups each warp
//   processes one after the other, WARPS per CTA, MINB = CTAs per SM the registers
//   are capped for.  The scan itself is ~5% of the time (a variant without the
//   threshold tests ran 1.17 vs 1.23 ms), a deeper pipeline did not help: DRAM row
//   locality of 65,536 interleaved row streams is the limit, so big batches halve the
//   streams and double the bursts:
//   16 / 1 / 2 / 8 -> 1.23 ms (74% of the copy peak); 32 / 2 / 2 / 4 -> 1.10-1.12;
//   32 / 2 / 4 / 2 -> 1.07 (84%); 32 / 2 / 7 / 1 -> 1.09; 32 / 3 / 2 / 3 -> 1.26;
//   64 / 4 / 2 / 2 -> 1.28 (the scan becomes the bound at 3.5 warps per SM).
struct RedShapeSmall { static constexpr int CH = 16, NE = 1, WARPS = 2, MINB = 8; };
struct RedShapeBig { static constexpr int CH = 32, NE = 2, WARPS = 4, MINB = 2; };

struct ReduceParams {
    int32_t E;
    int64_t ld;
    const double* reward;
    const uint8_t* flags;
    const int64_t* n_events;
    const int64_t* seg_off;
    const int64_t* seg_start;
    const int32_t* seg_bucket;
    int32_t n_buckets;
    int32_t exact_k;  // index of the theta == 1.0 threshold (interval test), -1 if none
    double lo[MAX_THETA];
    double hi;        // upper end of the theta == 1.0 interval
    int64_t* win_counts;
    int64_t* n_windows;
    int64_t* bucket_miss;
    int64_t* bucket_req;
    double* bucket_reward;
};

__device__ __forceinline__ void cp_async(void* smem, const void* gmem, int bytes, bool valid) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    int src_size = valid ? bytes : 0;  // 0 -> zero-fill
    if (bytes == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_size));
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_size));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

struct Acc {
    double c;         // running prefix sum
    double ring[32];  // ring[j] = prefix sum after request (32 m + j)
    double c_bucket;  // prefix sum when the current bucket started
    int miss, req;    // current bucket
};

// cnt[k] counts windows with d >= lo[k]; the theta == 1.0 interval [lo, hi] is
// #(d >= lo) - #(d > hi), so the exact test costs one extra compare (cnt[NT])
// and no per-threshold select; the subtraction happens once at the end.
#ifndef RED_NOSCAN
#define RED_NOSCAN 0  // measurement aid: 1 = skip the window tests (memory-pattern bound of the kernel)
#endif
template <int NT>
__device__ __forceinline__ void count_window(const ReduceParams& p, int (&cnt)[NT + 1], double d) {
    if (RED_NOSCAN) {
        cnt[0] += d > 1e300 ? 1 : 0;  // keep d live
        return;
    }
#pragma unroll
    for (int k = 0; k < NT; ++k) cnt[k] += d >= p.lo[k] ? 1 : 0;
    cnt[NT] += d > p.hi ? 1 : 0;
}

__device__ __forceinline__ void flush_bucket(const ReduceParams& p, Acc& a, int64_t env, int bucket) {
    if (a.req) {
        const int64_t o = env * p.n_buckets + bucket;
        p.bucket_miss[o] += a.miss;
        p.bucket_req[o] += a.req;
        p.bucket_reward[o] = __dadd_rn(p.bucket_reward[o], __dsub_rn(a.c, a.c_bucket));
    }
    a.miss = a.req = 0;
    a.c_bucket = a.c;
}

// General path: ragged tails, the first windows, segment boundaries.
template <int NT, int OFF, int CH, int NFW = CH / 16>
__device__ __forceinline__ void scan_chunk_slow(const ReduceParams& p, Acc& a, int (&cnt)[NT + 1],
                                                const double* row, const uint4 (&fl)[NFW], int64_t i0, int64_t n,
                                                int64_t& next_seg, int64_t& seg, int64_t seg_end,
                                                int& bucket, int64_t env) {
    uint32_t fw[4 * NFW];
#pragma unroll
    for (int q = 0; q < NFW; ++q) {
        fw[4 * q] = fl[q].x;
        fw[4 * q + 1] = fl[q].y;
        fw[4 * q + 2] = fl[q].z;
        fw[4 * q + 3] = fl[q].w;
    }
#pragma unroll
    for (int s = 0; s < CH; ++s) {
        const int64_t i = i0 + s;
        if (i < n) {
            while (i >= next_seg) {  // segment boundary
                flush_bucket(p, a, env, bucket);
                bucket = p.seg_bucket ? p.seg_bucket[seg] : 0;
                ++seg;
                next_seg = seg < seg_end ? p.seg_start[seg] : INT64_MAX;
            }
            a.c = __dadd_rn(a.c, row[s]);
            const double prev = a.ring[(OFF + s - W + 64) & 31];  // prefix sum W requests back
            a.ring[(OFF + s) & 31] = a.c;
            if (i >= W - 1) count_window<NT>(p, cnt, __dsub_rn(a.c, prev));
            a.miss += (fw[s >> 2] >> (8 * (s & 3) + 7)) & 1u;
            a.req += 1;
        }
    }
}

// Steady state: whole chunk valid, windows complete, no boundary inside.
template <int NT, int OFF, int CH, int NFW = CH / 16>
__device__ __forceinline__ void scan_chunk_fast(const ReduceParams& p, Acc& a, int (&cnt)[NT + 1],
                                                const double* row, const uint4 (&fl)[NFW]) {
#pragma unroll
    for (int s = 0; s < CH; ++s) {
        a.c = __dadd_rn(a.c, row[s]);
        const double prev = a.ring[(OFF + s - W + 64) & 31];
        a.ring[(OFF + s) & 31] = a.c;
        count_window<NT>(p, cnt, __dsub_rn(a.c, prev));
    }
#pragma unroll
    for (int q = 0; q < NFW; ++q)
        a.miss += __popc(fl[q].x & 0x80808080u) + __popc(fl[q].y & 0x80808080u) +
                  __popc(fl[q].z & 0x80808080u) + __popc(fl[q].w & 0x80808080u);
    a.req += CH;
}

template <class S>
constexpr size_t red_smem_bytes() {
    return sizeof(double) * S::WARPS * NST * 32 * (S::CH + 2) + sizeof(int64_t) * S::WARPS * 32 +
           sizeof(uint4) * S::WARPS * NST * 32 * (S::CH / 16);
}

template <int NT, class S>
__global__ void __launch_bounds__(S::WARPS * 32, S::MINB) reduce_kernel(const ReduceParams p) {
    constexpr int CH = S::CH, NE = S::NE, RED_WARPS = S::WARPS, NFW = CH / 16, TSTRIDE = CH + 2;
    static_assert(CH == 16 || CH == 32 || CH == 64, "CH must be 16, 32 or 64");
    extern __shared__ __align__(16) double red_smem[];
    typedef double TileT[NST][32][TSTRIDE];
    TileT* tile = reinterpret_cast<TileT*>(red_smem);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int64_t* n_row = reinterpret_cast<int64_t*>(red_smem + RED_WARPS * NST * 32 * TSTRIDE) + warp * 32;
    typedef uint4 FlT[NST][32][NFW];
    FlT* fl_tile = reinterpret_cast<FlT*>(reinterpret_cast<int64_t*>(red_smem + RED_WARPS * NST * 32 * TSTRIDE) +
                                          RED_WARPS * 32);
    const int64_t n_groups = (p.E + 31) / 32;
    for (int pass = 0; pass < NE; ++pass) {
    const int64_t g = ((int64_t)blockIdx.x * RED_WARPS + warp) * NE + pass;
    if (g >= n_groups) return;
    const int64_t e0 = g * 32;
    const int64_t env = e0 + lane;
    const bool live = env < p.E;
    const int64_t n = live ? (p.n_events ? p.n_events[env] : p.ld) : 0;
    int64_t nmax = n, nmin = live ? n : INT64_MAX;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        int64_t o = __shfl_xor_sync(0xffffffffu, nmax, off);
        nmax = o > nmax ? o : nmax;
        o = __shfl_xor_sync(0xffffffffu, nmin, off);
        nmin = o < nmin ? o : nmin;
    }
    const bool full_group = e0 + 32 <= p.E;
    const int64_t nchunks = (nmax + CH - 1) / CH;
    __syncwarp();  // the previous pass's readers of n_row are done
    n_row[lane] = live ? n : -1;
    __syncwarp();
    // staging, 16-byte copies: LPR = CH / 2 lanes per row (CH * 8 contiguous bytes),
    // RPI = 32 / LPR rows per instruction; CH = 64: a row per instruction, 2 copies per lane
    constexpr int LPR = CH / 2 < 32 ? CH / 2 : 32, RPI = 32 / LPR, CPL = CH / 2 / LPR;
    const bool vec16 = ((reinterpret_cast<uintptr_t>(p.reward) | (uintptr_t)(p.ld * 8)) & 15) == 0;
    const int q4 = lane / LPR, c4 = (lane % LPR) * 2;
    const double* src16 = p.reward + (e0 + q4) * p.ld + c4;  // + k * RPI * ld + i0
    const int64_t step16 = RPI * p.ld;

    const bool fl_vec = ((reinterpret_cast<uintptr_t>(p.flags) | (uintptr_t)p.ld) & 15) == 0;
    const uint8_t* fsrc = p.flags + (live ? env * p.ld : 0);
    auto issue = [&](int64_t ch) {
        if (ch < nchunks) {
            const int st = (int)(ch % NST);
            const int64_t i0 = ch * CH;
            // own row of flags (CH bytes) rides in the same cp.async group
            if (fl_vec) {
#pragma unroll
                for (int q = 0; q < NFW; ++q)
                    cp_async(&fl_tile[warp][st][lane][q], fsrc + i0 + 16 * q, 16, live && i0 + CH <= n);
            }
            if (vec16 && full_group && i0 + CH <= nmin) {  // every row complete
                const double* s = src16 + i0;
#pragma unroll
                for (int k = 0; k < 32 / RPI; ++k) {
#pragma unroll
                    for (int c = 0; c < CPL; ++c)
                        cp_async(&tile[warp][st][RPI * k + q4][c4 + 2 * LPR * c], s + 2 * LPR * c, 16, true);
                    s += step16;
                }
            } else {  // ragged group: 8-byte copies, element lane + 32 k of the [32][CH] tile
#pragma unroll
                for (int k = 0; k < CH; ++k) {
                    const int idx = lane + 32 * k, r = idx / CH, c = idx % CH;
                    const int64_t i = i0 + c;
                    const bool v = i < n_row[r];
                    const double* s = p.reward + (v ? (e0 + r) * p.ld + i : 0);
                    cp_async(&tile[warp][st][r][c], s, 8, v);
                }
            }
        }
        cp_commit();  // uniform group accounting (possibly empty)
    };

    int64_t seg = live ? p.seg_off[env] : 0;
    const int64_t seg_end = live ? p.seg_off[env + 1] : 0;
    int bucket = 0;
    int64_t next_seg = seg < seg_end ? p.seg_start[seg] : INT64_MAX;
    if (live)
        for (int b = 0; b < p.n_buckets; ++b) {
            p.bucket_miss[env * p.n_buckets + b] = 0;
            p.bucket_req[env * p.n_buckets + b] = 0;
            p.bucket_reward[env * p.n_buckets + b] = 0.0;
        }
    Acc a;
    a.c = 0.0;
    a.c_bucket = 0.0;
    a.miss = a.req = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) a.ring[j] = 0.0;
    int cnt[NT + 1];
#pragma unroll
    for (int k = 0; k <= NT; ++k) cnt[k] = 0;

    const uint8_t* frow = p.flags + (live ? env * p.ld : 0);
    auto load_flags = [&](int64_t ch, uint4 (&f)[NFW]) {
#pragma unroll
        for (int q = 0; q < NFW; ++q) f[q] = make_uint4(0, 0, 0, 0);
        const int64_t i0 = ch * CH;
        if (live && i0 < n) {
            if (fl_vec && i0 + CH <= n) {
#pragma unroll
                for (int q = 0; q < NFW; ++q) f[q] = fl_tile[warp][ch % NST][lane][q];  // staged by issue()
            } else {
                uint32_t w[4 * NFW];
#pragma unroll
                for (int q = 0; q < 4 * NFW; ++q) w[q] = 0;
                for (int k = 0; k < CH && i0 + k < n; ++k) {
                    const uint32_t b = (uint32_t)frow[i0 + k] << (8 * (k & 3));
#pragma unroll
                    for (int q = 0; q < 4 * NFW; ++q)
                        if ((k >> 2) == q) w[q] |= b;
                }
#pragma unroll
                for (int q = 0; q < NFW; ++q) f[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
            }
        }
    };

#pragma unroll
    for (int s = 0; s < NST - 1; ++s) issue(s);
    for (int64_t ch = 0; ch < nchunks; ++ch) {
        issue(ch + NST - 1);
        cp_wait<NST - 1>();
        __syncwarp();
        uint4 fl[NFW];
        load_flags(ch, fl);
        const double* row = &tile[warp][ch % NST][lane][0];
        const int64_t i0 = ch * CH;
        const bool fast = i0 >= 32 && i0 + CH <= n && next_seg >= i0 + CH;
        if (CH == 16 && (ch & 1)) {  // the 32-entry prefix ring: chunk halves alternate
            if (fast) scan_chunk_fast<NT, (CH == 16 ? 16 : 0), CH>(p, a, cnt, row, fl);
            else scan_chunk_slow<NT, (CH == 16 ? 16 : 0), CH>(p, a, cnt, row, fl, i0, n, next_seg, seg, seg_end, bucket, env);
        } else {
            if (fast) scan_chunk_fast<NT, 0, CH>(p, a, cnt, row, fl);
            else scan_chunk_slow<NT, 0, CH>(p, a, cnt, row, fl, i0, n, next_seg, seg, seg_end, bucket, env);
        }
        __syncwarp();  // stage ch % NST is refilled by the next iteration's issue
    }
    cp_wait<0>();
    if (live) {
        flush_bucket(p, a, env, bucket);
#pragma unroll
        for (int k = 0; k < NT; ++k) p.win_counts[env * NT + k] = cnt[k] - (k == p.exact_k ? cnt[NT] : 0);
        p.n_windows[env] = n >= W ? n - W + 1 : 0;
    }
    }  // pass
}

// smallest double x with RN(x / w) >= theta (x >= 0 domain; -inf if all qualify)
double tau_ge(double theta, double w) {
    if (0.0 / w >= theta) return -INFINITY;
    // binary search over the bit patterns of non-negative doubles
    uint64_t lo = 0, hi = 0x7ff0000000000000ULL;  // +inf qualifies (inf/w = inf)
    while (hi - lo > 1) {
        uint64_t mid = lo + (hi - lo) / 2;
        double x;
        memcpy(&x, &mid, 8);
        if (x / w >= theta) hi = mid;
        else lo = mid;
    }
    double x;
    memcpy(&x, &hi, 8);
    return x;
}

// largest double x with RN(x / w) <= theta
double tau_le(double theta, double w) {
    uint64_t lo = 0, hi = 0x7ff0000000000000ULL;
    double x0 = 0.0;
    if (!(x0 / w <= theta)) return -INFINITY;
    while (hi - lo > 1) {
        uint64_t mid = lo + (hi - lo) / 2;
        double x;
        memcpy(&x, &mid, 8);
        if (x / w <= theta) lo = mid;
        else hi = mid;
    }
    double x;
    memcpy(&x, &lo, 8);
    return x;
}

template <int NT, class S>
static int launch_shape(const ReduceParams& p, cudaStream_t st) {
    const int64_t groups = (p.E + 31) / 32;
    const int64_t warps = (groups + S::NE - 1) / S::NE;
    const int blocks = (int)((warps + S::WARPS - 1) / S::WARPS);
    constexpr size_t smem = red_smem_bytes<S>();
    static bool configured = false;  // one flag per (NT, shape) instantiation
    if (!configured) {
        cudaFuncSetAttribute(reduce_kernel<NT, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = true;
    }
    reduce_kernel<NT, S><<<blocks, S::WARPS * 32, smem, st>>>(p);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "reduce launch");
}

// big batches: halve the row streams, double the bursts (every warp of the grid still
// resident: 2 groups per warp, 4 warps per CTA, 2 CTAs per SM); small batches keep one
// group per warp so more SMs share the work
template <int NT>
static int launch_nt(const ReduceParams& p, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t groups = (p.E + 31) / 32;
    if (groups >= (int64_t)sms * RedShapeBig::WARPS * RedShapeBig::NE)  // at least a CTA per SM
        return launch_shape<NT, RedShapeBig>(p, st);
    return launch_shape<NT, RedShapeSmall>(p, st);
}

int launch_reduce(const be_trace_soa* tr, const uint8_t* flags, const double* reward, int window,
                  const double* thetas, int n_theta, int n_buckets, int64_t* win_counts,
                  int64_t* n_windows, int64_t* bucket_miss, int64_t* bucket_req,
                  double* bucket_reward, cudaStream_t st) {
    if (window != W) return set_error(BE_EINVAL, "reducer window must be 20 (evalkit.WINDOW)");
    if (n_theta < 1 || n_theta > MAX_THETA) return set_error(BE_EINVAL, "n_theta must be in [1, 8]");
    ReduceParams p{};
    p.E = tr->n_envs;
    p.ld = tr->ld;
    p.reward = reward;
    p.flags = flags;
    p.n_events = tr->n_events;
    p.seg_off = tr->seg_offsets;
    p.seg_start = tr->seg_start;
    p.seg_bucket = tr->seg_bucket;
    p.n_buckets = n_buckets;
    p.exact_k = -1;
    p.hi = INFINITY;
    const double w = (double)window;
    for (int k = 0; k < MAX_THETA; ++k) p.lo[k] = INFINITY;
    for (int k = 0; k < n_theta; ++k) {
        double th = thetas[k];
        if (!(th >= 0.0 && th <= 1.0)) return set_error(BE_EINVAL, "thresholds must lie in [0, 1]");
        p.lo[k] = tau_ge(th, w);
        if (th == 1.0) {
            // theta == 1.0 counts exact peak windows only (evalkit.py:237-238)
            if (p.exact_k >= 0) return set_error(BE_EINVAL, "threshold 1.0 given twice");
            p.exact_k = k;
            p.hi = tau_le(1.0, w);
        }
    }
    p.win_counts = win_counts;
    p.n_windows = n_windows;
    p.bucket_miss = bucket_miss;
    p.bucket_req = bucket_req;
    p.bucket_reward = bucket_reward;
    switch (n_theta) {
        case 1: return launch_nt<1>(p, st);
        case 2: return launch_nt<2>(p, st);
        case 3: return launch_nt<3>(p, st);
        case 4: return launch_nt<4>(p, st);
        case 5: return launch_nt<5>(p, st);
        case 6: return launch_nt<6>(p, st);
        case 7: return launch_nt<7>(p, st);
        default: return launch_nt<8>(p, st);
    }
}

}  // namespace be
