// reduce.cu — on-device evaluation reducer (K5).
//
//   windowed(rewards, 20) + threshold_counts   evalkit.py:217-241
//   miss fraction by segment rate              evalkit.py:61-68
//   mean reward by segment rate                evalkit.py:70-74
//
// One thread per environment owns the strictly sequential fp64 prefix sum
// c_{k+1} = c_k + r_k (np.cumsum order — any parallel scan would change the
// rounding and therefore the threshold counts).  Rewards
// are env-major in HBM, so each warp streams a 32-env x 16-request tile per
// stage with cp.async (16-byte LDGSTS, every env row a fully used 128-byte
// segment) into padded shared memory, NST stages deep, while the lanes scan
// an earlier stage row by row.  The trailing-window quotient
// (c[k+w] - c[k]) / w is never formed: RN(x / w) is monotone in x, so
// `RN(x/w) >= theta` is exactly `x >= tau(theta)` for a host-precomputed
// double tau (and `== 1.0` an interval) — bit-identical counts, no DDIV.
// HBM-bound: 9 algorithmic bytes per request (8 B reward + 1 B flags).
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
#ifndef RED_W
#define RED_W 2
#endif
#ifndef RED_NST
#define RED_NST 2
#endif
#ifndef RED_MINB
#define RED_MINB 8
#endif
constexpr int RED_WARPS = RED_W;
constexpr int MAX_THETA = BE_MAX_THETA;
constexpr int CH = 16;       // requests per stage
constexpr int NST = RED_NST;  // pipeline stages
constexpr int W = 20;        // evalkit.WINDOW
constexpr int TSTRIDE = 18;  // padded tile row (doubles): 16-byte aligned rows

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
template <int NT>
__device__ __forceinline__ void count_window(const ReduceParams& p, int (&cnt)[NT + 1], double d) {
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
template <int NT, int OFF>
__device__ __forceinline__ void scan_chunk_slow(const ReduceParams& p, Acc& a, int (&cnt)[NT + 1],
                                                const double* row, uint4 fl, int64_t i0, int64_t n,
                                                int64_t& next_seg, int64_t& seg, int64_t seg_end,
                                                int& bucket, int64_t env) {
    const uint32_t fw[4] = {fl.x, fl.y, fl.z, fl.w};
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
            a.ring[OFF + s] = a.c;
            if (i >= W - 1) count_window<NT>(p, cnt, __dsub_rn(a.c, prev));
            a.miss += (fw[s >> 2] >> (8 * (s & 3) + 7)) & 1u;
            a.req += 1;
        }
    }
}

// Steady state: whole chunk valid, windows complete, no boundary inside.
template <int NT, int OFF>
__device__ __forceinline__ void scan_chunk_fast(const ReduceParams& p, Acc& a, int (&cnt)[NT + 1],
                                                const double* row, uint4 fl) {
#pragma unroll
    for (int s = 0; s < CH; ++s) {
        a.c = __dadd_rn(a.c, row[s]);
        const double prev = a.ring[(OFF + s - W + 64) & 31];
        a.ring[OFF + s] = a.c;
        count_window<NT>(p, cnt, __dsub_rn(a.c, prev));
    }
    a.miss += __popc(fl.x & 0x80808080u) + __popc(fl.y & 0x80808080u) +
              __popc(fl.z & 0x80808080u) + __popc(fl.w & 0x80808080u);
    a.req += CH;
}

template <int NT>
__global__ void __launch_bounds__(RED_WARPS * 32, RED_MINB) reduce_kernel(const ReduceParams p) {
    extern __shared__ __align__(16) double red_smem[];
    typedef double TileT[NST][32][TSTRIDE];
    TileT* tile = reinterpret_cast<TileT*>(red_smem);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int64_t* n_row = reinterpret_cast<int64_t*>(red_smem + RED_WARPS * NST * 32 * TSTRIDE) + warp * 32;
    typedef uint4 FlT[NST][32];
    FlT* fl_tile = reinterpret_cast<FlT*>(reinterpret_cast<int64_t*>(red_smem + RED_WARPS * NST * 32 * TSTRIDE) +
                                          RED_WARPS * 32);
    const int64_t n_groups = (p.E + 31) / 32;
    const int64_t g = (int64_t)blockIdx.x * RED_WARPS + warp;
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
    n_row[lane] = live ? n : -1;
    __syncwarp();
    // staging, 16-byte copies: lanes 8q..8q+7 copy row 4k+q (128 contiguous bytes)
    const bool vec16 = ((reinterpret_cast<uintptr_t>(p.reward) | (uintptr_t)(p.ld * 8)) & 15) == 0;
    const int q4 = lane >> 3, c4 = (lane & 7) * 2;
    const double* src16 = p.reward + (e0 + q4) * p.ld + c4;  // + k * 4 * ld + i0
    const int64_t step16 = 4 * p.ld;
    const int half = lane >> 4, col = lane & 15;
    const bool fl_vec = ((reinterpret_cast<uintptr_t>(p.flags) | (uintptr_t)p.ld) & 15) == 0;
    const uint8_t* fsrc = p.flags + (live ? env * p.ld : 0);
    auto issue = [&](int64_t ch) {
        if (ch < nchunks) {
            const int st = (int)(ch % NST);
            const int64_t i0 = ch * CH;
            // own row of flags (16 bytes) rides in the same cp.async group
            if (fl_vec) cp_async(&fl_tile[warp][st][lane], fsrc + i0, 16, live && i0 + CH <= n);
            if (vec16 && full_group && i0 + CH <= nmin) {  // every row complete
                const double* s = src16 + i0;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    cp_async(&tile[warp][st][4 * k + q4][c4], s, 16, true);
                    s += step16;
                }
            } else {
                const int64_t i = i0 + col;
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const int r = 2 * k + half;
                    const bool v = i < n_row[r];
                    const double* s = p.reward + (v ? (e0 + r) * p.ld + i : 0);
                    cp_async(&tile[warp][st][r][col], s, 8, v);
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
    auto load_flags = [&](int64_t ch) {
        uint4 f = make_uint4(0, 0, 0, 0);
        const int64_t i0 = ch * CH;
        if (live && i0 < n) {
            if (fl_vec && i0 + CH <= n) {
                f = fl_tile[warp][ch % NST][lane];  // staged by issue() with the rewards
            } else {
                uint32_t w0 = 0, w1 = 0, w2 = 0, w3 = 0;
                for (int k = 0; k < CH && i0 + k < n; ++k) {
                    const uint32_t b = (uint32_t)frow[i0 + k] << (8 * (k & 3));
                    if (k < 4) w0 |= b; else if (k < 8) w1 |= b; else if (k < 12) w2 |= b; else w3 |= b;
                }
                f = make_uint4(w0, w1, w2, w3);
            }
        }
        return f;
    };

#pragma unroll
    for (int s = 0; s < NST - 1; ++s) issue(s);
    for (int64_t ch = 0; ch < nchunks; ++ch) {
        issue(ch + NST - 1);
        cp_wait<NST - 1>();
        __syncwarp();
        const uint4 fl = load_flags(ch);
        const double* row = &tile[warp][ch % NST][lane][0];
        const int64_t i0 = ch * CH;
        const bool fast = i0 >= 32 && i0 + CH <= n && next_seg >= i0 + CH;
        if (ch & 1) {
            if (fast) scan_chunk_fast<NT, 16>(p, a, cnt, row, fl);
            else scan_chunk_slow<NT, 16>(p, a, cnt, row, fl, i0, n, next_seg, seg, seg_end, bucket, env);
        } else {
            if (fast) scan_chunk_fast<NT, 0>(p, a, cnt, row, fl);
            else scan_chunk_slow<NT, 0>(p, a, cnt, row, fl, i0, n, next_seg, seg, seg_end, bucket, env);
        }
        __syncwarp();  // stage ch % NST is refilled by the next iteration's issue
    }
    cp_wait<0>();
    if (!live) return;
    flush_bucket(p, a, env, bucket);
#pragma unroll
    for (int k = 0; k < NT; ++k) p.win_counts[env * NT + k] = cnt[k] - (k == p.exact_k ? cnt[NT] : 0);
    p.n_windows[env] = n >= W ? n - W + 1 : 0;
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

template <int NT>
static int launch_nt(const ReduceParams& p, cudaStream_t st) {
    int64_t groups = (p.E + 31) / 32;
    int blocks = (int)((groups + RED_WARPS - 1) / RED_WARPS);
    const size_t smem = sizeof(double) * RED_WARPS * NST * 32 * TSTRIDE + sizeof(int64_t) * RED_WARPS * 32 +
                        sizeof(uint4) * RED_WARPS * NST * 32;
    static bool configured[MAX_THETA + 1] = {false};
    if (!configured[NT]) {
        cudaFuncSetAttribute(reduce_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured[NT] = true;
    }
    reduce_kernel<NT><<<blocks, RED_WARPS * 32, smem, st>>>(p);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "reduce launch");
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
