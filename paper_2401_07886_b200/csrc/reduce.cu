// reduce.cu — on-device evaluation reducer (K5).
//
//   windowed(rewards, 20) + threshold_counts   evalkit.py:217-241
//   miss fraction by segment rate              evalkit.py:61-68
//   mean reward by segment rate                evalkit.py:70-74
//
// One thread per environment owns the strictly sequential fp64 prefix sum
// c_{k+1} = c_k + r_k (np.cumsum order — any parallel scan would change the
// rounding and therefore the threshold counts).  Rewards
// are env-major in HBM, so each warp stages a 32-env x 32-request tile with
// fully coalesced row loads (each row = 256 contiguous bytes) into padded
// shared memory, and every lane then scans its own row from there.  The
// trailing-window quotient (c[k+w] - c[k]) / w is never formed: because
// RN(x / w) is monotone in x, `RN(x/w) >= theta` is exactly `x >= tau(theta)`
// for a host-precomputed double tau (and `== 1.0` an interval), so the
// kernel compares differences directly — bit-identical counts, no DDIV.
// HBM-bound: 9 algorithmic bytes per request (8 B reward + 1 B flags).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "be200.h"
#include "be_internal.h"

namespace be {

constexpr int RED_WARPS = 4;
constexpr int MAX_THETA = 16;

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
    int32_t n_theta;
    double lo[MAX_THETA];
    double hi[MAX_THETA];
    int64_t* win_counts;
    int64_t* n_windows;
    int64_t* bucket_miss;
    int64_t* bucket_req;
    double* bucket_reward;
};

// W = window (template so the 32-slot prefix ring stays in registers).
template <int W>
__global__ void __launch_bounds__(RED_WARPS * 32) reduce_kernel(const ReduceParams p) {
    __shared__ double tile[RED_WARPS][32][33];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t e0 = ((int64_t)blockIdx.x * RED_WARPS + warp) * 32;
    if (e0 >= p.E) return;
    const int64_t env = e0 + lane;
    const bool live = env < p.E;
    const int64_t n = live ? (p.n_events ? p.n_events[env] : p.ld) : 0;
    int64_t nmax = n;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        int64_t o = __shfl_xor_sync(0xffffffffu, nmax, off);
        nmax = o > nmax ? o : nmax;
    }
    // segment cursor -> bucket
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
    int64_t acc_miss = 0, acc_req = 0;
    double acc_rw = 0.0;
    int64_t cnt[MAX_THETA];
#pragma unroll
    for (int k = 0; k < MAX_THETA; ++k) cnt[k] = 0;
    double lo[MAX_THETA], hi[MAX_THETA];
#pragma unroll
    for (int k = 0; k < MAX_THETA; ++k) {
        lo[k] = p.lo[k];
        hi[k] = p.hi[k];
    }
    double ring[32];  // ring[s] = prefix sum after request (chunk*32 + s)
#pragma unroll
    for (int s = 0; s < 32; ++s) ring[s] = 0.0;
    double c = 0.0;
    const double* rrow = p.reward;
    for (int64_t i0 = 0; i0 < nmax; i0 += 32) {
        // coalesced staging: row r of the tile = env e0 + r, requests i0..i0+31
        for (int r = 0; r < 32; ++r) {
            int64_t nr = __shfl_sync(0xffffffffu, n, r);
            double v = 0.0;
            if (e0 + r < p.E && i0 + lane < nr) v = rrow[(e0 + r) * p.ld + i0 + lane];
            tile[warp][r][lane] = v;
        }
        __syncwarp();
        // own row of flags: 32 bytes
        uint32_t fw[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) fw[k] = 0;
        if (live && i0 < n) {
            const uint8_t* fr = p.flags + env * p.ld + i0;
            if (((reinterpret_cast<uintptr_t>(fr) & 15) == 0) && i0 + 32 <= n) {
                uint4 a = *reinterpret_cast<const uint4*>(fr);
                uint4 b = *reinterpret_cast<const uint4*>(fr + 16);
                fw[0] = a.x; fw[1] = a.y; fw[2] = a.z; fw[3] = a.w;
                fw[4] = b.x; fw[5] = b.y; fw[6] = b.z; fw[7] = b.w;
            } else {
                for (int k = 0; k < 32 && i0 + k < n; ++k) fw[k >> 2] |= (uint32_t)fr[k] << (8 * (k & 3));
            }
        }
#pragma unroll
        for (int s = 0; s < 32; ++s) {
            const int64_t i = i0 + s;
            if (i < n) {
                while (i >= next_seg) {  // segment boundary: flush the bucket partials
                    if (acc_req) {
                        p.bucket_miss[env * p.n_buckets + bucket] += acc_miss;
                        p.bucket_req[env * p.n_buckets + bucket] += acc_req;
                        p.bucket_reward[env * p.n_buckets + bucket] = __dadd_rn(p.bucket_reward[env * p.n_buckets + bucket], acc_rw);
                    }
                    acc_miss = acc_req = 0;
                    acc_rw = 0.0;
                    bucket = p.seg_bucket ? p.seg_bucket[seg] : 0;
                    ++seg;
                    next_seg = seg < seg_end ? p.seg_start[seg] : INT64_MAX;
                }
                const double r = tile[warp][lane][s];
                c = __dadd_rn(c, r);
                const double prev = ring[(s - W + 64) & 31];  // prefix sum W requests back
                ring[s] = c;
                if (i >= W - 1) {
                    const double d = __dsub_rn(c, prev);
#pragma unroll
                    for (int k = 0; k < MAX_THETA; ++k)
                        if (k < p.n_theta) cnt[k] += (d >= lo[k] && d <= hi[k]) ? 1 : 0;
                }
                const uint32_t f = (fw[s >> 2] >> (8 * (s & 3))) & 0xffu;
                acc_miss += (f >> 7) & 1u;
                acc_req += 1;
                acc_rw = __dadd_rn(acc_rw, r);
            }
        }
        __syncwarp();
    }
    if (!live) return;
    if (acc_req) {
        p.bucket_miss[env * p.n_buckets + bucket] += acc_miss;
        p.bucket_req[env * p.n_buckets + bucket] += acc_req;
        p.bucket_reward[env * p.n_buckets + bucket] = __dadd_rn(p.bucket_reward[env * p.n_buckets + bucket], acc_rw);
    }
    for (int k = 0; k < p.n_theta; ++k) p.win_counts[env * p.n_theta + k] = cnt[k];
    p.n_windows[env] = n >= W ? n - W + 1 : 0;
}

// smallest double x with RN(x / w) >= theta (x >= 0 domain; -inf if all qualify)
static double tau_ge(double theta, double w) {
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
static double tau_le(double theta, double w) {
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

int launch_reduce(const be_trace_soa* tr, const uint8_t* flags, const double* reward, int window,
                  const double* thetas, int n_theta, int n_buckets, int64_t* win_counts,
                  int64_t* n_windows, int64_t* bucket_miss, int64_t* bucket_req,
                  double* bucket_reward, cudaStream_t st) {
    if (window != 20) return set_error(BE_EINVAL, "reducer window must be 20 (evalkit.WINDOW)");
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
    p.n_theta = n_theta;
    const double w = (double)window;
    for (int k = 0; k < MAX_THETA; ++k) {
        p.lo[k] = INFINITY;
        p.hi[k] = -INFINITY;
    }
    for (int k = 0; k < n_theta; ++k) {
        double th = thetas[k];
        if (!(th >= 0.0 && th <= 1.0)) return set_error(BE_EINVAL, "thresholds must lie in [0, 1]");
        p.lo[k] = tau_ge(th, w);
        // theta == 1.0 counts exact peak windows only (evalkit.py:237-238)
        p.hi[k] = th == 1.0 ? tau_le(1.0, w) : INFINITY;
    }
    p.win_counts = win_counts;
    p.n_windows = n_windows;
    p.bucket_miss = bucket_miss;
    p.bucket_req = bucket_req;
    p.bucket_reward = bucket_reward;
    int64_t warps = (p.E + 31) / 32;
    int blocks = (int)((warps + RED_WARPS - 1) / RED_WARPS);
    reduce_kernel<20><<<blocks, RED_WARPS * 32, 0, st>>>(p);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "reduce launch");
}

}  // namespace be
