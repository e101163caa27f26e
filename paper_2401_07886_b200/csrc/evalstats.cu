// evalstats.cu — secondary evaluation reducers on the device.
//
//   selection_distribution counts  evalkit.py:244-262 -> be_reduce_selection
//   windowed series                 evalkit.py:217-226 -> be_windowed
//
// be_reduce_selection: one warp per environment walks its requests 32 at a
// time (coalesced task / flag bytes), finds each request's segment (segments
// are sorted, so a lane only moves forward from the warp's current segment),
// and counts (task, rate bucket, tier) in a shared-memory histogram that is
// added to the global int64 counts once per CTA.  Integer counts: the result
// is exact and independent of the order of the atomics.
//
// be_windowed: the trailing-window means themselves, (c[k+w] - c[k]) / w with
// c the sequential fp64 prefix sum (np.cumsum order) — bit-identical to the
// reference series (used for trial_band, evalkit.py:280-288).
#include <cuda_runtime.h>
#include <stdint.h>

#include "be200.h"
#include "be_internal.h"

namespace be {

constexpr int SEL_THREADS = 256;

__global__ void __launch_bounds__(SEL_THREADS) selection_kernel(
    int E, int64_t ld, const uint8_t* __restrict__ task, const uint8_t* __restrict__ flags,
    const int64_t* __restrict__ n_events, const int64_t* __restrict__ seg_off,
    const int64_t* __restrict__ seg_start, const int32_t* __restrict__ seg_bucket, int T, int K,
    int M, unsigned long long* counts, int use_smem) {
    extern __shared__ unsigned int hist[];
    const int nb = T * K * M;
    if (use_smem) {
        for (int k = threadIdx.x; k < nb; k += blockDim.x) hist[k] = 0u;
        __syncthreads();
    }
    const int lane = threadIdx.x & 31;
    const int warps = blockDim.x >> 5;
    for (int e = blockIdx.x * warps + (threadIdx.x >> 5); e < E; e += gridDim.x * warps) {
        const int64_t n = n_events ? n_events[e] : ld;
        const int64_t s_end = seg_off[e + 1];
        int64_t cur = seg_off[e];  // warp-uniform: segment of the chunk's first request
        for (int64_t i0 = 0; i0 < n; i0 += 32) {
            const int64_t i = i0 + lane;
            int64_t s = cur;
            while (s + 1 < s_end && seg_start[s + 1] <= i) ++s;
            if (i < n) {
                const int t = task[(int64_t)e * ld + i];
                const int m = flags[(int64_t)e * ld + i] & 0x3f;
                const int b = (seg_bucket && s < s_end) ? seg_bucket[s] : 0;
                if (t < T && m < M && b >= 0 && b < K) {
                    const int k = (t * K + b) * M + m;
                    if (use_smem) atomicAdd(&hist[k], 1u);
                    else atomicAdd(&counts[k], 1ull);
                }
            }
            cur = __shfl_sync(0xffffffffu, s, 31);
        }
    }
    if (use_smem) {
        __syncthreads();
        for (int k = threadIdx.x; k < nb; k += blockDim.x)
            if (hist[k]) atomicAdd(&counts[k], (unsigned long long)hist[k]);
    }
}

// One thread per env; out[e][k] for k in [0, n - w] (evalkit.py:225-226).
__global__ void windowed_kernel(int E, int64_t ld, const int64_t* __restrict__ n_events,
                                const double* __restrict__ reward, int w, double* out) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    const int64_t n = n_events ? n_events[e] : ld;
    const double* r = reward + (int64_t)e * ld;
    double* o = out + (int64_t)e * ld;
    // ring of the last w + 1 prefix sums is avoided: c[k] is recomputed by
    // keeping a second running sum that trails by w requests (same adds, same
    // order, so the same bits as np.cumsum)
    double c = 0.0, c_lag = 0.0;
    const double wd = (double)w;
    for (int64_t i = 0; i < n; ++i) {
        c = __dadd_rn(c, r[i]);
        if (i >= w - 1) {
            o[i - (w - 1)] = __ddiv_rn(__dsub_rn(c, c_lag), wd);
            c_lag = __dadd_rn(c_lag, r[i - (w - 1)]);
        }
    }
}

int launch_selection(const be_trace_soa* tr, const uint8_t* flags, int T, int M, int K,
                     int64_t* counts, cudaStream_t st) {
    const size_t smem = sizeof(unsigned) * (size_t)T * K * M;
    const int use_smem = smem <= 48 * 1024;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int warps = SEL_THREADS / 32;
    long long blocks = ((long long)tr->n_envs + warps - 1) / warps;
    if (blocks > (long long)sms * 8) blocks = (long long)sms * 8;
    selection_kernel<<<(unsigned)blocks, SEL_THREADS, use_smem ? smem : 0, st>>>(
        tr->n_envs, tr->ld, tr->task, flags, tr->n_events, tr->seg_offsets, tr->seg_start,
        tr->seg_bucket, T, K, M, reinterpret_cast<unsigned long long*>(counts), use_smem);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "selection launch");
}

int launch_windowed(const be_trace_soa* tr, const double* reward, int w, double* out, cudaStream_t st) {
    windowed_kernel<<<(tr->n_envs + 127) / 128, 128, 0, st>>>(tr->n_envs, tr->ld, tr->n_events, reward, w,
                                                               out);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "windowed launch");
}

}  // namespace be

using namespace be;

extern "C" {

int32_t be_reduce_selection(const be_trace_soa* trace, const uint8_t* flags, int32_t n_tasks,
                            int32_t n_tiers, int32_t n_buckets, int64_t* counts, void* stream) {
    if (!trace || !flags || !counts || !trace->task || !trace->seg_offsets)
        return set_error(BE_EINVAL, "NULL argument");
    if (n_tasks < 1 || n_tasks > 255 || n_tiers < 1 || n_tiers > BE_MAX_TIERS || n_buckets < 1)
        return set_error(BE_EINVAL, "bad sizes");
    return launch_selection(trace, flags, n_tasks, n_tiers, n_buckets, counts, (cudaStream_t)stream);
}

int32_t be_windowed(const be_trace_soa* trace, const double* reward, int32_t window, double* out,
                    void* stream) {
    if (!trace || !reward || !out) return set_error(BE_EINVAL, "NULL argument");
    if (window < 1) return set_error(BE_EINVAL, "window must be >= 1");
    return launch_windowed(trace, reward, window, out, (cudaStream_t)stream);
}

}  // extern "C"
