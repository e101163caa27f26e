// be_route.cuh — the fp64 router arithmetic of be_qnet_route_f64
// (QNetwork.forward + argmax, policy.py:111-132) for one state per warp.
// Shared by route_kernel and the tensor-core router's fallback so both give
// the same bits: lane l owns hidden units l + 32k; layer 1 is the dense
// x @ W1 in input order, then + b1; layer 2 accumulates over j in increasing
// order per lane, then a warp butterfly.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace be {

// xv: lane d (< D) holds x[d].  W2 element (j, m) at w2[j * w2_sj + m * w2_sm].
template <int M>
__device__ __forceinline__ void route_row_f64(double xv, int D, int H, const double* __restrict__ w1,
                                              const double* __restrict__ b1, const double* __restrict__ w2,
                                              int w2_sj, int w2_sm, const double* __restrict__ b2,
                                              double (&q)[M]) {
    const int lane = threadIdx.x & 31;
    double acc[M];
#pragma unroll
    for (int m = 0; m < M; ++m) acc[m] = 0.0;
    // blocks of 8 units per lane (j = j0 + lane + 32k): the 8 layer-1 chains
    // advance together over d (independent, so their fp64 latencies overlap);
    // every unit's own chain and the layer-2 accumulation order over j are
    // those of the one-unit-at-a-time loop, so the bits are the same
    for (int j0 = 0; j0 < H; j0 += 256) {
        double pre[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) pre[k] = 0.0;
        for (int d = 0; d < D; ++d) {
            const double xd = __shfl_sync(0xffffffffu, xv, d);
            const double* wr = w1 + (size_t)d * H + j0 + lane;
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (j0 + lane + 32 * k < H) pre[k] = __fma_rn(xd, wr[32 * k], pre[k]);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int j = j0 + lane + 32 * k;
            if (j < H) {
                const double p1 = __dadd_rn(pre[k], b1[j]);
                const double h = p1 > 0.0 ? p1 : 0.0;
#pragma unroll
                for (int m = 0; m < M; ++m) acc[m] = __fma_rn(h, w2[j * w2_sj + m * w2_sm], acc[m]);
            }
        }
    }
    // lanes >= H would contribute zeros; xor butterfly is bit-identical on all lanes
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int m = 0; m < M; ++m) acc[m] = __dadd_rn(acc[m], __shfl_xor_sync(0xffffffffu, acc[m], off));
#pragma unroll
    for (int m = 0; m < M; ++m) q[m] = __dadd_rn(acc[m], b2[m]);
}

// np.argmax: the first NaN if any, else the first maximum
template <int M>
__device__ __forceinline__ int route_argmax(const double (&q)[M]) {
    int best = 0;
    double bv = q[0];
    bool nan_seen = bv != bv;
#pragma unroll
    for (int m = 1; m < M; ++m) {
        if (!nan_seen) {
            if (q[m] != q[m]) {
                best = m;
                nan_seen = true;
            } else if (q[m] > bv) {
                best = m;
                bv = q[m];
            }
        }
    }
    return best;
}

}  // namespace be
