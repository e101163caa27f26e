// be_route.cuh — the fp64 router arithmetic of be_qnet_route_f64
// (QNetwork.forward + argmax, policy.py:111-132) for one state per warp.
// Shared by route_kernel and the tensor-core router's fallback so both give
// the same bits: lane l owns hidden units l + 32k; layer 1 is the dense
// x @ W1 in input order, then + b1; layer 2 accumulates over j in increasing
// order per lane, then a warp butterfly.  The tensor-core router re-evaluates
// its uncertified states S at a time (route_rows_f64) with the same bits.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace be {

// S states at once (every weight load feeds S states): xv[s] on lane d (< D)
// holds x_s[d].  W2 element (j, m) at w2[j * w2_sj + m * w2_sm].  Lane l owns
// units j = l + 32k, taken in blocks of KB per lane: the KB x S layer-1 chains
// advance together over d (independent, so their fp64 latencies overlap);
// every unit's own chain and the layer-2 accumulation order over j are those
// of the one-unit-at-a-time loop, so the bits do not depend on S, KB or the
// unroll depth UD of the input loop.
template <int M, int S, int KB, int UD>
__device__ __forceinline__ void route_rows_f64(const double (&xv)[S], int D, int H, const double* __restrict__ w1,
                                               const double* __restrict__ b1, const double* __restrict__ w2,
                                               int w2_sj, int w2_sm, const double* __restrict__ b2,
                                               double (&q)[S][M]) {
    const int lane = threadIdx.x & 31;
    double acc[S][M];
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
        for (int m = 0; m < M; ++m) acc[s][m] = 0.0;
    for (int j0 = 0; j0 < H; j0 += 32 * KB) {
        double pre[S][KB];
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int k = 0; k < KB; ++k) pre[s][k] = 0.0;
#pragma unroll(UD)
        for (int d = 0; d < D; ++d) {
            double xd[S];
#pragma unroll
            for (int s = 0; s < S; ++s) xd[s] = __shfl_sync(0xffffffffu, xv[s], d);
            const double* wr = w1 + (size_t)d * H + j0 + lane;
#pragma unroll
            for (int k = 0; k < KB; ++k)
                if (j0 + lane + 32 * k < H) {
                    const double w = wr[32 * k];
#pragma unroll
                    for (int s = 0; s < S; ++s) pre[s][k] = __fma_rn(xd[s], w, pre[s][k]);
                }
        }
#pragma unroll
        for (int k = 0; k < KB; ++k) {
            const int j = j0 + lane + 32 * k;
            if (j < H) {
                const double bj = b1[j];
                double w2j[M];
#pragma unroll
                for (int m = 0; m < M; ++m) w2j[m] = w2[j * w2_sj + m * w2_sm];
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const double p1 = __dadd_rn(pre[s][k], bj);
                    const double h = p1 > 0.0 ? p1 : 0.0;
#pragma unroll
                    for (int m = 0; m < M; ++m) acc[s][m] = __fma_rn(h, w2j[m], acc[s][m]);
                }
            }
        }
    }
    // lanes >= H would contribute zeros; xor butterfly is bit-identical on all lanes
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int m = 0; m < M; ++m) acc[s][m] = __dadd_rn(acc[s][m], __shfl_xor_sync(0xffffffffu, acc[s][m], off));
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
        for (int m = 0; m < M; ++m) q[s][m] = __dadd_rn(acc[s][m], b2[m]);
}

// one state: xv on lane d (< D) holds x[d]
template <int M>
__device__ __forceinline__ void route_row_f64(double xv, int D, int H, const double* __restrict__ w1,
                                              const double* __restrict__ b1, const double* __restrict__ w2,
                                              int w2_sj, int w2_sm, const double* __restrict__ b2,
                                              double (&q)[M]) {
    const double x1[1] = {xv};
    double q1[1][M];
    route_rows_f64<M, 1, 8, 4>(x1, D, H, w1, b1, w2, w2_sj, w2_sm, b2, q1);
#pragma unroll
    for (int m = 0; m < M; ++m) q[m] = q1[0][m];
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
