// route.cu — batched router: QNetwork.forward + select_action
// (policy.py:111-132) over B encoded states in fp64.  One warp per state;
// lane l owns hidden units l + 32k; weights staged once per block in shared
// memory (W2 transposed so lanes read consecutive doubles).  Layer 1 is the
// dense x @ W1 (inputs need not be one-hot here), layer 2 a warp butterfly.
#include <cuda_runtime.h>
#include <stdint.h>

#include "be_internal.h"
#include "be_philox.cuh"
#include "be_route.cuh"

namespace be {

template <int M>
__global__ void __launch_bounds__(256) route_kernel(int D, int H, const double* w1, const double* b1,
                                                    const double* w2, const double* b2,
                                                    const double* x, int B, double eps,
                                                    uint64_t seed, uint64_t counter, double* q_out,
                                                    uint8_t* a_out) {
    extern __shared__ __align__(16) double sm[];
    double* sW1 = sm;
    double* sb1 = sW1 + D * H;
    double* sW2t = sb1 + H;
    double* sb2 = sW2t + M * H;
    for (int k = threadIdx.x; k < D * H; k += blockDim.x) sW1[k] = w1[k];
    for (int k = threadIdx.x; k < H; k += blockDim.x) sb1[k] = b1[k];
    for (int k = threadIdx.x; k < M * H; k += blockDim.x) sW2t[k] = w2[(k % H) * M + k / H];
    for (int k = threadIdx.x; k < M; k += blockDim.x) sb2[k] = b2[k];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    for (int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < B; row += warps) {
        double xv = lane < D ? x[(int64_t)row * D + lane] : 0.0;
        double q[M];
        route_row_f64<M>(xv, D, H, sW1, sb1, sW2t, 1, H, sb2, q);
        int best = route_argmax<M>(q);
        if (eps > 0.0) {
            P4 r = philox4x32_10(counter, (uint64_t)row, seed);
            if (u01(r.x[0], r.x[1]) < eps) best = (int)below(r.x[2], (uint32_t)M);
        }
        if (lane < M && q_out) {
#pragma unroll
            for (int m = 0; m < M; ++m)
                if (lane == m) q_out[(int64_t)row * M + m] = q[m];
        }
        if (lane == 0) a_out[row] = (uint8_t)best;
    }
}

template <int M>
static int launch_route_m(const be_qweights* W, int T, const double* x, int B, double eps,
                          uint64_t seed, uint64_t counter, double* q_out, uint8_t* a_out,
                          cudaStream_t st) {
    const int D = T + M + 1, H = W->hidden;
    if (D > 32) return set_error(BE_EINVAL, "input dim must be <= 32");
    size_t smem = sizeof(double) * ((size_t)D * H + H + (size_t)M * H + M);
    if (smem > 200 * 1024) return set_error(BE_EINVAL, "Q-network too large for shared memory");
    auto kern = route_kernel<M>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int blocks = (B + 7) / 8;
    if (blocks > sms * 4) blocks = sms * 4;
    kern<<<blocks, 256, smem, st>>>(D, H, W->w1, W->b1, W->w2, W->b2, x, B, eps, seed, counter, q_out, a_out);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "route launch");
}

int launch_route(const be_qweights* W, int T, int M, const double* x, int B, double eps,
                 uint64_t seed, uint64_t counter, double* q_out, uint8_t* a_out, cudaStream_t st) {
    switch (M) {
        case 1: return launch_route_m<1>(W, T, x, B, eps, seed, counter, q_out, a_out, st);
        case 2: return launch_route_m<2>(W, T, x, B, eps, seed, counter, q_out, a_out, st);
        case 3: return launch_route_m<3>(W, T, x, B, eps, seed, counter, q_out, a_out, st);
        case 4: return launch_route_m<4>(W, T, x, B, eps, seed, counter, q_out, a_out, st);
        case 5: return launch_route_m<5>(W, T, x, B, eps, seed, counter, q_out, a_out, st);
        case 6: return launch_route_m<6>(W, T, x, B, eps, seed, counter, q_out, a_out, st);
        case 7: return launch_route_m<7>(W, T, x, B, eps, seed, counter, q_out, a_out, st);
        case 8: return launch_route_m<8>(W, T, x, B, eps, seed, counter, q_out, a_out, st);
        default: return set_error(BE_EINVAL, "n_tiers out of range");
    }
}

}  // namespace be
