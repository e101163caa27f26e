// be_route_tc.cuh — the tensor-core router's packed weight image and its
// certified-decision error bounds, shared by route_tc.cu (the batched router)
// and step.cu (the training env step with the decision on the tensor cores).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "be_tc.cuh"

namespace be {

constexpr int TC_CW = 16;     // TMEM columns per tcgen05.ld in the epilogue
constexpr int TC_K = 16;      // inputs (D <= 15) + the bias input, two tf32 K-steps of 8
constexpr int TC_MP = 4;      // layer-2 outputs padded (n_tiers <= 4)
constexpr int TC_NP = TC_MP * (TC_MP - 1) / 2;  // action pairs (b < s) of the pairwise bounds


struct TcLayout {  // byte offsets inside the packed image (= the shared-memory image)
    int H;
    __host__ __device__ int b1h() const { return 0; }
    __host__ __device__ int b1l() const { return H * TC_K * 4; }
    __host__ __device__ int w2p() const { return 2 * H * TC_K * 4; }         // [H/4][4] float4
    __host__ __device__ int b2() const { return w2p() + (H / 2) * TC_MP * 8; }  // [TC_MP] float
    __host__ __device__ int bound() const { return b2() + TC_MP * 4; }         // [TC_K] float
    __host__ __device__ int pairs() const { return bound() + TC_K * 4; }       // [TC_NP][TC_K] float
    __host__ __device__ int bytes() const { return pairs() + TC_NP * TC_K * 4; }  // multiple of 16
};

// element (n, k) of a K-major no-swizzle UMMA operand with K = 16: 8 x 16-byte core
// matrices, K-groups of 4 at 128 B (LBO), 8-row groups at 512 B (SBO); in floats
__host__ __device__ __forceinline__ int umma_off(int n, int k) {
    return (n >> 3) * 128 + (k >> 2) * 32 + (n & 7) * 4 + (k & 3);
}

// Error bound of the fp32 decision (units of u = 2^-24).  Layer 1: input / weight
// rounding and the dropped lo.lo term (14) + 6 MMAs x 9 accumulations x 2 (108)
// bound |h32_j - h_j| <= 122 u P_j, P_j = sum_k |x_k| |W1[k][j]| + |b1[j]|; in the
// difference q_b - q_s of two actions they enter as sum_j (W2[j][b] - W2[j][s]) dh_j,
// so with K1 = (122 + 8) u:  K1 sum_j |W2[j][b] - W2[j][s]| P_j.  Layer 2: FFMA2
// chains of <= L = 8 ceil(H / 64) terms (a thread's share of a state: 2 passes x
// <= ceil(H / 64) chunks of 16 units over 2 sets x 2 lanes) + the lower/upper merge,
// the lane merge, the set merge and the bias add + W2 / b2 rounding (<= L + 7),
// independent per action: K2 = (L + 7 + 16) u times S_m = sum_j |W2[j][m]| P_j + |b2[m]|
// for each of the two.  The leader b is certified when, for every other action s,
// q32_b - q32_s > K1 D_bs + 2 K2 max_m S_m (evaluated with upward-rounded fp32 terms
// and a downward-rounded fp64 difference).
__host__ __device__ __forceinline__ double tc_bound_k1() { return (double)(122 + 8) * 0x1p-24; }
__host__ __device__ __forceinline__ double tc_bound_k2(int H) {
    return (double)(8 * ((H + 63) / 64) + 7 + 16) * 0x1p-24;
}
__host__ __device__ constexpr int tc_pair(int b, int s) {  // b < s < TC_MP
    return b * TC_MP - b * (b + 1) / 2 + (s - b - 1);
}

// Packs the router's shared-memory image (TcLayout) from fp64 weights; (tid, nt): this
// thread's index among the nt threads sharing the work (whole warps: the bound tables
// are reduced one warp per row).  route_tc_pack_kernel and the training step's prep
// launch both run it.
template <int M>
__device__ __forceinline__ void tc_pack_image(const double* w1, const double* b1, const double* w2,
                                              const double* b2, int D, int H, float* img, int tid, int nt) {
    const TcLayout L{H};
    float* b1h = img + L.b1h() / 4;
    float* b1l = img + L.b1l() / 4;
    for (int e = tid; e < H * TC_K; e += nt) {
        const int n = e / TC_K, k = e % TC_K;
        const double w = k < D ? w1[(size_t)k * H + n] : (k == D ? b1[n] : 0.0);
        const float f = __double2float_rn(w);
        const float hi = tc::to_tf32(f);
        b1h[umma_off(n, k)] = hi;
        b1l[umma_off(n, k)] = tc::to_tf32(__fsub_rn(f, hi));
    }
    // W2 in groups of four hidden units j..j+3 (two FFMA2 pairs), four float4 each:
    // (w[j][0], w[j+1][0], w[j][1], w[j+1][1]), the same for j+2, j+3, then
    // (w[j..j+3][2]) and (w[j..j+3][3]) — M = 3 needs 3 loads per 4 units, not 4
    float* w2q = img + L.w2p() / 4;
    for (int e = tid; e < (H / 4) * 16; e += nt) {
        const int g = e / 16, f = e % 16, v = f / 4, c = f % 4;
        int j, m;
        if (v < 2) {
            j = 4 * g + 2 * v + (c & 1);
            m = c >> 1;
        } else {
            j = 4 * g + c;
            m = v;
        }
        w2q[e] = m < M ? __double2float_rn(w2[(size_t)j * M + m]) : 0.f;
    }
    float* fb2 = img + L.b2() / 4;
    for (int m = tid; m < TC_MP; m += nt) fb2[m] = m < M ? __double2float_rn(b2[m]) : 0.f;
    // bound tables, one warp per row: C[k] = 2 K2 max_m sum_j |W2[j][m]| |W1[k][j]|
    // (k < D), C[D] = 2 K2 max_m (sum_j |W2[j][m]| |b1[j]| + |b2[m]|); pairs
    // Dp[k] = K1 sum_j |W2[j][b] - W2[j][s]| |W1[k][j]| (k < D), Dp[D] = K1 sum_j
    // |W2[j][b] - W2[j][s]| |b1[j]|; non-finite weights give NaN (never certified)
    float* C = img + L.bound() / 4;
    float* Dp = img + L.pairs() / 4;
    const double K1 = tc_bound_k1(), K2 = tc_bound_k2(H);
    const int lane = threadIdx.x & 31, gw = tid >> 5, nw = nt >> 5;
    for (int row = gw; row < TC_K * (1 + TC_NP); row += nw) {
        const int k = row % TC_K, pr = row / TC_K - 1;  // pr < 0: the per-action table C
        double mx = 0.0;
        bool bad = false;
        if (pr < 0) {
            for (int m = 0; m < M; ++m) {
                double acc = 0.0;
                for (int j = lane; j < H; j += 32) {
                    const double a = k < D ? w1[(size_t)k * H + j] : (k == D ? b1[j] : 0.0);
                    acc = __fma_rn(fabs(w2[(size_t)j * M + m]), fabs(a), acc);
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
                if (k == D) acc = __dadd_ru(acc, fabs(b2[m]));
                mx = fmax(mx, acc);
                bad = bad || acc != acc;
            }
            if (lane == 0) C[k] = bad ? __int_as_float(0x7fc00000) : __double2float_ru(__dmul_ru(2.0 * K2, mx));
        } else {
            int b = 0, sx = 1;  // the pair of index pr
            for (int q = 0; q < pr; ++q)
                if (++sx == TC_MP) sx = ++b + 1;
            double acc = 0.0;
            if (sx < M) {
                for (int j = lane; j < H; j += 32) {
                    const double a = k < D ? w1[(size_t)k * H + j] : (k == D ? b1[j] : 0.0);
                    acc = __fma_rn(fabs(__dsub_rn(w2[(size_t)j * M + b], w2[(size_t)j * M + sx])), fabs(a), acc);
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, off));
            }
            // |W2 b - W2 s| is rounded to nearest in fp64: the relative error u_64 is far
            // inside the slack of K1
            if (lane == 0) Dp[pr * TC_K + k] = acc != acc ? __int_as_float(0x7fc00000) : __double2float_ru(__dmul_ru(K1, acc));
        }
    }
}

}  // namespace be
