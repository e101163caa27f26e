// route_tc.cu — batched router on the 5th-generation tensor cores:
// QNetwork.forward + select_action (policy.py:111-132) over B encoded states,
// be_qnet_route_tc in include/be200.h.
//
// Persistent CTAs of 256 threads, two per SM (each owns half of the SM's 512
// TMEM columns); per 256-state tile (two 128-row halves):
//   * every thread converts one state row (fp64, D <= 15 inputs + a constant-1
//     bias input) to a 3xTF32 split (hi + lo) in shared memory, K-major
//     no-swizzle UMMA layout;
//   * two passes over the hidden units (H/2 each): one elected thread issues
//     twelve tcgen05.mma.kind::tf32 (2 halves x 2 K-steps x {hi.hi, hi.lo,
//     lo.hi}, M = 128, N = H/2) accumulating the pass's layer-1 pre-activations
//     of both halves in fp32 in TMEM (columns [0, H/2) and [H/2, H));
//     tcgen05.commit -> mbarrier;
//   * epilogue: warps w and w + 4 read the same TMEM lanes r, each half of the
//     pass's columns of BOTH states r and r + 128, relu, and the N = M (<= 4)
//     layer-2 dot products on packed FFMA2 — every W2 shared-memory load feeds
//     two states; after the second pass the two threads exchange partial sums
//     in shared memory and each finalizes one state;
//   * the decision is certified with pairwise error bounds (tc_bound_k1/k2
//     below; the layer-1 term models each tensor-core accumulation step of 8
//     products as 9 fp32 roundings of <= 2u each and enters through the W2
//     column differences); states it cannot certify are re-evaluated four per
//     warp with route_rows_f64 — the exact arithmetic of be_qnet_route_f64 —
//     so every greedy decision equals the fp64 router's.
// Weights are packed once per call (route_tc_pack_kernel: tf32 hi/lo UMMA
// images of [W1; b1]^T, W2 pairs, bound tables) and staged per CTA with one
// bulk asynchronous copy (TMA engine, mbarrier completion).  Q values out are
// the fp32 screen values (fp64 values for fallback states), within 1e-5
// relative of the fp64 router.
#include <cuda_runtime.h>
#include <stdint.h>

#include "be200.h"
#include "be_internal.h"
#include "be_philox.cuh"
#include "be_route.cuh"
#include "be_route_tc.cuh"
#include "be_tc.cuh"

namespace be {

constexpr int TC_ROWS = 128;  // MMA M: states per tile = TMEM lanes
constexpr int TC_TILE = 256;  // states per tile: two 128-row MMA halves
constexpr int TC_THREADS = 256;  // per TMEM lane two threads (lower / upper), each half of the hidden units of both states
constexpr int TC_FBS = 4;     // fp64 fallback: states per warp
constexpr int TC_FBKB = 4;    // fp64 fallback: hidden units per lane per block
constexpr int TC_FLIST = 4096;  // deferred fp64 re-evaluations per CTA (shared-memory list)

template <int M>
__global__ void __launch_bounds__(256) route_tc_pack_kernel(const double* w1, const double* b1, const double* w2,
                                                            const double* b2, int D, int H, float* img) {
    tc_pack_image<M>(w1, b1, w2, b2, D, H, img, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

struct RouteTcParams {
    const double* w1;
    const double* b1;
    const double* w2;
    const double* b2;
    const float* img;
    int32_t D, H, B, ncols;
    const double* x;
    double eps;
    uint64_t seed, counter;
    float* q_out;
    uint8_t* a_out;
    unsigned long long* stats;  // [2] states, fp64 fallbacks (nullable)
    // device-iteration mode (nullable): x / a_out advance by slot * B rows, slot =
    // *iter_dev % pending_P; epsilon = epsilon_at(*iter_dev), Philox counter = *iter_dev
    const int64_t* iter_dev;
    double eps_start, eps_end;
    int64_t eps_decay;
    int32_t pending_P;
};

// DM: compile-time bound of the input count D (8 for the shipped 4 tasks x 3 tiers)
template <int M, int DM>
__global__ void __launch_bounds__(TC_THREADS, 2) route_tc_kernel(const RouteTcParams p) {
    extern __shared__ __align__(1024) unsigned char smem[];
    const TcLayout L{p.H};
    const int img_bytes = L.bytes();
    float* img = reinterpret_cast<float*>(smem);
    float* Ah = reinterpret_cast<float*>(smem + ((img_bytes + 1023) & ~1023));  // [2 halves][TC_ROWS x TC_K]
    float* Al = Ah + 2 * TC_ROWS * TC_K;
    float2* part = reinterpret_cast<float2*>(Al + 2 * TC_ROWS * TC_K);  // [2 sets][TC_MP][TC_TILE] exchanged sums
    uint64_t* bars = reinterpret_cast<uint64_t*>(part + 2 * TC_MP * TC_TILE);  // [0] image, [1] MMA
    uint32_t* tmem_sh = reinterpret_cast<uint32_t*>(bars + 2);
    int* fcount = reinterpret_cast<int*>(tmem_sh + 1);
    int* flist = fcount + 1;  // [TC_FLIST]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int r = tid & (TC_ROWS - 1);  // TMEM lane of this thread
    const double* X = p.x;
    uint8_t* A = p.a_out;
    double eps = p.eps;
    uint64_t ctr = p.counter;
    if (p.iter_dev) {
        const int64_t it = *p.iter_dev;
        const size_t slot = (size_t)(it % p.pending_P);
        X += slot * (size_t)p.B * p.D;
        A += slot * (size_t)p.B;
        eps = epsilon_at(it, p.eps_start, p.eps_end, p.eps_decay);
        ctr = (uint64_t)it;
    }
    const int hs = tid >> 7;            // 0: lower threads, 1: upper threads
    const int D = p.D, H = p.H, HP = H / 2;
    const int nch = HP / TC_CW, c_mid = (nch + 1) / 2;

    if (tid == 0) {
        tc::mbar_init(&bars[0], 1);
        tc::mbar_init(&bars[1], 1);
        tc::fence_mbar_init();
        *fcount = 0;
    }
    if (warp == 0) tc::tmem_alloc(tmem_sh, (uint32_t)p.ncols);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *tmem_sh;
    if (tid == 0) {  // weights: one bulk asynchronous copy of the packed image
        tc::mbar_expect_tx(&bars[0], (uint32_t)img_bytes);
        tc::bulk_g2s(img, p.img, (uint32_t)img_bytes, &bars[0]);
    }
    tc::mbar_wait(&bars[0], 0);

    const float* B1h = img + L.b1h() / 4;
    const float* B1l = img + L.b1l() / 4;
    const float4* W2q = reinterpret_cast<const float4*>(img + L.w2p() / 4);
    const float* fb2 = img + L.b2() / 4;
    const float* C = img + L.bound() / 4;
    const float* Dp = img + L.pairs() / 4;
    const uint32_t idesc = tc::idesc_tf32(TC_ROWS, HP);
    const int ntiles = (p.B + TC_TILE - 1) / TC_TILE;
    uint32_t phase = 0;
    unsigned n_rows = 0, n_fb = 0;

    // fp64 re-evaluation of the states the bound could not certify, TC_FBS states
    // per warp (each weight load feeds all of them); deferred (CTA list in shared
    // memory) so no tile waits for it
    auto fallback = [&](int nf) {
        for (int f0 = warp * TC_FBS; f0 < nf; f0 += TC_THREADS / 32 * TC_FBS) {
            int rf[TC_FBS];
            double xv[TC_FBS];
#pragma unroll
            for (int s = 0; s < TC_FBS; ++s) {
                rf[s] = flist[f0 + s < nf ? f0 + s : f0];  // past the end: repeat the first, no output
                xv[s] = lane < D ? __ldg(X + (size_t)rf[s] * D + lane) : 0.0;
            }
            double q64[TC_FBS][M];
            route_rows_f64<M, TC_FBS, TC_FBKB, 1>(xv, D, H, p.w1, p.b1, p.w2, M, 1, p.b2, q64);
#pragma unroll
            for (int s = 0; s < TC_FBS; ++s) {
                if (f0 + s >= nf) break;
                int b = route_argmax<M>(q64[s]);
                if (eps > 0.0) {
                    P4 rn = philox4x32_10(ctr, (uint64_t)rf[s], p.seed);
                    if (u01(rn.x[0], rn.x[1]) < eps) b = (int)below(rn.x[2], (uint32_t)M);
                }
                if (lane < M && p.q_out) {
#pragma unroll
                    for (int m = 0; m < M; ++m)
                        if (lane == m) p.q_out[(size_t)rf[s] * M + m] = (float)q64[s][m];
                }
                if (lane == 0) A[rf[s]] = (uint8_t)b;
            }
        }
    };
    // relu + layer 2 of one TC_CW-unit chunk for BOTH states of this lane (u0:
    // state r, u1: state r + 128), so every W2 shared-memory load feeds two
    // states; units (2i, 2i+1) accumulate into set 0, (2i+2, 2i+3) into set 1
    float2 a0[2][M], a1[2][M];
    auto consume = [&](const float(&u0)[TC_CW], const float(&u1)[TC_CW], int jb) {
#pragma unroll
        for (int i = 0; i < TC_CW / 2; i += 2) {
            const float2 h00 = make_float2(fmaxf(u0[2 * i], 0.f), fmaxf(u0[2 * i + 1], 0.f));
            const float2 h01 = make_float2(fmaxf(u0[2 * i + 2], 0.f), fmaxf(u0[2 * i + 3], 0.f));
            const float2 h10 = make_float2(fmaxf(u1[2 * i], 0.f), fmaxf(u1[2 * i + 1], 0.f));
            const float2 h11 = make_float2(fmaxf(u1[2 * i + 2], 0.f), fmaxf(u1[2 * i + 3], 0.f));
            const float4* g = W2q + (size_t)((jb + 2 * i) >> 2) * 4;
            const float4 g0 = g[0], g1 = g[1];
            a0[0][0] = ffma2(h00, make_float2(g0.x, g0.y), a0[0][0]);
            a0[1][0] = ffma2(h01, make_float2(g1.x, g1.y), a0[1][0]);
            a1[0][0] = ffma2(h10, make_float2(g0.x, g0.y), a1[0][0]);
            a1[1][0] = ffma2(h11, make_float2(g1.x, g1.y), a1[1][0]);
            if (M > 1) {
                constexpr int m1 = M > 1 ? 1 : 0;
                a0[0][m1] = ffma2(h00, make_float2(g0.z, g0.w), a0[0][m1]);
                a0[1][m1] = ffma2(h01, make_float2(g1.z, g1.w), a0[1][m1]);
                a1[0][m1] = ffma2(h10, make_float2(g0.z, g0.w), a1[0][m1]);
                a1[1][m1] = ffma2(h11, make_float2(g1.z, g1.w), a1[1][m1]);
            }
            if (M > 2) {
                constexpr int m2 = M > 2 ? 2 : 0;
                const float4 g2 = g[2];
                a0[0][m2] = ffma2(h00, make_float2(g2.x, g2.y), a0[0][m2]);
                a0[1][m2] = ffma2(h01, make_float2(g2.z, g2.w), a0[1][m2]);
                a1[0][m2] = ffma2(h10, make_float2(g2.x, g2.y), a1[0][m2]);
                a1[1][m2] = ffma2(h11, make_float2(g2.z, g2.w), a1[1][m2]);
            }
            if (M > 3) {
                constexpr int m3 = M > 3 ? 3 : 0;
                const float4 g3 = g[3];
                a0[0][m3] = ffma2(h00, make_float2(g3.x, g3.y), a0[0][m3]);
                a0[1][m3] = ffma2(h01, make_float2(g3.z, g3.w), a0[1][m3]);
                a1[0][m3] = ffma2(h10, make_float2(g3.x, g3.y), a1[0][m3]);
                a1[1][m3] = ffma2(h11, make_float2(g3.z, g3.w), a1[1][m3]);
            }
        }
    };
    // this thread's state row of a tile (thread t stages state t of the tile)
    auto load_row = [&](int tile, double (&xd)[DM]) {
        const int row = tile * TC_TILE + tid;
#pragma unroll
        for (int k = 0; k < DM; ++k)
            xd[k] = (k < D && tile < ntiles && row < p.B) ? __ldg(X + (size_t)row * D + k) : 0.0;
    };
    // one pass: layer 1 for hidden units [pass * HP, pass * HP + HP) of both
    // 128-state halves (TMEM columns [0, HP) and [HP, 2 HP)); one thread issues
    auto issue_mma = [&](int pass) {
        tc::fence_after_sync();
        const float* bh0 = B1h + pass * HP * TC_K;  // 8-row groups of 128 floats: row n0 at n0 * 16
        const float* bl0 = B1l + pass * HP * TC_K;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t d = tmem + (uint32_t)(h * HP);
            const float* ah0 = Ah + h * TC_ROWS * TC_K;
            const float* al0 = Al + h * TC_ROWS * TC_K;
#pragma unroll
            for (int s = 0; s < TC_K / 8; ++s) {  // K-step s reads K-groups 2s, 2s + 1
                const uint64_t ah = tc::smem_desc(ah0 + s * 64, 128, 512), al = tc::smem_desc(al0 + s * 64, 128, 512);
                const uint64_t bh = tc::smem_desc(bh0 + s * 64, 128, 512), bl = tc::smem_desc(bl0 + s * 64, 128, 512);
                tc::mma_tf32(d, ah, bh, idesc, s > 0);
                tc::mma_tf32(d, ah, bl, idesc, true);
                tc::mma_tf32(d, al, bh, idesc, true);
            }
        }
        tc::mma_commit(&bars[1]);
    };
    // epilogue of one pass: lower threads take chunks [0, c_mid), upper [c_mid, nch)
    const uint32_t lane_addr = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    auto epilogue = [&](int pass) {
        const int c0 = hs ? c_mid : 0, c1 = hs ? nch : c_mid;
        for (int c = c0; c < c1; ++c) {
            float u0[TC_CW], u1[TC_CW];
            tc::tmem_ld_issue(lane_addr + (uint32_t)(c * TC_CW), u0);
            tc::tmem_ld_issue(lane_addr + (uint32_t)(HP + c * TC_CW), u1);
            tc::tmem_ld_wait(u0);
            tc::tmem_ld_wait(u1);
            consume(u0, u1, pass * HP + c * TC_CW);
        }
    };

    double xn[DM];  // next tile's state row, loaded during this tile's MMAs and epilogue
    load_row(blockIdx.x, xn);

    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int row = tile * TC_TILE + tid;
        const bool valid = row < p.B;
        // ---- A operand: this thread's state row, 3xTF32 split (+ the bias input = 1)
        float xf[DM];
#pragma unroll
        for (int k = 0; k < DM; ++k) xf[k] = __double2float_rn(xn[k]);
        auto in = [&](int k) { return k < DM && k < D ? xf[k < DM ? k : 0] : (k == D ? 1.f : 0.f); };
        float* ahm = Ah + hs * TC_ROWS * TC_K;
        float* alm = Al + hs * TC_ROWS * TC_K;
#pragma unroll
        for (int kg = 0; kg < TC_K / 4; ++kg) {
            float4 h, l;
            h.x = tc::to_tf32(in(4 * kg + 0));
            h.y = tc::to_tf32(in(4 * kg + 1));
            h.z = tc::to_tf32(in(4 * kg + 2));
            h.w = tc::to_tf32(in(4 * kg + 3));
            l.x = tc::to_tf32(__fsub_rn(in(4 * kg + 0), h.x));
            l.y = tc::to_tf32(__fsub_rn(in(4 * kg + 1), h.y));
            l.z = tc::to_tf32(__fsub_rn(in(4 * kg + 2), h.z));
            l.w = tc::to_tf32(__fsub_rn(in(4 * kg + 3), h.w));
            *reinterpret_cast<float4*>(ahm + umma_off(r, 4 * kg)) = h;
            *reinterpret_cast<float4*>(alm + umma_off(r, 4 * kg)) = l;
        }
        // decision bound (needs only the inputs): against exact arithmetic on the
        // fp32-rounded inputs; the fp64 inputs differ by <= u |x|, covered by the slack in K
        float Bd = C[D];
        float Bp[TC_NP > 0 && M > 1 ? M * (M - 1) / 2 : 1];
#pragma unroll
        for (int k = 0; k < DM; ++k)
            if (k < D) Bd = __fmaf_ru(fabsf(xf[k]), C[k], Bd);
#pragma unroll
        for (int b = 0; b < M; ++b)
#pragma unroll
            for (int sx = b + 1; sx < M; ++sx) {
                const int pq = b * (2 * M - b - 1) / 2 + (sx - b - 1);  // dense index among M actions
                const float* dp = Dp + tc_pair(b, sx) * TC_K;
                float v = dp[D];
#pragma unroll
                for (int k = 0; k < DM; ++k)
                    if (k < D) v = __fmaf_ru(fabsf(xf[k]), dp[k], v);
                Bp[pq] = __fadd_ru(v, Bd);
            }
        tc::fence_proxy_async_smem();
        tc::fence_before_sync();  // the previous tile's TMEM loads are complete
        __syncthreads();
        if (tid == 0) issue_mma(0);
        load_row(tile + gridDim.x, xn);  // overlaps the MMAs and the epilogues
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
            for (int m = 0; m < M; ++m) a0[s][m] = a1[s][m] = make_float2(0.f, 0.f);
        tc::mbar_wait(&bars[1], phase);
        phase ^= 1u;
        tc::fence_after_sync();
        epilogue(0);
        tc::fence_before_sync();
        __syncthreads();
        if (tid == 0) issue_mma(1);
        tc::mbar_wait(&bars[1], phase);
        phase ^= 1u;
        tc::fence_after_sync();
        epilogue(1);
        // ---- exchange: the lower thread of lane r finalizes state r, the upper one
        // state r + 128; each hands the other its partial sums of the other state
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
            for (int m = 0; m < M; ++m) part[(s * TC_MP + m) * TC_TILE + (tid ^ TC_ROWS)] = hs ? a0[s][m] : a1[s][m];
        __syncthreads();
        {
            float q[M];
            int best = 0;
            float bv = 0.f;
            bool fin = true;
#pragma unroll
            for (int m = 0; m < M; ++m) {
                float2 t[2];
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const float2 own = hs ? a1[s][m] : a0[s][m];
                    const float2 u = part[(s * TC_MP + m) * TC_TILE + tid];
                    t[s] = make_float2(__fadd_rn(own.x, u.x), __fadd_rn(own.y, u.y));
                }
                const float t0 = __fadd_rn(t[0].x, t[0].y), t1 = __fadd_rn(t[1].x, t[1].y);
                q[m] = __fadd_rn(__fadd_rn(t0, t1), fb2[m]);
                fin = fin && isfinite(q[m]);
                if (m == 0 || q[m] > bv) {  // first maximum (a tie is never certified)
                    best = m;
                    bv = q[m];
                }
            }
            // every other action must trail the leader by more than the pair's bound
            bool sure = fin;
#pragma unroll
            for (int b = 0; b < M; ++b)
#pragma unroll
                for (int sx = b + 1; sx < M; ++sx) {
                    const int pq = b * (2 * M - b - 1) / 2 + (sx - b - 1);
                    if (best == b || best == sx) {
                        const float other = best == b ? q[sx] : q[b];
                        sure = sure && isfinite(Bp[pq]) && __dsub_rd((double)bv, (double)other) > (double)Bp[pq];
                    }
                }
            sure = M == 1 || sure;
            if (valid) {
                ++n_rows;
                if (!sure) {
                    ++n_fb;
                    flist[atomicAdd(fcount, 1)] = row;
                } else {
                    if (eps > 0.0) {
                        P4 rn = philox4x32_10(ctr, (uint64_t)row, p.seed);
                        if (u01(rn.x[0], rn.x[1]) < eps) best = (int)below(rn.x[2], (uint32_t)M);
                    }
                    if (p.q_out) {
#pragma unroll
                        for (int m = 0; m < M; ++m) p.q_out[(size_t)row * M + m] = q[m];
                    }
                    A[row] = (uint8_t)best;
                }
            }
        }
        // the deferred list can take one more full tile?  else drain it now
        __syncthreads();
        const int nf = *fcount;
        if (nf > TC_FLIST - TC_TILE) {
            fallback(nf);
            __syncthreads();
            if (tid == 0) *fcount = 0;
        }
    }
    __syncthreads();
    fallback(*fcount);
    if (p.stats) {
        const unsigned s0 = __reduce_add_sync(0xffffffffu, n_rows);
        const unsigned s1 = __reduce_add_sync(0xffffffffu, n_fb);
        if (lane == 0) {
            atomicAdd(&p.stats[0], (unsigned long long)s0);
            atomicAdd(&p.stats[1], (unsigned long long)s1);
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, (uint32_t)p.ncols);
}

bool route_tc_supported(int T, int M, int H) {
    const int D = T + M + 1;
    return M >= 1 && M <= TC_MP && D + 1 <= TC_K && H >= 32 && H <= 256 && H % 32 == 0;
}

size_t route_tc_workspace_bytes(int H) { return (size_t)TcLayout{H}.bytes(); }

static size_t route_tc_smem(int H);

template <int M>
static void route_tc_prepare_m(int D, int H) {
    auto kern = D <= 8 ? route_tc_kernel<M, 8> : route_tc_kernel<M, TC_K - 1>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)route_tc_smem(H));
}

void route_tc_prepare(int T, int M, int H) {
    const int D = T + M + 1;
    switch (M) {
        case 1: route_tc_prepare_m<1>(D, H); break;
        case 2: route_tc_prepare_m<2>(D, H); break;
        case 3: route_tc_prepare_m<3>(D, H); break;
        case 4: route_tc_prepare_m<4>(D, H); break;
        default: break;
    }
}

static size_t route_tc_smem(int H) {
    const size_t img = ((size_t)TcLayout{H}.bytes() + 1023) & ~size_t(1023);
    const size_t need = img + 4 * sizeof(float) * TC_ROWS * TC_K + sizeof(float2) * 2 * TC_MP * TC_TILE + 2 * 8 +
                        4 + 4 + 4 * TC_FLIST;
    // at most two CTAs per SM: each owns up to 256 of the SM's 512 TMEM columns
    return need > 80 * 1024 ? need : 80 * 1024;
}

struct TcDevIter {
    const int64_t* iter_dev;
    double eps_start, eps_end;
    int64_t eps_decay;
    int32_t pending_P;
};

template <int M>
static int launch_route_tc_m(const be_qweights* W, int T, const double* x, int B, double eps, uint64_t seed,
                             uint64_t counter, float* q_out, uint8_t* a_out, void* workspace,
                             unsigned long long* stats, cudaStream_t st, const TcDevIter* dv = nullptr) {
    const int D = T + M + 1, H = W->hidden;
    float* img = reinterpret_cast<float*>(workspace);
    route_tc_pack_kernel<M><<<8, 256, 0, st>>>(W->w1, W->b1, W->w2, W->b2, D, H, img);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e, "route_tc pack launch");
    if (B == 0) return BE_OK;
    RouteTcParams p{};
    p.w1 = W->w1;
    p.b1 = W->b1;
    p.w2 = W->w2;
    p.b2 = W->b2;
    p.img = img;
    p.D = D;
    p.H = H;
    p.B = B;
    p.ncols = H <= 32 ? 32 : H <= 64 ? 64 : H <= 128 ? 128 : 256;
    p.x = x;
    p.eps = eps;
    p.seed = seed;
    p.counter = counter;
    p.q_out = q_out;
    p.a_out = a_out;
    p.stats = stats;
    if (dv) {
        p.iter_dev = dv->iter_dev;
        p.eps_start = dv->eps_start;
        p.eps_end = dv->eps_end;
        p.eps_decay = dv->eps_decay;
        p.pending_P = dv->pending_P;
    }
    const size_t smem = route_tc_smem(H);
    auto kern = D <= 8 ? route_tc_kernel<M, 8> : route_tc_kernel<M, TC_K - 1>;
    if (!dv) {  // the device-iteration form is configured at learner creation (graph capture)
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return set_cuda_error(e, "route_tc smem attribute");
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int ntiles = (B + TC_TILE - 1) / TC_TILE;
    const int blocks = ntiles < 2 * sms ? ntiles : 2 * sms;
    kern<<<blocks, TC_THREADS, smem, st>>>(p);
    e = cudaGetLastError();
    return e == cudaSuccess ? BE_OK : set_cuda_error(e, "route_tc launch");
}

int launch_route_tc(const be_qweights* W, int T, int M, const double* x, int B, double eps, uint64_t seed,
                    uint64_t counter, float* q_out, uint8_t* a_out, void* workspace, int64_t* stats,
                    cudaStream_t st) {
    auto* s = reinterpret_cast<unsigned long long*>(stats);
    switch (M) {
        case 1: return launch_route_tc_m<1>(W, T, x, B, eps, seed, counter, q_out, a_out, workspace, s, st);
        case 2: return launch_route_tc_m<2>(W, T, x, B, eps, seed, counter, q_out, a_out, workspace, s, st);
        case 3: return launch_route_tc_m<3>(W, T, x, B, eps, seed, counter, q_out, a_out, workspace, s, st);
        case 4: return launch_route_tc_m<4>(W, T, x, B, eps, seed, counter, q_out, a_out, workspace, s, st);
        default: return set_error(BE_EINVAL, "route_tc: n_tiers must be <= 4");
    }
}

int launch_route_tc_dev(const be_qweights* W, int T, int M, const double* x_base, int B, uint64_t seed,
                        const int64_t* iter_dev, double eps_start, double eps_end, int64_t eps_decay,
                        int32_t pending_P, uint8_t* a_base, void* workspace, int64_t* stats, cudaStream_t st) {
    const TcDevIter dv{iter_dev, eps_start, eps_end, eps_decay, pending_P};
    auto* s = reinterpret_cast<unsigned long long*>(stats);
    switch (M) {
        case 1: return launch_route_tc_m<1>(W, T, x_base, B, 0.0, seed, 0, nullptr, a_base, workspace, s, st, &dv);
        case 2: return launch_route_tc_m<2>(W, T, x_base, B, 0.0, seed, 0, nullptr, a_base, workspace, s, st, &dv);
        case 3: return launch_route_tc_m<3>(W, T, x_base, B, 0.0, seed, 0, nullptr, a_base, workspace, s, st, &dv);
        case 4: return launch_route_tc_m<4>(W, T, x_base, B, 0.0, seed, 0, nullptr, a_base, workspace, s, st, &dv);
        default: return set_error(BE_EINVAL, "route_tc: n_tiers must be <= 4");
    }
}

}  // namespace be
