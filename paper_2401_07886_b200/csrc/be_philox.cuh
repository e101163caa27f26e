// be_philox.cuh — counter-based Philox4x32-10 (Salmon et al., SC'11).
// Used wherever the reference draws from numpy PCG64: epsilon-greedy routing
// (policy.py:125-132), replay sampling (trainer.py:158-163), on-device trace
// generation (workload.py:94-141).  PCG64 streams cannot be reproduced, so
// parity for these draws is statistical.
#pragma once
#include <stdint.h>

namespace be {

struct P4 {
    uint32_t x[4];
};

__host__ __device__ __forceinline__ P4 philox4x32_10(uint64_t counter_lo, uint64_t counter_hi,
                                                     uint64_t key) {
    uint32_t c0 = (uint32_t)counter_lo, c1 = (uint32_t)(counter_lo >> 32);
    uint32_t c2 = (uint32_t)counter_hi, c3 = (uint32_t)(counter_hi >> 32);
    uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0;
        c1 = n1;
        c2 = n2;
        c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    P4 out;
    out.x[0] = c0;
    out.x[1] = c1;
    out.x[2] = c2;
    out.x[3] = c3;
    return out;
}

// 53-bit uniform double in [0, 1) from two 32-bit words (numpy's recipe).
__host__ __device__ __forceinline__ double u01(uint32_t a, uint32_t b) {
    return ((double)(a >> 5) * 67108864.0 + (double)(b >> 6)) * (1.0 / 9007199254740992.0);
}

// Unbiased-enough integer in [0, n) (Lemire multiply-shift; n << 2^32).
__host__ __device__ __forceinline__ uint32_t below(uint32_t r, uint32_t n) {
    return (uint32_t)(((uint64_t)r * n) >> 32);
}

// TrainConfig.epsilon_at (trainer.py:85-90), the same IEEE operations as the host
__host__ __device__ __forceinline__ double epsilon_at(int64_t it, double start, double end, int64_t decay) {
    if (decay <= 0) return end;
#ifdef __CUDA_ARCH__
    const double frac = fmin(1.0, __ddiv_rn((double)it, (double)decay));
    return __dadd_rn(start, __dmul_rn(__dsub_rn(end, start), frac));
#else
    const double q = (double)it / (double)decay;
    const double frac = q < 1.0 ? q : 1.0;
    return start + (end - start) * frac;
#endif
}

}  // namespace be
