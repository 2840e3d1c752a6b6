// sprout_device.cuh -- device helpers shared by the CUDA kernels of libsprout.
// (The CPU oracle in oracle/ has its own independent implementation.)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "sprout.h"

namespace sprout {

constexpr int kMaxLevels = SPROUT_MAX_LEVELS;
constexpr int kMaxClasses = SPROUT_MAX_CLASSES;

// Philox4x32-10 (Salmon et al., SC'11; Random123 constants).  The paper only
// says x_i is "the probability of applying the i-th directive level";
// the counter-based draw is reading L10.  mul.wide.u32 gives hi/lo in one
// IMAD.WIDE.U32; the three-input XORs fold into LOP3.
struct Philox4 {
    uint32_t v[4];
};

__device__ __forceinline__ Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                 uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    Philox4 o;
    o.v[0] = c0; o.v[1] = c1; o.v[2] = c2; o.v[3] = c3;
    return o;
}

// Same generator with the key schedule precomputed (round r uses
// (k0 + r*W0, k1 + r*W1)); rk0/rk1 live in the kernel's parameter space.
__device__ __forceinline__ Philox4 philox4x32_10_rk(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                    const uint32_t (&rk0)[10], const uint32_t (&rk1)[10]) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ rk0[r];
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ rk1[r];
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
    }
    Philox4 o;
    o.v[0] = c0; o.v[1] = c1; o.v[2] = c2; o.v[3] = c3;
    return o;
}

// Constant per-launch cost coefficients (copied from the host struct).
struct CostConst {
    double ef[kMaxClasses][kMaxLevels];
    double et[kMaxClasses][kMaxLevels];
    double pf[kMaxClasses][kMaxLevels];
    double pt[kMaxClasses][kMaxLevels];
};

__device__ __forceinline__ bool finite_nonneg(double v) { return v >= 0.0 && v <= 1.7976931348623157e308; }

// Static-grid points (Sprout_Sta sweep; reading L18): compositions
// (k_0..k_{n-1}) of D into n non-negative parts, ordered by k_0 descending,
// then k_1 descending, ...  compositions(r, m) = C(r + m - 1, m - 1).
__host__ __device__ inline int64_t compositions(int r, int m) {
    if (m <= 1) return 1;
    int64_t c = 1;   // C(r + m - 1, m - 1), exact: each step is an integer binomial
    for (int i = 1; i < m; ++i) c = c * (r + i) / i;
    return c;
}

// Unrank point j (0 <= j < compositions(D, n)) into k[0..n-1]: skip whole
// blocks of equal k_i (largest first) by their sizes.
__device__ inline void grid_unrank_rt(int n, int D, int64_t j, int *k) {   // runtime n (small kernels)
    int rem = D;
    for (int i = 0; i < n - 1; ++i) {
        int v = rem;
        for (;;) {
            const int64_t block = compositions(rem - v, n - 1 - i);
            if (j < block || v == 0) break;
            j -= block;
            --v;
        }
        k[i] = v;
        rem -= v;
    }
    k[n - 1] = rem;
    for (int i = n; i < SPROUT_MAX_LEVELS; ++i) k[i] = 0;
}

template <int N>
__device__ __forceinline__ void grid_unrank(int D, int64_t j, int (&k)[N]) {
    int rem = D;
#pragma unroll
    for (int i = 0; i < N - 1; ++i) {
        int v = rem;
        for (;;) {
            const int64_t block = compositions(rem - v, N - 1 - i);   // points with k_i = v
            if (j < block || v == 0) break;
            j -= block;
            --v;
        }
        k[i] = v;
        rem -= v;
    }
    k[N - 1] = rem;
}

}  // namespace sprout
