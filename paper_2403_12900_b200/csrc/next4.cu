// next4.cu -- SURVEY 8(f) NEXT-4: per-request outputs (the per-request carbon
// normalised to Base of Fig. eval2), the latent best level of every
// request and the head-to-head preference statistics against Base (P:168,
// P:190; readings L21, L22), and the Oracle scheme (reading
// L23).  The oracle counterparts are orc_request_outputs, orc_preference and
// orc_oracle_scheme (oracle/sprout_oracle.c); the arithmetic is written out
// independently here.
#include <cuda_runtime.h>
#include "sprout_device.cuh"
#include "sprout_kernels.cuh"

namespace sprout {

constexpr int kN4Warps = 8;

// Inverse-CDF thresholds of a probability vector (a4): cum_i sequential in
// fp64, T_i = min(ceil(cum_i * 2^32), 2^32) stored saturated, max_level the
// first i with T_i = 2^32 (else n - 1).  Used with q as the vector: the
// latent best level of reading L21.
template <int N>
__device__ __forceinline__ void vec_thresholds(const double *v, uint32_t (&T)[N > 1 ? N - 1 : 1], int &ml) {
    ml = N - 1;
    double cum = 0.0;
    bool found = false;
#pragma unroll
    for (int i = 0; i + 1 < N; ++i) {
        cum = __dadd_rn(cum, v[i]);
        const double cl = ceil(__dmul_rn(cum, 4294967296.0));
        if (cl >= 4294967296.0) {
            T[i] = 0xFFFFFFFFu;
            if (!found) { ml = i; found = true; }
        } else {
            T[i] = (uint32_t)(uint64_t)cl;
        }
    }
}

// the a6 rule: min(#{i : w >= T_i}, max_level); opted-out requests at L0
template <int N>
__device__ __forceinline__ int n4_level(uint32_t w, const uint32_t (&T)[N > 1 ? N - 1 : 1], int ml, bool pinned) {
    int L = 0;
#pragma unroll
    for (int i = 0; i + 1 < N; ++i) L += (w >= T[i]) ? 1 : 0;
    L = L < ml ? L : ml;
    return pinned ? 0 : L;
}

__device__ __forceinline__ const double *q_row(const N4Args &a, int64_t s) {
    return a.q + (a.profile_per_interval ? s : (s / a.T)) * a.n;
}

// Eq. 1 for one request at one level, in the oracle's operation
// order without contraction (reading L7): E = ef + et*tok, Tq = pf + pt*tok,
// C = (k0*PUE)*E + k1*Tq.
__device__ __forceinline__ double n4_carbon(const N4Args &a, double kp, int c, int L, uint32_t tok) {
    const double t = (double)tok;
    const double e = __dadd_rn(a.cost.ef[c][L], __dmul_rn(a.cost.et[c][L], t));
    const double p = __dadd_rn(a.cost.pf[c][L], __dmul_rn(a.cost.pt[c][L], t));
    return __dadd_rn(__dmul_rn(kp, e), __dmul_rn(a.k1, p));
}

// Philox words of quad blk on stream `stream` (readings L10 / L21)
__device__ __forceinline__ Philox4 n4_words(const N4Args &a, uint64_t blk, uint32_t stream) {
    return philox4x32_10_rk((uint32_t)blk, (uint32_t)(blk >> 32), stream, 0u, a.rk0, a.rk1);
}

// ---- per-request outputs of one cell column ----
// One warp per segment, each lane an aligned quad of 4 requests per step.
template <int N>
__global__ void __launch_bounds__(32 * kN4Warps) request_outputs_kernel(const __grid_constant__ N4Args a) {
    const uint32_t lane = threadIdx.x & 31u;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int j = a.column;
    for (int64_t sl = gw; sl < a.n_segments; sl += nw) {
        const int64_t s = a.first_segment + sl, cell = sl * a.X + j;
        const int64_t s0 = a.seg_offsets[sl], s1 = a.seg_offsets[sl + 1];
        if (!(s0 >= 0 && s0 <= s1 && s1 <= a.n_requests)) continue;
        const bool ok = a.cell_status[cell] == SPROUT_CELL_OK;
        uint32_t T[N > 1 ? N - 1 : 1], Tq[N > 1 ? N - 1 : 1];
#pragma unroll
        for (int i = 0; i + 1 < N; ++i) T[i] = a.threshold[cell * (N - 1) + i];
        const int ml = a.max_level[cell];
        int mlq;
        vec_thresholds<N>(q_row(a, s), Tq, mlq);
        const double kp = __dmul_rn(a.k0[s], a.pue);
        const double qnan = __longlong_as_double(0x7ff8000000000000ll);
        for (int64_t q0 = (s0 & ~(int64_t)3) + 4 * (int64_t)lane; q0 < s1; q0 += 128) {
            const uint64_t blk = (a.first_request + (uint64_t)q0) >> 2;
            const Philox4 d = n4_words(a, blk, 0u), dp = n4_words(a, blk, 2u);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t r = q0 + k;
                if (r < s0 || r >= s1) continue;
                const uint32_t fb = a.flags ? a.flags[r] : 0u;
                const int c = (int)((fb >> 1) & 3u);
                const int ls = n4_level<N>(dp.v[k], Tq, mlq, false);
                if (a.pref_out) a.pref_out[r] = (uint8_t)ls;
                if (!ok || c >= a.NC) {
                    a.level_out[r] = 0xFF;
                    a.carbon_out[r] = qnan;
                    a.base_out[r] = qnan;
                    a.ratio_out[r] = qnan;
                    continue;
                }
                const int L = n4_level<N>(d.v[k], T, ml, fb & 1u);
                const double cl = n4_carbon(a, kp, c, L, a.tokens[(size_t)L * a.pitch + r]);
                const double c0 = n4_carbon(a, kp, c, 0, a.tokens[r]);
                a.level_out[r] = (uint8_t)L;
                a.carbon_out[r] = cl;
                a.base_out[r] = c0;
                a.ratio_out[r] = __ddiv_rn(cl, c0);
            }
        }
    }
}

// ---- head-to-head statistics per cell ----
// One warp per segment: lanes take aligned quads (both Philox streams once
// per quad); every cell of the segment is evaluated from the same words and
// its (hits, wins, losses) summed over the warp into shared counters.
template <int N>
__global__ void __launch_bounds__(32 * kN4Warps) pref_stats_kernel(const __grid_constant__ N4Args a) {
    extern __shared__ uint32_t cnt_s[];                       // [warps][X][3]
    const uint32_t lane = threadIdx.x & 31u;
    const int warp = threadIdx.x >> 5;
    uint32_t *cnt = cnt_s + (size_t)warp * a.X * 3;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t sl = gw; sl < a.n_segments; sl += nw) {
        const int64_t s = a.first_segment + sl;
        const int64_t s0 = a.seg_offsets[sl], s1 = a.seg_offsets[sl + 1];
        for (int i = lane; i < a.X * 3; i += 32) cnt[i] = 0u;
        __syncwarp();
        const bool good = s0 >= 0 && s0 <= s1 && s1 <= a.n_requests;
        uint32_t Tq[N > 1 ? N - 1 : 1];
        int mlq;
        vec_thresholds<N>(q_row(a, s), Tq, mlq);
        for (int64_t q0 = (s0 & ~(int64_t)3); good && q0 < s1; q0 += 128) {
            const int64_t mq = q0 + 4 * (int64_t)lane;
            const uint64_t blk = (a.first_request + (uint64_t)mq) >> 2;
            const Philox4 d = n4_words(a, blk, 0u), dp = n4_words(a, blk, 2u);
            uint32_t fbk[4];
            int lsk[4];
            bool vk[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t r = mq + k;
                fbk[k] = (r >= s0 && r < s1 && a.flags) ? a.flags[r] : 0u;
                vk[k] = r >= s0 && r < s1 && (int)((fbk[k] >> 1) & 3u) < a.NC;
                lsk[k] = n4_level<N>(dp.v[k], Tq, mlq, false);
            }
            for (int j = 0; j < a.X; ++j) {
                const int64_t cell = sl * a.X + j;
                uint32_t T[N > 1 ? N - 1 : 1];
#pragma unroll
                for (int i = 0; i + 1 < N; ++i) T[i] = a.threshold[cell * (N - 1) + i];
                const int ml = a.max_level[cell];
                const bool ok = a.cell_status[cell] == SPROUT_CELL_OK;
                uint32_t h = 0u, wn = 0u, ls_ = 0u;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (!(vk[k] && ok)) continue;
                    const int L = n4_level<N>(d.v[k], T, ml, fbk[k] & 1u);
                    h += L == lsk[k] ? 1u : 0u;
                    wn += (L != 0 && lsk[k] == L) ? 1u : 0u;
                    ls_ += (L != 0 && lsk[k] == 0) ? 1u : 0u;
                }
                const uint32_t H = __reduce_add_sync(0xFFFFFFFFu, h), Wn = __reduce_add_sync(0xFFFFFFFFu, wn),
                               Ls = __reduce_add_sync(0xFFFFFFFFu, ls_);
                if (lane == 0) { cnt[j * 3 + 0] += H; cnt[j * 3 + 1] += Wn; cnt[j * 3 + 2] += Ls; }
            }
        }
        __syncwarp();
        for (int i = lane; i < a.X * 3; i += 32) a.stats[sl * a.X * 3 + i] = cnt[i];
        __syncwarp();
    }
}

static int sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

static void round_keys(N4Args &a) {
    uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32);
    for (int r = 0; r < 10; ++r) {
        a.rk0[r] = k0; a.rk1[r] = k1;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
}

cudaError_t launch_request_outputs(N4Args &a, cudaStream_t stream, int *launches) {
    if (a.n_segments == 0) return cudaSuccess;
    round_keys(a);
    int64_t blocks = (a.n_segments + kN4Warps - 1) / kN4Warps;
    if (blocks > (int64_t)sm_count() * 16) blocks = (int64_t)sm_count() * 16;
#define RO_CASE(NN) case NN: request_outputs_kernel<NN><<<(unsigned)blocks, 32 * kN4Warps, 0, stream>>>(a); break;
    switch (a.n) {
        RO_CASE(1) RO_CASE(2) RO_CASE(3) RO_CASE(4) RO_CASE(5) RO_CASE(6) RO_CASE(7) RO_CASE(8)
        default: return cudaErrorInvalidValue;
    }
#undef RO_CASE
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_pref_stats(N4Args &a, cudaStream_t stream, int *launches) {
    if (a.n_segments == 0) return cudaSuccess;
    round_keys(a);
    int warps = kN4Warps;
    while (warps > 1 && (size_t)warps * a.X * 12 > 96 * 1024) warps >>= 1;
    const size_t smem = (size_t)warps * a.X * 12;
    if (smem > 200 * 1024) return cudaErrorInvalidValue;
    int64_t blocks = (a.n_segments + warps - 1) / warps;
    if (blocks > (int64_t)sm_count() * 16) blocks = (int64_t)sm_count() * 16;
    cudaError_t e = cudaSuccess;
#define PS_CASE(NN)                                                                                      \
    case NN:                                                                                             \
        e = cudaFuncSetAttribute(pref_stats_kernel<NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        if (e != cudaSuccess) return e;                                                                  \
        pref_stats_kernel<NN><<<(unsigned)blocks, 32 * warps, smem, stream>>>(a);                         \
        break;
    switch (a.n) {
        PS_CASE(1) PS_CASE(2) PS_CASE(3) PS_CASE(4) PS_CASE(5) PS_CASE(6) PS_CASE(7) PS_CASE(8)
        default: return cudaErrorInvalidValue;
    }
#undef PS_CASE
    ++*launches;
    return cudaGetLastError();
}

}  // namespace sprout
