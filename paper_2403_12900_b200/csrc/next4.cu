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

namespace sprout {

// ---- the Oracle scheme (reading L23) ----
// One CTA per segment (persistent, a queue of segments).  Pass 1 over the
// segment: every request's carbon at every level (Eq. 1), its cheapest level
// m (lowest index among ties), its latent best level l*, the base choice
// (opted-out: L0, else m) and its statistics; the candidates (not opted out,
// l* != m) are compacted in request order with key = the bits of
// Delta = C_l* - C_m (a non-negative double: bit order = value order) and
// their move (class, m, l*, tokens at m and l*).  A stable LSD radix sort of
// the keys (8 passes of 8 bits, passes with one digit skipped) orders them
// by (Delta, request index).  Then every xi cell takes the first
// need = ceil(b m) - base hits of them: chunk sums of the moves, a block
// scan, and per cell the partial chunk.  Integer statistics are exact; fp64
// totals follow from them in trace_sim.cu's closed form.
constexpr int kOrThreads = 512;
constexpr int kOrWarps = kOrThreads / 32;

// per CTA: keys x2 (8 B), indices x2 (4 B), moves (8 B) per request of a segment, then the
// chunk sums of the moves ([kOrThreads][<= 2*4*8 + 3] signed 64-bit)
constexpr int kOrMaxMv = 2 * kMaxClasses * kMaxLevels + 3;
__host__ __device__ inline size_t or_cta_bytes(int64_t cap) {
    return (size_t)32 * (size_t)(cap > 0 ? cap : 1) + (size_t)kOrThreads * kOrMaxMv * 8;
}

// the queue ticket (256 B), then one scratch region per CTA of the persistent grid (one CTA per SM)
size_t oracle_scheme_workspace_bytes(int64_t cap) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return 256 + (size_t)sms * or_cta_bytes(cap);
}

// radix digits of the candidates' 64-bit keys: 11 bits (six passes over the key,
// those with a single digit value skipped); per-warp digit histograms in dynamic
// shared memory ([kOrWarps][kOrDigits] u32, 128 KB)
constexpr int kOrBits = 11;
constexpr int kOrDigits = 1 << kOrBits;
constexpr size_t kOrDynSmem = (size_t)kOrWarps * kOrDigits * 4;

struct OrSmem {
    uint32_t hist[kOrWarps][256];   // pass 1: per-warp candidate counts
    uint32_t dtot[kOrDigits];       // the sort: per-digit totals, then exclusive digit offsets
    uint32_t wsum[kOrWarps];
    int64_t seg;
    int skip;
};

template <int N, int NCM>
__global__ void __launch_bounds__(kOrThreads) oracle_scheme_kernel(const __grid_constant__ N4Args a) {
    __shared__ OrSmem sm;
    extern __shared__ uint32_t hdyn[];   // [kOrWarps][kOrDigits]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t cap = a.cap;
    uint8_t *scr = a.scratch + (size_t)blockIdx.x * or_cta_bytes(cap);
    unsigned long long *keyA = reinterpret_cast<unsigned long long *>(scr);
    unsigned long long *keyB = keyA + cap;
    uint32_t *idxA = reinterpret_cast<uint32_t *>(keyB + cap);
    uint32_t *idxB = idxA + cap;
    unsigned long long *move = reinterpret_cast<unsigned long long *>(idxB + cap);   // by local request index
    const int NC = a.NC;
    uint32_t err = 0u;
    // layout of the per-segment sums (u64): [0, NCM*N) base cnt, [NCM*N, 2NCM*N) base tok,
    // then hits, wins, losses, valid requests, candidates; segment: per class count, pinned, tok[N]
    constexpr int B_CNT = 0, B_TOK = NCM * N, B_HIT = 2 * NCM * N, B_WIN = B_HIT + 1, B_LOSS = B_HIT + 2,
                  B_M = B_HIT + 3, B_NC = B_HIT + 4, S_BASE = B_HIT + 5;   // + NCM * (N + 2)
    constexpr int NSUM = S_BASE + NCM * (N + 2);
    __shared__ unsigned long long tot[NSUM];
    __shared__ unsigned long long red[kOrWarps][NSUM];
    for (;;) {
        if (tid == 0) sm.seg = (int64_t)atomicAdd(a.queue, 1u);
        __syncthreads();
        const int64_t sl = sm.seg;
        if (sl >= a.n_segments) break;
        const int64_t s = a.first_segment + sl, r = s / a.T;
        const int64_t s0 = a.seg_offsets[sl], s1 = a.seg_offsets[sl + 1];
        const bool good = s0 >= 0 && s0 <= s1 && s1 <= a.n_requests;
        const bool fits = s1 - s0 <= cap;
        if (tid == 0 && !good) err |= SPROUT_TRACE_BAD_OFFSETS;
        if (tid == 0 && good && !fits) err |= SPROUT_TRACE_TOO_LONG;
        const int64_t m_all = (good && fits) ? s1 - s0 : 0;
        const double kp = __dmul_rn(a.k0[s], a.pue);
        const double *qr = q_row(a, s);
        uint32_t Tq[N > 1 ? N - 1 : 1];
        int mlq;
        vec_thresholds<N>(qr, Tq, mlq);
        // ---- pass 1: tiles of kOrThreads * 4 requests (each thread an aligned quad) ----
        uint32_t bc[NCM][N], bt[NCM][N], sc[NCM][N + 2];
        uint32_t hit = 0u, win = 0u, loss = 0u, mv = 0u;
#pragma unroll
        for (int c = 0; c < NCM; ++c) {
#pragma unroll
            for (int L = 0; L < N; ++L) { bc[c][L] = 0u; bt[c][L] = 0u; }
#pragma unroll
            for (int f = 0; f < N + 2; ++f) sc[c][f] = 0u;
        }
        uint32_t ncand = 0u;   // candidates so far (block-uniform, running)
        for (int64_t t0 = s0 & ~(int64_t)3; t0 < s0 + m_all; t0 += 4 * kOrThreads) {
            const int64_t q0 = t0 + 4 * (int64_t)tid;
            const uint64_t blk = (a.first_request + (uint64_t)q0) >> 2;
            const bool anyq = q0 + 4 > s0 && q0 < s0 + m_all;
            Philox4 dp;
            if (anyq) dp = n4_words(a, blk, 2u);
            unsigned long long key[4], mvk[4];
            uint32_t isc = 0u;   // bit k: request k is a candidate
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t rq = q0 + k;
                key[k] = 0ull; mvk[k] = 0ull;
                if (!(anyq && rq >= s0 && rq < s0 + m_all)) continue;
                const uint32_t fb = a.flags ? a.flags[rq] : 0u;
                const int c = (int)((fb >> 1) & 3u);
                if (c >= NC) { err |= SPROUT_TRACE_BAD_CLASS; continue; }
                const bool pinned = fb & 1u;
                uint32_t tk[N];
                double C[N];
#pragma unroll
                for (int L = 0; L < N; ++L) {
                    tk[L] = a.tokens[(size_t)L * a.pitch + rq];
                    C[L] = n4_carbon(a, kp, c, L, tk[L]);
                }
                int mbest = 0;
#pragma unroll
                for (int L = 1; L < N; ++L) mbest = C[L] < C[mbest] ? L : mbest;
                int ls = n4_level<N>(dp.v[k], Tq, mlq, false);
                const int ch = pinned ? 0 : mbest;
                double cm = C[0], cl = C[0];
                uint32_t tm = tk[0], tl = tk[0];
#pragma unroll
                for (int L = 0; L < N; ++L) {
                    if (L == mbest) { cm = C[L]; tm = tk[L]; }
                    if (L == ls) { cl = C[L]; tl = tk[L]; }
                }
#pragma unroll
                for (int cc = 0; cc < NCM; ++cc) {
                    if (cc != c) continue;
                    sc[cc][0] += 1u;
                    sc[cc][1] += pinned ? 1u : 0u;
#pragma unroll
                    for (int L = 0; L < N; ++L) {
                        sc[cc][2 + L] += tk[L];
                        if (L == ch) { bc[cc][L] += 1u; bt[cc][L] += tk[L]; }
                    }
                }
                hit += ch == ls ? 1u : 0u;
                win += (ch != 0 && ls == ch) ? 1u : 0u;
                loss += (ch != 0 && ls == 0) ? 1u : 0u;
                mv += 1u;
                if (!pinned && ls != mbest) {
                    isc |= 1u << k;
                    key[k] = (unsigned long long)__double_as_longlong(__dsub_rn(cl, cm));
                    mvk[k] = (unsigned long long)c | ((unsigned long long)mbest << 2) | ((unsigned long long)ls << 5) |
                             ((unsigned long long)tm << 8) | ((unsigned long long)tl << 24);
                }
            }
            // compaction in request order: block-wide exclusive scan of the candidate counts
            const uint32_t cnt4 = __popc(isc);
            uint32_t x = cnt4;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, d);
                if (lane >= d) x += y;
            }
            if (lane == 31) sm.hist[0][warp] = x;
            __syncthreads();
            uint32_t base = ncand, total = 0u;
            for (int w2 = 0; w2 < kOrWarps; ++w2) {
                const uint32_t v = sm.hist[0][w2];
                base += w2 < warp ? v : 0u;
                total += v;
            }
            base += x - cnt4;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (!((isc >> k) & 1u)) continue;
                keyA[base] = key[k];
                idxA[base] = (uint32_t)(q0 + k - s0);
                move[q0 + k - s0] = mvk[k];
                ++base;
            }
            ncand += total;
            __syncthreads();   // sm.hist reused
        }
        // ---- block sums of pass 1 ----
        {
            int v = 0;
            auto put = [&](uint32_t x) {
                const uint32_t sx = __reduce_add_sync(0xFFFFFFFFu, x);
                if (lane == 0) red[warp][v] = sx;
                ++v;
            };
#pragma unroll
            for (int c = 0; c < NCM; ++c)
#pragma unroll
                for (int L = 0; L < N; ++L) put(bc[c][L]);
#pragma unroll
            for (int c = 0; c < NCM; ++c)
#pragma unroll
                for (int L = 0; L < N; ++L) put(bt[c][L]);
            put(hit); put(win); put(loss); put(mv); put(0u);
#pragma unroll
            for (int c = 0; c < NCM; ++c)
#pragma unroll
                for (int f = 0; f < N + 2; ++f) put(sc[c][f]);
        }
        __syncthreads();
        if (tid < NSUM) {
            unsigned long long t = 0ull;
            for (int w2 = 0; w2 < kOrWarps; ++w2) t += red[w2][tid];
            tot[tid] = tid == B_NC ? (unsigned long long)ncand : t;
        }
        __syncthreads();
        const int64_t nc = (int64_t)ncand;
        // ---- stable LSD radix sort of (key, index), kOrBits bits per pass ----
        unsigned long long *ks = keyA, *kd = keyB;
        uint32_t *is = idxA, *id = idxB;
        const int64_t per = (nc + kOrWarps - 1) / kOrWarps;   // warp w: [w*per, (w+1)*per)
        const int64_t lo = min(nc, (int64_t)warp * per), hi = min(nc, lo + per);
        uint32_t *wh = hdyn + (size_t)warp * kOrDigits;      // this warp's digit histogram
        for (int sh = 0; sh < 64; sh += kOrBits) {
            const unsigned long long dmask = (unsigned long long)(kOrDigits - 1);
            for (int i = lane; i < kOrDigits; i += 32) wh[i] = 0u;
            __syncwarp();
            for (int64_t i = lo + lane; i < hi; i += 32) atomicAdd(&wh[(ks[i] >> sh) & dmask], 1u);
            __syncthreads();
            // per-digit totals; skip the pass if one digit holds every key
            if (tid == 0) sm.skip = 0;
            for (int d = tid; d < kOrDigits; d += kOrThreads) {
                uint32_t t = 0u;
                for (int w2 = 0; w2 < kOrWarps; ++w2) t += hdyn[(size_t)w2 * kOrDigits + d];
                sm.dtot[d] = t;
            }
            __syncthreads();
            for (int d = tid; d < kOrDigits; d += kOrThreads)
                if ((int64_t)sm.dtot[d] == nc) sm.skip = 1;
            __syncthreads();
            if (sm.skip) continue;
            // exclusive offsets in (digit, warp) order: a block scan of the digit totals
            // (thread t owns digits [t*D, (t+1)*D), D = kOrDigits / kOrThreads), then
            // each digit's warps in order
            {
                constexpr int D = kOrDigits / kOrThreads;
                uint32_t loc[D], run = 0u;
#pragma unroll
                for (int k = 0; k < D; ++k) { loc[k] = run; run += sm.dtot[tid * D + k]; }
                uint32_t x = run;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, d);
                    if (lane >= d) x += y;
                }
                if (lane == 31) sm.wsum[warp] = x;
                __syncthreads();
                uint32_t before = x - run;
                for (int w2 = 0; w2 < warp; ++w2) before += sm.wsum[w2];
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    const int dg = tid * D + k;
                    uint32_t off = before + loc[k];
                    for (int w2 = 0; w2 < kOrWarps; ++w2) {
                        uint32_t *h = &hdyn[(size_t)w2 * kOrDigits + dg];
                        const uint32_t v = *h;
                        *h = off;
                        off += v;
                    }
                }
            }
            __syncthreads();
            // scatter, each warp its range in order: rank among equal digits by match_any
            for (int64_t i0 = lo; i0 < hi; i0 += 32) {
                const int64_t i = i0 + lane;
                const bool in = i < hi;
                const unsigned long long kv = in ? ks[i] : 0ull;
                const uint32_t dg = in ? (uint32_t)((kv >> sh) & dmask) : (uint32_t)kOrDigits + (uint32_t)lane;
                const uint32_t peers = __match_any_sync(0xFFFFFFFFu, dg);
                if (in) {
                    const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
                    const uint32_t pos = wh[dg] + rank;
                    kd[pos] = kv;
                    id[pos] = is[i];
                }
                __syncwarp();
                if (in && (__ffs(peers) - 1) == lane) wh[dg] += __popc(peers);
                __syncwarp();
            }
            __syncthreads();
            unsigned long long *tk2 = ks; ks = kd; kd = tk2;
            uint32_t *ti = is; is = id; id = ti;
        }
        // ---- chunk sums of the moves over the sorted candidates ----
        // per move: cnt[c][m] -1, cnt[c][l*] +1, tok[c][m] -tok_m, tok[c][l*] +tok_l*, hits +1,
        // wins +[l* != 0], losses -[m != 0 and l* == 0]
        const int64_t chunk = (nc + kOrThreads - 1) / kOrThreads;
        const int64_t c_lo = min(nc, (int64_t)tid * chunk), c_hi = min(nc, c_lo + chunk);
        constexpr int MV = 2 * NCM * N + 3;   // [cnt c,L][tok c,L] hits wins losses (signed)
        auto apply = [&](unsigned long long mvv, long long (&acc)[MV]) {
            const int c = (int)(mvv & 3u), mf = (int)((mvv >> 2) & 7u), lt = (int)((mvv >> 5) & 7u);
            const long long tm = (long long)((mvv >> 8) & 0xFFFFu), tl = (long long)((mvv >> 24) & 0xFFFFu);
#pragma unroll
            for (int cc = 0; cc < NCM; ++cc)
#pragma unroll
                for (int L = 0; L < N; ++L) {
                    if (cc != c) continue;
                    if (L == mf) { acc[cc * N + L] -= 1; acc[NCM * N + cc * N + L] -= tm; }
                    if (L == lt) { acc[cc * N + L] += 1; acc[NCM * N + cc * N + L] += tl; }
                }
            acc[2 * NCM * N] += 1;
            acc[2 * NCM * N + 1] += lt != 0 ? 1 : 0;
            acc[2 * NCM * N + 2] -= (mf != 0 && lt == 0) ? 1 : 0;
        };
        long long acc[MV];
#pragma unroll
        for (int v = 0; v < MV; ++v) acc[v] = 0;
        for (int64_t i = c_lo; i < c_hi; ++i) apply(move[is[i]], acc);
        // block exclusive scan of the chunk sums ([kOrThreads][MV] signed, after the moves)
        long long *csum = reinterpret_cast<long long *>(move + cap);
        if (nc > 0) {
#pragma unroll
            for (int v = 0; v < MV; ++v) csum[(size_t)tid * MV + v] = acc[v];
        }
        __syncthreads();
        if (tid < MV && nc > 0) {
            long long run = 0;
            for (int t2 = 0; t2 < kOrThreads; ++t2) {
                const long long v = csum[(size_t)t2 * MV + tid];
                csum[(size_t)t2 * MV + tid] = run;
                run += v;
            }
        }
        __syncthreads();
        // ---- every xi cell of the segment ----
        const double kmin_r = a.kmin[r], kmax_r = a.kmax[r], k0_s = a.k0[s];
        const unsigned long long mreq = tot[B_M], hit0 = tot[B_HIT];
        for (int j = tid; j < a.X; j += kOrThreads) {
            const int64_t cell = sl * a.X + j;
            const double xi = a.xi[j];
            bool ok = (xi >= 0.0 && xi <= 1.0) && finite_nonneg(k0_s) && finite_nonneg(kmin_r) &&
                      finite_nonneg(kmax_r) && (kmax_r >= kmin_r) && good && fits;
#pragma unroll
            for (int i = 0; i < N; ++i) ok = ok && (qr[i] >= 0.0 && qr[i] <= 1.0);
            long long cur[MV];
#pragma unroll
            for (int v = 0; v < MV; ++v) cur[v] = 0;
            uint8_t status = ok ? SPROUT_CELL_OK : SPROUT_CELL_INVALID;
            if (ok) {
                // Eq. 3 floor (lp_cell.cuh's formula and order) and k = ceil(fl(b * m))
                double f = 0.0;
                if (kmax_r > kmin_r) {
                    f = __ddiv_rn(__dsub_rn(k0_s, kmin_r), __dsub_rn(kmax_r, kmin_r));
                    f = f < 0.0 ? 0.0 : (f > 1.0 ? 1.0 : f);
                }
                const double b = __dmul_rn(__dsub_rn(1.0, __dmul_rn(f, xi)), qr[0]);
                const double kk = ceil(__dmul_rn(b, (double)mreq));
                int64_t need = (int64_t)kk - (int64_t)hit0;
                if (need < 0) need = 0;
                if (need > nc) { need = nc; status = SPROUT_CELL_INFEASIBLE; }
                if (need > 0) {
                    const int64_t owner = min((need - 1) / chunk, (int64_t)kOrThreads - 1);
#pragma unroll
                    for (int v = 0; v < MV; ++v) cur[v] = csum[(size_t)owner * MV + v];
                    for (int64_t i = owner * chunk; i < need; ++i) apply(move[is[i]], cur);
                }
            }
            a.cell_status_out[cell] = status;
            double E = 0.0, Tm = 0.0, Q = 0.0;
            for (int c = 0; c < NC; ++c) {
#pragma unroll
                for (int L = 0; L < N; ++L) {
                    unsigned long long cn = 0ull, tk2 = 0ull;
                    if (ok && c < NCM) {
                        cn = (unsigned long long)((long long)tot[B_CNT + c * N + L] + cur[c * N + L]);
                        tk2 = (unsigned long long)((long long)tot[B_TOK + c * N + L] + cur[NCM * N + c * N + L]);
                    }
                    a.cnt[(cell * NC + c) * N + L] = cn;
                    a.tok[(cell * NC + c) * N + L] = tk2;
                    const double n_ = (double)cn, t_ = (double)tk2;
                    E += n_ * a.cost.ef[c][L] + t_ * a.cost.et[c][L];
                    Tm += n_ * a.cost.pf[c][L] + t_ * a.cost.pt[c][L];
                    Q += n_ * qr[L];
                }
            }
            a.energy[cell] = E;
            a.time_s[cell] = Tm;
            a.carbon[cell] = ok ? __dmul_rn(k0_s, a.pue) * E + a.k1 * Tm : 0.0;
            a.quality[cell] = Q;
            a.stats[cell * 3 + 0] = ok ? (unsigned long long)((long long)hit0 + cur[2 * NCM * N]) : 0ull;
            a.stats[cell * 3 + 1] = ok ? (unsigned long long)((long long)tot[B_WIN] + cur[2 * NCM * N + 1]) : 0ull;
            a.stats[cell * 3 + 2] = ok ? (unsigned long long)((long long)tot[B_LOSS] + cur[2 * NCM * N + 2]) : 0ull;
        }
        if (tid == 0) {   // segment statistics and the Base counterfactual (write_seg_stats' formulas)
            double bE = 0.0, bT = 0.0, mm = 0.0;
            for (int c = 0; c < NC; ++c) {
                const unsigned long long *ss = tot + S_BASE + (c < NCM ? c : 0) * (N + 2);
                const unsigned long long mc = c < NCM ? ss[0] : 0ull;
                a.seg_count[sl * NC + c] = mc;
                a.seg_pinned[sl * NC + c] = c < NCM ? ss[1] : 0ull;
                for (int L = 0; L < N; ++L) a.seg_tok[(sl * NC + c) * N + L] = c < NCM ? ss[2 + L] : 0ull;
                const unsigned long long t0 = c < NCM ? ss[2] : 0ull;
                bE += (double)mc * a.cost.ef[c][0] + (double)t0 * a.cost.et[c][0];
                bT += (double)mc * a.cost.pf[c][0] + (double)t0 * a.cost.pt[c][0];
                mm += (double)mc;
            }
            const double kp2 = a.k0[s] * a.pue;
            a.seg_base[sl * 4 + 0] = bE;
            a.seg_base[sl * 4 + 1] = bT;
            a.seg_base[sl * 4 + 2] = kp2 * bE + a.k1 * bT;
            a.seg_base[sl * 4 + 3] = mm * qr[0];
        }
        __syncthreads();
    }
    err = __reduce_or_sync(0xFFFFFFFFu, err);
    if (lane == 0 && err) atomicOr(a.trace_status, err);
}

cudaError_t launch_oracle_scheme(N4Args &a, cudaStream_t stream, int *launches) {
    round_keys(a);
    if (cudaMemsetAsync(a.queue, 0, 4, stream) != cudaSuccess) return cudaErrorUnknown;
    if (a.n_segments == 0) return cudaSuccess;
    int64_t grid = sm_count();
    if (grid > a.n_segments) grid = a.n_segments;
#define OR_CASE(NN)                                                                                     \
    case NN: {                                                                                          \
        auto kern = a.NC > 1 ? oracle_scheme_kernel<NN, kMaxClasses> : oracle_scheme_kernel<NN, 1>;     \
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kOrDynSmem); \
        if (e != cudaSuccess) return e;                                                                 \
        kern<<<(unsigned)grid, kOrThreads, kOrDynSmem, stream>>>(a);                                    \
        break;                                                                                          \
    }
    switch (a.n) {
        OR_CASE(1) OR_CASE(2) OR_CASE(3) OR_CASE(4) OR_CASE(5) OR_CASE(6) OR_CASE(7) OR_CASE(8)
        default: return cudaErrorInvalidValue;
    }
#undef OR_CASE
    ++*launches;
    return cudaGetLastError();
}

}  // namespace sprout
