// closed_loop.cu -- closed-loop profiles ("the
// average energy consumption and processing time for recent requests at each
// level"; reading L20).  The open-loop path takes e and p as inputs; here they
// follow the trace: per (region, xi) chain, in interval order, the profile of
// level L is the mean E and T of the last W requests this chain ran at level
// L (the caller's prior while none has), the interval's LP is solved with it
// (lp_cell.cuh, the same arithmetic as step 1), and the interval's requests
// are replayed and pushed into their level's window.
//
// The chain is sequential in time by definition, so one CTA runs one chain;
// inside an interval its 256 threads take one request each per chunk.  The
// window of level L is a ring of the last W (class, tokens) pairs in shared
// memory; a request's slot is fixed by its rank among the chunk's level-L
// requests (warp ballots + a prefix over the 8 warps), so the ring holds the
// FIFO order exactly.  With E = ef + et*tok (reading L11) the window mean is
// a function of per-class counts and token sums -- exact integers, summed in
// any order -- so the profile, and the LP decision it feeds, are
// bit-identical to the oracle's.
#include <cuda_runtime.h>
#include "sprout_device.cuh"
#include "sprout_kernels.cuh"
#include "lp_cell.cuh"

namespace sprout {

constexpr int kClThreads = 256;
constexpr int kClWarps = kClThreads / 32;

template <int N>
__global__ void __launch_bounds__(kClThreads) closed_loop_kernel(const __grid_constant__ ClosedArgs a) {
    extern __shared__ uint32_t ring[];                      // [N][W] (class << 16 | tokens)
    __shared__ unsigned long long wsum[N][kMaxClasses][2];  // window: requests, tokens per (level, class)
    __shared__ unsigned long long csum[kMaxClasses][N][2];  // the interval's cell: requests, tokens
    __shared__ int head[N], size[N];
    __shared__ uint32_t thr_s[N > 1 ? N - 1 : 1];
    __shared__ int ml_s, ok_s;
    __shared__ int wcount[kClWarps][N];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int chain = blockIdx.x;
    const int r = chain / a.X, j = chain % a.X;
    const int W = a.W, NC = a.NC;
    const CostConst &cost = a.cost;
    if (tid < N) { head[tid] = 0; size[tid] = 0; }
    for (int i = tid; i < N * kMaxClasses * 2; i += kClThreads) (&wsum[0][0][0])[i] = 0ull;
    __syncthreads();
    uint32_t err = 0u;
    for (int64_t t = 0; t < a.T; ++t) {
        const int64_t s = (int64_t)r * a.T + t;
        const int64_t cell = s * a.X + j;
        if (tid == 0) {
            double e[N], p[N], q[N];
#pragma unroll
            for (int L = 0; L < N; ++L) {
                q[L] = a.q[(int64_t)r * N + L];
                unsigned long long m = 0;
                for (int c = 0; c < NC; ++c) m += wsum[L][c][0];
                if (m == 0) {
                    e[L] = a.e[(int64_t)r * N + L];
                    p[L] = a.p[(int64_t)r * N + L];
                } else {
                    double se = 0.0, sp = 0.0;
                    for (int c = 0; c < NC; ++c) {
                        const double nc = (double)wsum[L][c][0], kc = (double)wsum[L][c][1];
                        se = __dadd_rn(se, __dadd_rn(__dmul_rn(nc, cost.ef[c][L]), __dmul_rn(kc, cost.et[c][L])));
                        sp = __dadd_rn(sp, __dadd_rn(__dmul_rn(nc, cost.pf[c][L]), __dmul_rn(kc, cost.pt[c][L])));
                    }
                    e[L] = __ddiv_rn(se, (double)m);
                    p[L] = __ddiv_rn(sp, (double)m);
                }
                if (a.profile) {
                    a.profile[(cell * 2 + 0) * N + L] = e[L];
                    a.profile[(cell * 2 + 1) * N + L] = p[L];
                }
            }
            LpCell<N> o;
            lp_cell<N>(a.k0[s], a.kmin[r], a.kmax[r], a.xi[j], e, p, q, a.k1, a.pue, 0, 0, j, o);
#pragma unroll
            for (int i = 0; i < N; ++i) a.x[cell * N + i] = o.x[i];
            a.objective[cell] = o.objective;
            a.q_lb[cell] = o.q_lb;
            a.vertex[cell] = o.vertex;
            a.cell_status[cell] = o.status;
#pragma unroll
            for (int i = 0; i + 1 < N; ++i) { a.threshold[cell * (N - 1) + i] = o.T[i]; thr_s[i] = o.T[i]; }
            a.max_level[cell] = o.max_level;
            ml_s = o.max_level;
            ok_s = o.status == SPROUT_CELL_OK;
        }
        for (int i = tid; i < kMaxClasses * N * 2; i += kClThreads) (&csum[0][0][0])[i] = 0ull;
        __syncthreads();
        const bool cell_ok = ok_s;
        uint32_t T[N > 1 ? N - 1 : 1];
#pragma unroll
        for (int i = 0; i + 1 < N; ++i) T[i] = thr_s[i];
        const int ml = ml_s;
        const int64_t s0 = a.seg_offsets[s], s1 = a.seg_offsets[s + 1];
        uint32_t cc[kMaxClasses][N], ct[kMaxClasses][N];
#pragma unroll
        for (int c = 0; c < kMaxClasses; ++c)
#pragma unroll
            for (int L = 0; L < N; ++L) { cc[c][L] = 0u; ct[c][L] = 0u; }
        if (cell_ok) {
            int64_t nchunk = 0;
            for (int64_t base = s0; base < s1; base += kClThreads, ++nchunk) {
                const int64_t rq = base + tid;
                const bool inr = rq < s1;
                int lev = -1;
                uint32_t cls = 0u, tl = 0u;
                if (inr) {
                    const uint64_t g = a.first_request + (uint64_t)rq;
                    const uint64_t blk = g >> 2;
                    const Philox4 d = philox4x32_10_rk((uint32_t)blk, (uint32_t)(blk >> 32), 0u, 0u, a.rk0, a.rk1);
                    const uint32_t k3 = (uint32_t)(g & 3u);
                    const uint32_t w = k3 == 0 ? d.v[0] : k3 == 1 ? d.v[1] : k3 == 2 ? d.v[2] : d.v[3];
                    uint32_t pin = 0u;
                    if (a.flags) {
                        const uint32_t fb = a.flags[rq];
                        pin = fb & 1u;
                        cls = (fb >> 1) & 3u;
                    }
                    if (cls >= (uint32_t)NC) {
                        err |= SPROUT_TRACE_BAD_CLASS;
                    } else {
                        int L = 0;
#pragma unroll
                        for (int i = 0; i + 1 < N; ++i) L += (w >= T[i]) ? 1 : 0;
                        L = pin ? 0 : min(L, ml);
                        lev = L;
                        tl = a.tokens[(size_t)L * a.pitch + rq];
#pragma unroll
                        for (int c = 0; c < kMaxClasses; ++c)
#pragma unroll
                            for (int LL = 0; LL < N; ++LL) {
                                const bool hit = (uint32_t)c == cls && LL == L;
                                cc[c][LL] += hit ? 1u : 0u;
                                ct[c][LL] += hit ? tl : 0u;
                            }
                    }
                }
                // window push in request order: rank among the chunk's level-L requests
                uint32_t bal[N];
#pragma unroll
                for (int L = 0; L < N; ++L) {
                    bal[L] = __ballot_sync(0xFFFFFFFFu, lev == L);
                    if (lane == 0) wcount[warp][L] = __popc(bal[L]);
                }
                __syncthreads();
                if (lev >= 0) {
                    int before = 0, total = 0;
                    for (int w2 = 0; w2 < kClWarps; ++w2) {
                        const int c2 = wcount[w2][lev];
                        before += w2 < warp ? c2 : 0;
                        total += c2;
                    }
                    uint32_t bl = bal[0];
#pragma unroll
                    for (int L = 1; L < N; ++L) bl = lev == L ? bal[L] : bl;
                    const int rank = before + __popc(bl & ((1u << lane) - 1u));
                    if (rank >= total - W) ring[lev * W + (head[lev] + rank) % W] = (cls << 16) | tl;
                }
                __syncthreads();
                if (tid < N) {
                    int total = 0;
                    for (int w2 = 0; w2 < kClWarps; ++w2) total += wcount[w2][tid];
                    head[tid] = (head[tid] + total) % W;
                    size[tid] = min(size[tid] + total, W);
                }
                __syncthreads();
                if ((nchunk & 4095) == 4095) {   // fold the 32-bit sums before they can overflow
#pragma unroll
                    for (int c = 0; c < kMaxClasses; ++c)
#pragma unroll
                        for (int L = 0; L < N; ++L) {
                            const uint32_t sc = __reduce_add_sync(0xFFFFFFFFu, cc[c][L]);
                            const uint32_t st = __reduce_add_sync(0xFFFFFFFFu, ct[c][L]);
                            if (lane == 0 && (sc | st)) { atomicAdd(&csum[c][L][0], (unsigned long long)sc);
                                                          atomicAdd(&csum[c][L][1], (unsigned long long)st); }
                            cc[c][L] = 0u; ct[c][L] = 0u;
                        }
                }
            }
        }
        // the interval's cell totals
#pragma unroll
        for (int c = 0; c < kMaxClasses; ++c)
#pragma unroll
            for (int L = 0; L < N; ++L) {
                const uint32_t sc = __reduce_add_sync(0xFFFFFFFFu, cc[c][L]);
                const uint32_t st = __reduce_add_sync(0xFFFFFFFFu, ct[c][L]);
                if (lane == 0 && (sc | st)) { atomicAdd(&csum[c][L][0], (unsigned long long)sc);
                                              atomicAdd(&csum[c][L][1], (unsigned long long)st); }
            }
        // the windows' sums for the next interval (exact integers, any order)
        for (int i = tid; i < N * kMaxClasses * 2; i += kClThreads) (&wsum[0][0][0])[i] = 0ull;
        __syncthreads();
        for (int L = 0; L < N; ++L) {
            uint32_t wn[kMaxClasses], wk[kMaxClasses];
#pragma unroll
            for (int c = 0; c < kMaxClasses; ++c) { wn[c] = 0u; wk[c] = 0u; }
            for (int i = tid; i < size[L]; i += kClThreads) {
                const uint32_t v = ring[L * W + i];
#pragma unroll
                for (int c = 0; c < kMaxClasses; ++c) {
                    const bool hit = (v >> 16) == (uint32_t)c;
                    wn[c] += hit ? 1u : 0u;
                    wk[c] += hit ? (v & 0xFFFFu) : 0u;
                }
            }
#pragma unroll
            for (int c = 0; c < kMaxClasses; ++c) {
                const uint32_t sn = __reduce_add_sync(0xFFFFFFFFu, wn[c]);
                const uint32_t sk = __reduce_add_sync(0xFFFFFFFFu, wk[c]);
                if (lane == 0 && (sn | sk)) { atomicAdd(&wsum[L][c][0], (unsigned long long)sn);
                                              atomicAdd(&wsum[L][c][1], (unsigned long long)sk); }
            }
        }
        __syncthreads();
        if (tid == 0) {   // cell_epilogue's formulas and order
            const double kp = a.k0[s] * a.pue;
            const double *qrow = a.q + (int64_t)r * N;
            double E = 0.0, Tm = 0.0, Q = 0.0;
            for (int c = 0; c < NC; ++c) {
#pragma unroll
                for (int L = 0; L < N; ++L) {
                    const unsigned long long cn = cell_ok ? csum[c][L][0] : 0ull, tk = cell_ok ? csum[c][L][1] : 0ull;
                    a.cnt[(cell * NC + c) * N + L] = cn;
                    a.tok[(cell * NC + c) * N + L] = tk;
                    const double n_ = (double)cn, t_ = (double)tk;
                    E += n_ * cost.ef[c][L] + t_ * cost.et[c][L];
                    Tm += n_ * cost.pf[c][L] + t_ * cost.pt[c][L];
                    Q += n_ * qrow[L];
                }
            }
            a.energy[cell] = E;
            a.time_s[cell] = Tm;
            a.carbon[cell] = cell_ok ? kp * E + a.k1 * Tm : 0.0;
            a.quality[cell] = Q;
        }
        __syncthreads();
    }
    err = __reduce_or_sync(0xFFFFFFFFu, err);
    if (lane == 0 && err) atomicOr(a.trace_status, err);
}

cudaError_t launch_closed_loop(const ClosedArgs &a, cudaStream_t stream, int *launches) {
    const int64_t chains = (int64_t)a.R * a.X;
    if (chains == 0) return cudaSuccess;
    const size_t smem = (size_t)a.n * a.W * 4;
    cudaError_t e = cudaSuccess;
#define CL_CASE(NN)                                                                                  \
    case NN: {                                                                                       \
        auto kern = closed_loop_kernel<NN>;                                                          \
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);      \
        if (e != cudaSuccess) return e;                                                              \
        kern<<<(unsigned)chains, kClThreads, smem, stream>>>(a);                                     \
        break;                                                                                       \
    }
    switch (a.n) {
        CL_CASE(1) CL_CASE(2) CL_CASE(3) CL_CASE(4) CL_CASE(5) CL_CASE(6) CL_CASE(7) CL_CASE(8)
        default: return cudaErrorInvalidValue;
    }
#undef CL_CASE
    ++*launches;
    return cudaGetLastError();
}

}  // namespace sprout
