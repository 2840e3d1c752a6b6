// closed_loop.cu -- closed-loop profiles ("the
// average energy consumption and processing time for recent requests at each
// level"; reading L20).  The open-loop path takes e and p as inputs; here they
// follow the trace: per (region, xi) chain, in interval order, the profile of
// level L is the mean E and T of the last W requests this chain ran at level
// L (the caller's prior while none has), the interval's LP is solved with it
// (lp_cell.cuh, the same arithmetic as step 1), and the interval's requests
// are replayed and pushed into their level's window.
//
// Chains cost very different times (an interval is scanned back until every
// level its mix reaches has W requests, so a level with a small share makes
// the scan deep): two small kernels first estimate each chain's time from
// the LP on the priors and plan the launch order (MULTIFIT packing of the
// chains into the resident slots, then planned start order), so long chains
// do not start last.  A chain gets 512 threads (one CTA per SM) when the
// intervals are long, 256 otherwise.
//
// A chain is sequential in time by definition, but only the LP decisions and
// the windows are: once every interval's thresholds are known, the cell
// totals are exactly the open-loop totals of those thresholds.  So the chain
// kernel below (one CTA per (region, xi) chain) does only what is sequential
// -- each interval's LP, and the window update, for which it needs just the
// interval's LAST W requests of each level: it scans the interval backwards
// and stops as soon as every level the mix can reach has W of them (on C4
// about a quarter of the requests) -- and sprout_abi.cu then runs the
// streaming simulate kernel (trace_sim.cu) over all requests with the solved
// thresholds for the cell and segment totals.  The window of a level is a
// ring of its last W (class, tokens) entries in shared memory, appended in
// request order from a scratch indexed by reverse rank, so it keeps FIFO
// order exactly.  With E = ef + et*tok (reading L11) the window mean is a
// function of per-class counts and token sums -- exact integers -- so the
// profile, and the LP decision it feeds, are bit-identical to the oracle's.
#include <algorithm>
#include <cstdio>
#include <cuda_runtime.h>
#include "sprout_device.cuh"
#include "sprout_kernels.cuh"
#include "lp_cell.cuh"

namespace sprout {

#ifndef SPROUT_CL_TIMING_NO_MEM
#define SPROUT_CL_TIMING_NO_MEM 0
#endif
// threads per chain: 512 (one CTA per SM) when the intervals are long enough
// that fewer, larger scan pieces pay; 256 (two per SM) for short intervals,
// where a piece covers the whole interval and a 16-warp barrier only costs
constexpr int kClThreadsLong = 512, kClThreadsShort = 256;
constexpr int64_t kClLongInterval = 2 * 8 * kClThreadsShort;   // mean requests per interval for 512

__device__ __forceinline__ uint32_t cl_half(uint4 u, int k) {   // u16 token k of a 16-byte group
    const uint32_t w = (k >> 1) == 0 ? u.x : (k >> 1) == 1 ? u.y : (k >> 1) == 2 ? u.z : u.w;
    return (k & 1) ? (w >> 16) : (w & 0xFFFFu);
}

// level of a draw in a chain: pinned ? 0 : min(#{i : w >= T_i}, max_level) (a6)
template <int N>
__device__ __forceinline__ int cl_level(uint32_t w, const uint32_t (&T)[N > 1 ? N - 1 : 1], int ml, bool pinned) {
    int L = 0;
#pragma unroll
    for (int i = 0; i + 1 < N; ++i) L += (w >= T[i]) ? 1 : 0;
    L = L < ml ? L : ml;
    return pinned ? 0 : L;
}


// 8 consecutive requests [c0, c0 + 8) of a piece: tokens (one 128-bit load
// per plane), flags, the 8 selection draws (two Philox calls, reading L10)
template <int N>
struct Chunk {
    uint4 tk[N];
    uint2 fw;
    uint32_t w[8];
};
template <int N, bool FLAGS = true>
__device__ __forceinline__ void load_chunk(const ClosedArgs &a, int64_t c0, bool any, Chunk<N> &ch) {
    if (any) {
#pragma unroll
#if SPROUT_CL_TIMING_NO_MEM   // timing-only A/B: every chunk from one 2 KB window (cache hits)
        for (int L = 0; L < N; ++L) ch.tk[L] = __ldca(reinterpret_cast<const uint4 *>(a.tokens + (size_t)L * a.pitch + (c0 & 1023)));
#else
        for (int L = 0; L < N; ++L) ch.tk[L] = __ldcs(reinterpret_cast<const uint4 *>(a.tokens + (size_t)L * a.pitch + c0));
#endif
        ch.fw = (FLAGS && a.flags) ? __ldcs(reinterpret_cast<const uint2 *>(a.flags + c0)) : make_uint2(0u, 0u);
        const uint64_t blk = (a.first_request + (uint64_t)c0) >> 2;
#if SPROUT_CL_TIMING_NO_PHILOX   // timing-only A/B: a cheap hash instead of the draws (wrong levels)
#pragma unroll
        for (int k = 0; k < 8; ++k) ch.w[k] = ((uint32_t)blk + 0x9E3779B9u * (uint32_t)(k + 1)) * 0x85EBCA6Bu;
#else
        const Philox4 d0 = philox4x32_10_rk((uint32_t)blk, (uint32_t)(blk >> 32), 0u, 0u, a.rk0, a.rk1);
        const Philox4 d1 = philox4x32_10_rk((uint32_t)(blk + 1), (uint32_t)((blk + 1) >> 32), 0u, 0u, a.rk0, a.rk1);
#pragma unroll
        for (int k = 0; k < 4; ++k) { ch.w[k] = d0.v[k]; ch.w[4 + k] = d1.v[k]; }
#endif
    } else {
#pragma unroll
        for (int L = 0; L < N; ++L) ch.tk[L] = make_uint4(0u, 0u, 0u, 0u);
        ch.fw = make_uint2(0u, 0u);
#pragma unroll
        for (int k = 0; k < 8; ++k) ch.w[k] = 0u;
    }
}
__device__ __forceinline__ uint32_t flag_byte(uint2 fw, int k) { return ((k < 4 ? fw.x : fw.y) >> (8 * (k & 3))) & 0xFFu; }

// L2 prefetch of the piece starting at local request p0 (up to s1): one 128-byte
// line per thread, 32 lines per token plane and 16 of flags
template <int N, int TH>
__device__ __forceinline__ void prefetch_piece(const ClosedArgs &a, int64_t p0, int64_t s1, int tid) {
    constexpr int kLines = 8 * TH * 2 / 128;   // the lines of one token plane of a piece
    if (SPROUT_CL_TIMING_NO_MEM || p0 >= s1) return;
    if (tid < kLines * N) {
        const int q = tid / kLines, l = tid % kLines;
        const int64_t r = p0 + 64 * (int64_t)l;
        if (r < s1) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.tokens + (size_t)q * a.pitch + r));
    } else if (a.flags && tid < kLines * N + kLines / 2) {
        const int64_t r = p0 + 128 * (int64_t)(tid - kLines * N);
        if (r < s1) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.flags + r));
    }
}

// One CTA per (region, xi) chain, sequential over the region's intervals.
// Per interval: thread 0 forms the profile from the window sums and solves
// the LP (lp_cell.cuh; the solution arrays receive x, thresholds, ...);
// then the interval is scanned BACKWARDS from its end in pieces of
// 8 * threads requests (8 per thread: one 128-bit load per token plane, two
// Philox calls), each request's level found with the interval's thresholds,
// and its reverse rank among the interval's level-L requests (a block-wide
// suffix scan of per-thread counts) decides whether it is among the last W:
// if so its (class, tokens) go to scratch slot [L][rank].  The scan stops
// as soon as every level the interval's mix can reach has W such requests
// (on C4 about a quarter of the requests), or at the interval start.  The
// scratch entries are then appended to the level's FIFO ring in request
// order, evicting the oldest, with exact integer window sums.  The cell and
// segment totals are not accumulated here: once every interval's thresholds
// are known they are exactly the open-loop totals of those thresholds, and
// the caller (sprout_abi.cu) runs the streaming simulate kernel for them.
template <int N, int NCM, bool FLAGS, int TH>
__global__ void __launch_bounds__(TH, TH >= 512 ? 1 : 2) cl_window_kernel(const __grid_constant__ ClosedArgs a) {
    constexpr int kClThreads = TH, kClWarps = TH / 32, kClPiece = 8 * TH;   // a piece: 8 requests per thread
    extern __shared__ uint32_t dyn[];                        // ring [N][W], then scratch [N][W]
    __shared__ unsigned long long wsum[N][NCM][2];          // window: requests, tokens per (level, class)
    __shared__ int head[N], size[N];
    __shared__ uint32_t thr_s[N > 1 ? N - 1 : 1];
    __shared__ int ml_s, ok_s, act_s, seg_ok_s;
    __shared__ uint32_t seen[N];                             // level-L requests scanned so far (from the end)
    __shared__ uint32_t wtot[2][kClWarps][N];                // per-warp counts of a piece (double-buffered by piece parity)
    __shared__ int part[kClWarps][N * NCM * 2];              // per-warp window deltas of the interval
    const int W = a.W, NC = a.NC;
    uint32_t *ring = dyn, *scr = dyn + (size_t)N * W;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int chain = a.chain_order ? a.chain_order[blockIdx.x] : (int)blockIdx.x;   // longest first
    const int rl = chain / a.X, j = chain % a.X;
#if SPROUT_CL_TIMING_PRINT
    long long cyc_lp = 0, cyc_scan = 0, cyc_merge = 0;
    unsigned long long t_start;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif
    const int r = a.r0 + rl;                                 // global region
    const CostConst &cost = a.cost;
    if (tid < N) { head[tid] = 0; size[tid] = 0; }
    for (int i = tid; i < N * NCM * 2; i += kClThreads) (&wsum[0][0][0])[i] = 0ull;
    // the chain's constants (thread 0 solves the LPs) and the first interval's inputs
    double pe[N], pp[N], qc[N], kmin_r = 0.0, kmax_r = 0.0, xi_j = 0.0;
    if (tid == 0) {
#pragma unroll
        for (int L = 0; L < N; ++L) { pe[L] = a.e[(int64_t)r * N + L]; pp[L] = a.p[(int64_t)r * N + L]; qc[L] = a.q[(int64_t)r * N + L]; }
        kmin_r = a.kmin[r]; kmax_r = a.kmax[r]; xi_j = a.xi[j];
    }
    const int64_t sfirst = (int64_t)r * a.T - a.first_segment;
    int64_t nx0 = a.seg_offsets[sfirst], nx1 = a.seg_offsets[sfirst + 1];
    double nk0 = tid == 0 ? a.k0[(int64_t)r * a.T] : 0.0;
    double nq[N];
#pragma unroll
    for (int L = 0; L < N; ++L) nq[L] = (tid == 0 && a.q_seg) ? a.q_seg[(int64_t)r * a.T * N + L] : 0.0;
#if SPROUT_CL_TIMING_NO_LP
    LpCell<N> o_keep;
#endif
    __syncthreads();
    for (int64_t t = 0; t < a.T; ++t) {
        const int64_t s = (int64_t)r * a.T + t;          // global segment (k0, profiles)
        const int64_t sl = s - a.first_segment;          // local segment (offsets, outputs)
        const int64_t s0 = nx0, s1 = nx1;
        const double k0_s = nk0;
        double qv[N];
#pragma unroll
        for (int L = 0; L < N; ++L) qv[L] = a.q_seg ? nq[L] : qc[L];
        if (t + 1 < a.T) {   // the next interval's inputs, one interval ahead
            nx0 = s1;
            nx1 = a.seg_offsets[sl + 2];
            if (tid == 0) {
                nk0 = a.k0[s + 1];
                if (a.q_seg) {
#pragma unroll
                    for (int L = 0; L < N; ++L) nq[L] = a.q_seg[(s + 1) * N + L];
                }
            }
        }
        // the interval's last piece (the backward scan's first): warps 1.. load it and
        // take its draws while thread 0 solves the LP (warp 0 loads it after)
        const int64_t e_al = (s1 + 7) & ~(int64_t)7;
        Chunk<N> ch;
        const int64_t c00 = e_al - kClPiece + 8 * (int64_t)tid;
        const bool any0 = s0 <= s1 && c00 + 8 > s0 && c00 < s1 && s1 <= a.n_requests && s0 >= 0;
        if (warp != 0) load_chunk<N, FLAGS>(a, c00, any0, ch);
#if SPROUT_CL_TIMING_PRINT
        long long ph0 = clock64();
#endif
        // ---- the interval's LP with the closed-loop profile ----
        if (tid == 0) {
            const int64_t cell = sl * a.X + j;
            double e[N], p[N], q[N];
#pragma unroll
            for (int L = 0; L < N; ++L) {
                q[L] = qv[L];
                unsigned long long m = 0;
#pragma unroll
                for (int cc = 0; cc < NCM; ++cc) m += cc < NC ? wsum[L][cc][0] : 0ull;
                if (m == 0) {
                    e[L] = pe[L];
                    p[L] = pp[L];
                } else {
                    double se = 0.0, sp = 0.0;
#pragma unroll
                    for (int cc = 0; cc < NCM; ++cc) {
                        if (cc >= NC) break;
                        const double nc = (double)wsum[L][cc][0], kc = (double)wsum[L][cc][1];
                        se = __dadd_rn(se, __dadd_rn(__dmul_rn(nc, cost.ef[cc][L]), __dmul_rn(kc, cost.et[cc][L])));
                        sp = __dadd_rn(sp, __dadd_rn(__dmul_rn(nc, cost.pf[cc][L]), __dmul_rn(kc, cost.pt[cc][L])));
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
#if SPROUT_CL_TIMING_NO_LP   // timing-only A/B: the first interval's LP reused
            if (t == 0) lp_cell<N>(k0_s, kmin_r, kmax_r, xi_j, e, p, q, a.k1, a.pue, 0, 0, j, o_keep);
            o = o_keep;
#else
            lp_cell<N>(k0_s, kmin_r, kmax_r, xi_j, e, p, q, a.k1, a.pue, 0, 0, j, o);
#endif
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
            const bool ok = o.status == SPROUT_CELL_OK;
            ok_s = ok;
            // levels the mix can reach (a6 is a step function of the draw with steps at the
            // thresholds, so evaluating it at 0, 2^32 - 1 and on both sides of every
            // threshold finds them all); opted-out requests reach L0
            int act = FLAGS ? 1 : 0;
            if (ok) {
                act |= 1 << cl_level<N>(0u, o.T, o.max_level, false);
                act |= 1 << cl_level<N>(0xFFFFFFFFu, o.T, o.max_level, false);
#pragma unroll
                for (int i = 0; i + 1 < N; ++i) {
                    act |= 1 << cl_level<N>(o.T[i], o.T, o.max_level, false);
                    if (o.T[i] > 0u) act |= 1 << cl_level<N>(o.T[i] - 1u, o.T, o.max_level, false);
                }
            }
            act_s = act;
            seg_ok_s = s0 >= 0 && s0 <= s1 && s1 <= a.n_requests && (s1 - s0) < (int64_t)0xFFFFFFFFll;
        }
        if (tid < N) seen[tid] = 0u;
        __syncthreads();
        const bool run = seg_ok_s && ok_s;
#if SPROUT_CL_TIMING_PRINT
        long long ph1 = clock64();
#endif
        uint32_t T[N > 1 ? N - 1 : 1];
#pragma unroll
        for (int i = 0; i + 1 < N; ++i) T[i] = thr_s[i];
        const int ml = ml_s;
        uint32_t thr_on[N > 1 ? N - 1 : 1];   // thresholds below the max level count
#pragma unroll
        for (int i = 0; i + 1 < N; ++i) thr_on[i] = i < ml ? 0xFFu : 0u;
        // ---- backward scan: the interval's last W requests of every reachable level ----
        if (run) {
            if (warp == 0) load_chunk<N, FLAGS>(a, c00, any0, ch);
            const int64_t b_al = s0 & ~(int64_t)7;
            const int n_pieces = (int)((e_al - b_al + kClPiece - 1) / kClPiece);
            uint32_t seen_r = 0u;   // lane L < N: level-L requests scanned so far (every warp the same)
            for (int pi = 0; pi < n_pieces; ++pi) {
                const int64_t base = e_al - (int64_t)(pi + 1) * kClPiece;
                prefetch_piece<N, TH>(a, base - 2 * (int64_t)kClPiece, s1, tid);
                const int64_t c0 = base + 8 * (int64_t)tid;
                if (pi > 0) load_chunk<N, FLAGS>(a, c0, c0 + 8 > s0 && c0 < s1, ch);
                // valid requests of the chunk: inside [s0, s1) (a bit range) with a class < NC
                uint32_t valid;
                {
                    const int64_t lo = min(max(s0 - c0, (int64_t)0), (int64_t)8), hi = min(max(s1 - c0, (int64_t)0), (int64_t)8);
                    valid = ((1u << (uint32_t)hi) - 1u) & ~((1u << (uint32_t)lo) - 1u);
                }
                // the chunk's requests of each level as bit masks: ge_i = {k : w_k >= T_i} over
                // the thresholds below the interval's max level -- an OK cell's thresholds are
                // non-decreasing, so #{i < ml : w >= T_i} = min(#{i : w >= T_i}, ml), the a6
                // level -- with opted-out requests at level 0
                uint32_t ge[N > 1 ? N - 1 : 1], pin = 0u;
#pragma unroll
                for (int i = 0; i + 1 < N; ++i) ge[i] = 0u;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (FLAGS) {
                        const uint32_t fb = flag_byte(ch.fw, k);
                        if (((fb >> 1) & 3u) >= (uint32_t)NC) valid &= ~(1u << k);
                        pin |= (fb & 1u) << k;
                    }
#pragma unroll
                    for (int i = 0; i + 1 < N; ++i) ge[i] |= (ch.w[k] >= T[i] ? 1u : 0u) << k;
                }
                uint32_t lm[N];   // valid requests of level L
                {
                    uint32_t below = valid;   // valid requests not yet placed at a lower level
#pragma unroll
                    for (int L = 0; L + 1 < N; ++L) {
                        const uint32_t up = ge[L] & thr_on[L] & ~pin;
                        lm[L] = below & ~up;
                        below &= up;
                    }
                    lm[N - 1] = below;
                }
                // requests of each level in LATER threads of the warp (suffix scan)
                uint32_t after[N];
                uint32_t (*wt)[N] = wtot[pi & 1];
#pragma unroll
                for (int L = 0; L < N; ++L) {
                    const uint32_t c = (uint32_t)__popc(lm[L]);
                    uint32_t x = c;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const uint32_t y = __shfl_down_sync(0xFFFFFFFFu, x, d);
                        if (lane + d < 32) x += y;
                    }
                    after[L] = x - c;
                    if (lane == 0) wt[warp][L] = x;
                }
                __syncthreads();
                // lane L of every warp: level-L requests in later warps of the piece, and the
                // piece total; then the stop test (identical in every warp)
                uint32_t later = 0u, ptot = 0u;
                if (lane < N) {
#pragma unroll
                    for (int w2 = 0; w2 < kClWarps; ++w2) {
                        const uint32_t v = wt[w2][lane];
                        later += w2 > warp ? v : 0u;
                        ptot += v;
                    }
                }
#pragma unroll
                for (int L = 0; L < N; ++L) after[L] += __shfl_sync(0xFFFFFFFFu, later + seen_r, L);
                seen_r += ptot;
                const bool done = __all_sync(0xFFFFFFFFu, lane >= N || !((act_s >> lane) & 1) || seen_r >= (uint32_t)W);
                // the thread's requests from the latest: reverse rank = level-L requests after it;
                // only levels whose window is not yet full need ranks
#pragma unroll
                for (int L = 0; L < N; ++L) {
                    if (after[L] >= (uint32_t)W || !lm[L]) continue;
#pragma unroll
                    for (int k = 7; k >= 0; --k) {
                        if (!((lm[L] >> k) & 1u)) continue;
                        const uint32_t rho = after[L]++;
                        if (rho < (uint32_t)W)
                            scr[(size_t)L * W + rho] =
                                (FLAGS ? (((flag_byte(ch.fw, k) >> 1) & 3u) << 16) : 0u) | cl_half(ch.tk[L], k);
                    }
                }
                if (done) break;
            }
            if (warp == 0 && lane < N) seen[lane] = seen_r;
            __syncthreads();   // every scratch entry written, seen final
        }
#if SPROUT_CL_TIMING_PRINT
        long long ph2 = clock64();
#endif
        // ---- append the scratch entries (forward order) to the rings, evicting the oldest ----
        int dn[N][NCM], dk[N][NCM];
#pragma unroll
        for (int L = 0; L < N; ++L)
#pragma unroll
            for (int cc = 0; cc < NCM; ++cc) { dn[L][cc] = 0; dk[L][cc] = 0; }
        if (run) {
#pragma unroll
            for (int L = 0; L < N; ++L) {
                const uint32_t k = min(seen[L], (uint32_t)W);
                const uint32_t h = (uint32_t)head[L], sz = (uint32_t)size[L];
                for (uint32_t i = tid; i < k; i += kClThreads) {
                    uint32_t pos = h + sz + i;   // < 3W
                    pos = pos >= (uint32_t)W ? pos - (uint32_t)W : pos;
                    pos = pos >= (uint32_t)W ? pos - (uint32_t)W : pos;
                    uint32_t *rp = ring + (size_t)L * W + pos;
                    if (sz + i >= (uint32_t)W) {   // the slot's old entry is the oldest: it leaves
                        const uint32_t old = *rp;
#pragma unroll
                        for (int cc = 0; cc < NCM; ++cc)
                            if ((uint32_t)cc == (old >> 16)) { dn[L][cc] -= 1; dk[L][cc] -= (int)(old & 0xFFFFu); }
                    }
                    const uint32_t nw = scr[(size_t)L * W + (k - 1u - i)];
                    *rp = nw;
#pragma unroll
                    for (int cc = 0; cc < NCM; ++cc)
                        if ((uint32_t)cc == (nw >> 16)) { dn[L][cc] += 1; dk[L][cc] += (int)(nw & 0xFFFFu); }
                }
            }
        }
        if (t + 1 < a.T) {   // the next interval's last two pieces into L2
            const int64_t n0 = a.seg_offsets[sl + 1], n1 = a.seg_offsets[sl + 2];
            if (n0 >= 0 && n0 <= n1 && n1 <= a.n_requests) {
                const int64_t e2 = (n1 + 7) & ~(int64_t)7;
                prefetch_piece<N, TH>(a, e2 - kClPiece, n1, tid);
                prefetch_piece<N, TH>(a, e2 - 2 * kClPiece, n1, tid);
            }
        }
        {
            int v = 0;
#pragma unroll
            for (int L = 0; L < N; ++L)
#pragma unroll
                for (int cc = 0; cc < NCM; ++cc) {
                    const uint32_t x0 = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)dn[L][cc]);
                    const uint32_t x1 = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)dk[L][cc]);
                    if (lane == 0) { part[warp][v] = (int)x0; part[warp][v + 1] = (int)x1; }
                    v += 2;
                }
        }
        __syncthreads();
        for (int v = tid; v < N * NCM * 2; v += kClThreads) {
            long long sum = 0;
            for (int w2 = 0; w2 < kClWarps; ++w2) sum += (long long)part[w2][v];
            unsigned long long *wp = &wsum[0][0][0] + v;
            *wp = (unsigned long long)((long long)*wp + sum);
        }
        if (tid < N && run) {
            const uint32_t k = min(seen[tid], (uint32_t)W);
            const uint32_t sz = (uint32_t)size[tid];
            const uint32_t ev = sz + k > (uint32_t)W ? sz + k - (uint32_t)W : 0u;
            const uint32_t hh = (uint32_t)head[tid] + ev;
            head[tid] = (int)(hh >= (uint32_t)W ? hh - (uint32_t)W : hh);
            size[tid] = (int)min(sz + k, (uint32_t)W);
        }
        __syncthreads();
#if SPROUT_CL_TIMING_PRINT
        const long long ph3 = clock64();
        cyc_lp += ph1 - ph0; cyc_scan += ph2 - ph1; cyc_merge += ph3 - ph2;
#endif
    }
#if SPROUT_CL_TIMING_PRINT
    if (tid == 0) {
        unsigned long long t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        printf("CHAIN %d %d %d %.3f %.3f %lld %lld %lld\n", (int)blockIdx.x, rl, j, t_start * 1e-6, (t_end - t_start) * 1e-6,
               cyc_lp, cyc_scan, cyc_merge);
    }
#endif
}

// Scheduling only (no result depends on it).  A chain's run time is its
// intervals' scan depths, and those vary a lot between chains: an interval
// is scanned back until each level the mix reaches has W requests, so a
// level the mix gives a small fraction x_L needs W / x_L requests, up to the
// whole interval.  The estimate solves each interval's LP with the priors
// (the open-loop decision; the closed-loop profiles move it, the depth order
// of the chains much less) and counts pieces; the chains then launch longest
// first, so the long ones do not start last behind a wave of short ones.
template <int N>
__global__ void __launch_bounds__(256) cl_estimate_kernel(const __grid_constant__ ClosedArgs a, int piece) {
    __shared__ float red[8];
    const int c = blockIdx.x, rl = c / a.X, j = c % a.X, r = a.r0 + rl;
    double e[N], p[N], qc[N];
#pragma unroll
    for (int L = 0; L < N; ++L) { e[L] = a.e[(int64_t)r * N + L]; p[L] = a.p[(int64_t)r * N + L]; qc[L] = a.q[(int64_t)r * N + L]; }
    const double kmin = a.kmin[r], kmax = a.kmax[r], xi = a.xi[j];
    float acc = 0.0f;
    for (int64_t t = threadIdx.x; t < a.T; t += blockDim.x) {
        const int64_t s = (int64_t)r * a.T + t, sl = s - a.first_segment;
        double q[N];
#pragma unroll
        for (int L = 0; L < N; ++L) q[L] = a.q_seg ? a.q_seg[s * N + L] : qc[L];
        LpCell<N> o;
        lp_cell<N>(a.k0[s], kmin, kmax, xi, e, p, q, a.k1, a.pue, 0, 0, j, o);
        const double m = (double)max(a.seg_offsets[sl + 1] - a.seg_offsets[sl], (int64_t)0);
        double need = 0.0;
        if (o.status == SPROUT_CELL_OK) {
#pragma unroll
            for (int L = 0; L < N; ++L)
                if (o.x[L] > 0.0) need = fmax(need, (double)a.W / o.x[L]);
        }
        // the requests scanned, in pieces, plus the interval's fixed part (LP, window merge,
        // barriers), which costs about 1.9 pieces' time (C4, per-chain phase timing:
        // 4.1 us per interval + 2.2 us per 4,096 requests scanned)
        acc += 1.9f + (float)(fmin(m, need) / (double)piece);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, d);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.0f;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        a.chain_cost[c] = t;
    }
}

// The launch order.  The block scheduler hands each freed slot (SMs x CTAs per
// SM) the next chain in launch order, i.e. list scheduling; longest-first
// list scheduling leaves the short chains to start last on busy slots.  So:
// MULTIFIT -- binary search of a capacity C for which first-fit-decreasing
// packs the chains into `slots` bins -- and then the chains in the order of
// their planned start times, which list scheduling reproduces when the
// estimates hold (each freed slot is the one whose chain was planned to end
// first).  No capacity packs (cannot happen for C >= sum / slots + max, the
// search's upper end): longest first.  One CTA; the first-fit scan is one
// warp, each lane holding every 32nd bin's load.
constexpr int kClMaxOrdered = 4000;   // chains scheduled (48 KB of static shared memory); more run in index order
constexpr int kClMaxSlots = 32 * 32;  // bins of the first-fit scan (32 per lane)

__global__ void __launch_bounds__(1024) cl_order_kernel(const float *cost, int n, int slots, int *order) {
    __shared__ float e[kClMaxOrdered], start[kClMaxOrdered];
    __shared__ int byc[kClMaxOrdered];   // chain ids by estimate, largest first
    __shared__ float bound[2];
    __shared__ int feasible;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < n; i += blockDim.x) e[i] = cost[i];
    __syncthreads();
    for (int i = tid; i < n; i += blockDim.x) {   // rank: larger first, ties by id
        const float ci = e[i];
        int rank = 0;
        for (int k = 0; k < n; ++k) rank += (e[k] > ci || (e[k] == ci && k < i)) ? 1 : 0;
        byc[rank] = i;
    }
    if (tid == 0) {
        float sum = 0.0f, mx = 0.0f;
        for (int i = 0; i < n; ++i) { sum += e[i]; mx = fmaxf(mx, e[i]); }
        bound[0] = fmaxf(mx, sum / (float)slots);           // no schedule is shorter
        bound[1] = sum / (float)slots + mx;                  // list scheduling reaches this
        feasible = 0;
    }
    __syncthreads();
    if (warp == 0) {
        float lo = bound[0], hi = bound[1];
        bool have = false;
        for (int it = 0; it < 14; ++it) {
            const float C = (it == 0) ? hi : 0.5f * (lo + hi);
            float load[kClMaxSlots / 32];
#pragma unroll
            for (int b = 0; b < kClMaxSlots / 32; ++b) load[b] = 0.0f;
            bool ok = true;
            for (int q = 0; q < n && ok; ++q) {
                const int c = byc[q];
                const float ec = e[c];
                int first = -1;   // the first bin (index b * 32 + lane) the chain fits in
#pragma unroll
                for (int b = 0; b < kClMaxSlots / 32; ++b) {
                    const bool fits = b * 32 + lane < slots && load[b] + ec <= C;
                    const unsigned bal = __ballot_sync(0xFFFFFFFFu, fits);
                    if (first < 0 && bal) first = b * 32 + __ffs(bal) - 1;
                }
                if (first < 0) {
                    ok = false;
                } else if ((first & 31) == lane) {
#pragma unroll
                    for (int b = 0; b < kClMaxSlots / 32; ++b)
                        if (b == (first >> 5)) { start[c] = load[b]; load[b] += ec; }
                }
            }
            if (ok) { hi = C; have = true; } else { lo = C; }
            if (it > 0 && hi - lo <= 1e-3f * hi) break;
        }
        // the starts of the final (smallest feasible) capacity
        if (have) {
            float load[kClMaxSlots / 32];
#pragma unroll
            for (int b = 0; b < kClMaxSlots / 32; ++b) load[b] = 0.0f;
            for (int q = 0; q < n; ++q) {
                const int c = byc[q];
                const float ec = e[c];
                int first = -1;
#pragma unroll
                for (int b = 0; b < kClMaxSlots / 32; ++b) {
                    const bool fits = b * 32 + lane < slots && load[b] + ec <= hi;
                    const unsigned bal = __ballot_sync(0xFFFFFFFFu, fits);
                    if (first < 0 && bal) first = b * 32 + __ffs(bal) - 1;
                }
                if (first >= 0 && (first & 31) == lane) {
#pragma unroll
                    for (int b = 0; b < kClMaxSlots / 32; ++b)
                        if (b == (first >> 5)) { start[c] = load[b]; load[b] += ec; }
                }
                if (first < 0) have = false;
            }
        }
        if (lane == 0) feasible = have ? 1 : 0;
    }
    __syncthreads();
    if (!feasible) {
        for (int i = tid; i < n; i += blockDim.x) order[i] = byc[i];
        return;
    }
    for (int i = tid; i < n; i += blockDim.x) {   // by planned start, ties: larger estimate first
        const int ci = byc[i];
        const float si = start[ci];
        int rank = 0;
        for (int k = 0; k < n; ++k) {
            const float sk = start[byc[k]];
            rank += (sk < si || (sk == si && k < i)) ? 1 : 0;
        }
        order[rank] = ci;
    }
}


cudaError_t launch_closed_loop(ClosedArgs &a, cudaStream_t stream, int *launches) {
    if ((int64_t)a.R_local * a.X == 0) return cudaSuccess;
    a.n_groups = a.X;
    const int64_t blocks = (int64_t)a.R_local * a.X;
    const int64_t local_segments = (int64_t)a.R_local * a.T;
    const int TH = a.n_requests >= kClLongInterval * local_segments ? kClThreadsLong : kClThreadsShort;
    if (a.chain_cost && a.chain_order && blocks <= kClMaxOrdered) {
#define CL_EST(NN) case NN: cl_estimate_kernel<NN><<<(unsigned)blocks, 256, 0, stream>>>(a, 8 * TH); break;
        switch (a.n) {
            CL_EST(1) CL_EST(2) CL_EST(3) CL_EST(4) CL_EST(5) CL_EST(6) CL_EST(7) CL_EST(8)
            default: return cudaErrorInvalidValue;
        }
#undef CL_EST
        int dev = 0, sms = 0, per_sm = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e != cudaSuccess) return e;
        const size_t smem_chain = (size_t)2 * a.n * a.W * 4;
#define CL_OCC(NN)                                                                                \
    case NN:                                                                                      \
        e = TH == kClThreadsLong                                                                  \
                ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(                                  \
                      &per_sm, cl_window_kernel<NN, 1, false, kClThreadsLong>, TH, smem_chain)    \
                : cudaOccupancyMaxActiveBlocksPerMultiprocessor(                                  \
                      &per_sm, cl_window_kernel<NN, 1, false, kClThreadsShort>, TH, smem_chain);  \
        break;
        switch (a.n) {
            CL_OCC(1) CL_OCC(2) CL_OCC(3) CL_OCC(4) CL_OCC(5) CL_OCC(6) CL_OCC(7) CL_OCC(8)
            default: return cudaErrorInvalidValue;
        }
#undef CL_OCC
        if (e != cudaSuccess) return e;
        const int slots = std::min(std::max(sms * std::max(per_sm, 1), 1), kClMaxSlots);
        cl_order_kernel<<<1, 1024, 0, stream>>>(a.chain_cost, (int)blocks, slots, a.chain_order);
        *launches += 2;
    } else {
        a.chain_order = nullptr;
    }
    const size_t smem = (size_t)2 * a.n * a.W * 4;
    cudaError_t e = cudaSuccess;
#define CL_LAUNCH(NN, NCM_)                                                                       \
    {                                                                                             \
        auto kern = TH == kClThreadsLong                                                          \
                        ? (a.flags ? cl_window_kernel<NN, NCM_, true, kClThreadsLong>             \
                                   : cl_window_kernel<NN, NCM_, false, kClThreadsLong>)           \
                        : (a.flags ? cl_window_kernel<NN, NCM_, true, kClThreadsShort>            \
                                   : cl_window_kernel<NN, NCM_, false, kClThreadsShort>);         \
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);   \
        if (e != cudaSuccess) return e;                                                           \
        kern<<<(unsigned)blocks, TH, smem, stream>>>(a);                                          \
    }
#define CL_N(NN)                                                                                  \
    case NN:                                                                                      \
        if (a.NC > 1) CL_LAUNCH(NN, kMaxClasses)                                                  \
        else CL_LAUNCH(NN, 1)                                                                     \
        break;
    switch (a.n) {
        CL_N(1) CL_N(2) CL_N(3) CL_N(4) CL_N(5) CL_N(6) CL_N(7) CL_N(8)
        default: return cudaErrorInvalidValue;
    }
#undef CL_N
#undef CL_LAUNCH
    ++*launches;
    return cudaGetLastError();
}

}  // namespace sprout
