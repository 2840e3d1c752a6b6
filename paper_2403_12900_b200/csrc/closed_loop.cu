// closed_loop.cu -- closed-loop profiles ("the
// average energy consumption and processing time for recent requests at each
// level"; reading L20).  The open-loop path takes e and p as inputs; here they
// follow the trace: per (region, xi) chain, in interval order, the profile of
// level L is the mean E and T of the last W requests this chain ran at level
// L (the caller's prior while none has), the interval's LP is solved with it
// (lp_cell.cuh, the same arithmetic as step 1), and the interval's requests
// are replayed and pushed into their level's window.
//
// A chain is sequential in time by definition; the chains of a region are
// not, and they share everything but the thresholds: the requests' draws
// (common random numbers, reading L10), tokens and flags.  So one CTA runs a
// GROUP of G chains of one region: per interval, threads 0..G-1 solve the G
// LPs; then the interval streams in pieces of kClPiece requests, each thread
// taking 8 consecutive requests (one 128-bit load per token plane, two
// Philox calls), and every request is selected in all G chains from the same
// registers.  The window of (chain, level) is a ring of the last W
// (class, tokens) entries in shared memory; a request's slot is its rank
// among the piece's requests of that chain and level (a block-wide scan of
// per-thread counts), so the ring keeps FIFO order exactly.  With
// E = ef + et*tok (reading L11) the window mean is a function of per-class
// counts and token sums -- exact integers -- so the profile, and the LP
// decision it feeds, are bit-identical to the oracle's.  The first group of
// each region also writes the segment statistics and the Base counterfactual
// (they do not depend on the chain), so the call's totals are complete.
#include <cuda_runtime.h>
#include "sprout_device.cuh"
#include "sprout_kernels.cuh"
#include "lp_cell.cuh"

namespace sprout {

constexpr int kClThreads = 256;
constexpr int kClWarps = kClThreads / 32;
constexpr int kClPiece = 8 * kClThreads;   // requests per piece: 8 per thread

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

constexpr int kClMaxPieces = 128;   // per-piece level counts kept for the window pass (intervals <= 2^20)

// 8 consecutive requests [c0, c0 + 8) of a piece: tokens (one 128-bit load
// per plane), flags, the 8 selection draws (two Philox calls, reading L10)
template <int N>
struct Chunk {
    uint4 tk[N];
    uint2 fw;
    uint32_t w[8];
};
template <int N>
__device__ __forceinline__ void load_chunk(const ClosedArgs &a, int64_t c0, bool any, Chunk<N> &ch) {
    if (any) {
#pragma unroll
        for (int L = 0; L < N; ++L) ch.tk[L] = __ldcs(reinterpret_cast<const uint4 *>(a.tokens + (size_t)L * a.pitch + c0));
        ch.fw = a.flags ? __ldcs(reinterpret_cast<const uint2 *>(a.flags + c0)) : make_uint2(0u, 0u);
        const uint64_t blk = (a.first_request + (uint64_t)c0) >> 2;
        const Philox4 d0 = philox4x32_10_rk((uint32_t)blk, (uint32_t)(blk >> 32), 0u, 0u, a.rk0, a.rk1);
        const Philox4 d1 = philox4x32_10_rk((uint32_t)(blk + 1), (uint32_t)((blk + 1) >> 32), 0u, 0u, a.rk0, a.rk1);
#pragma unroll
        for (int k = 0; k < 4; ++k) { ch.w[k] = d0.v[k]; ch.w[4 + k] = d1.v[k]; }
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
template <int N>
__device__ __forceinline__ void prefetch_piece(const ClosedArgs &a, int64_t p0, int64_t s1, int tid) {
    constexpr int kLines = kClPiece * 2 / 128;   // 32 lines of one token plane
    if (p0 >= s1) return;
    if (tid < kLines * N) {
        const int q = tid / kLines, l = tid % kLines;
        const int64_t r = p0 + 64 * (int64_t)l;
        if (r < s1) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.tokens + (size_t)q * a.pitch + r));
    } else if (a.flags && tid < kLines * N + kLines / 2) {
        const int64_t r = p0 + 128 * (int64_t)(tid - kLines * N);
        if (r < s1) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.flags + r));
    }
}

template <int N, int NCM, int G>
__global__ void __launch_bounds__(kClThreads) closed_loop_kernel(const __grid_constant__ ClosedArgs a) {
    extern __shared__ uint32_t ring[];                      // [G][N][W] class << 16 | tokens
    __shared__ unsigned long long wsum[G][N][NCM][2];       // window: requests, tokens per (chain, level, class)
    __shared__ int head[G][N], size[G][N];
    __shared__ uint32_t thr_s[G][N > 1 ? N - 1 : 1];
    __shared__ int ml_s[G], ok_s[G];
    __shared__ int seg_ok_s;
    __shared__ uint32_t pcnt[kClMaxPieces][G * N];          // level-L requests of (chain, piece)
    __shared__ uint32_t ctot[G * N], cfirst[G * N];         // interval totals; first piece holding a window entry
    __shared__ uint32_t wtot[kClWarps][G * N];              // per-warp counts (window-pass scan)
    constexpr int NCELL = G * NCM * N * 2, NDELTA = G * N * NCM * 2, NSEG = NCM * (N + 2);
    __shared__ uint32_t part[kClWarps][NDELTA];             // per-warp window deltas of the interval
    __shared__ unsigned long long part64[kClWarps][NCELL + NSEG];   // per-warp 64-bit cell / segment sums
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rl = blockIdx.x / a.n_groups, gi = blockIdx.x % a.n_groups;
    const int r = a.r0 + rl;                                 // global region
    const int j0 = gi * G;                                   // first xi of the group
    const int W = a.W, NC = a.NC;
    const bool seg_writer = gi == 0;                         // one group per region writes the segment fields
    const CostConst &cost = a.cost;
    for (int i = tid; i < G * N; i += kClThreads) { (&head[0][0])[i] = 0; (&size[0][0])[i] = 0; }
    for (int i = tid; i < G * N * NCM * 2; i += kClThreads) (&wsum[0][0][0][0])[i] = 0ull;
    __syncthreads();
    uint32_t err = 0u;
    for (int64_t t = 0; t < a.T; ++t) {
        const int64_t s = (int64_t)r * a.T + t;          // global segment (k0, profiles)
        const int64_t sl = s - a.first_segment;          // local segment (offsets, outputs)
        const int64_t s0 = a.seg_offsets[sl], s1 = a.seg_offsets[sl + 1];
        const double k0_s = a.k0[s];
        const double *qrow = a.q_seg ? a.q_seg + s * N : a.q + (int64_t)r * N;
        // ---- the G interval LPs, with the closed-loop profile ----
        if (tid < G) {
            const int c = tid, j = j0 + c;
            int ok = 0;
            if (j < a.X) {
                const int64_t cell = sl * a.X + j;
                double e[N], p[N], q[N];
#pragma unroll
                for (int L = 0; L < N; ++L) {
                    q[L] = qrow[L];
                    unsigned long long m = 0;
                    for (int cc = 0; cc < NC; ++cc) m += wsum[c][L][cc][0];
                    if (m == 0) {
                        e[L] = a.e[(int64_t)r * N + L];
                        p[L] = a.p[(int64_t)r * N + L];
                    } else {
                        double se = 0.0, sp = 0.0;
                        for (int cc = 0; cc < NC; ++cc) {
                            const double nc = (double)wsum[c][L][cc][0], kc = (double)wsum[c][L][cc][1];
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
                lp_cell<N>(k0_s, a.kmin[r], a.kmax[r], a.xi[j], e, p, q, a.k1, a.pue, 0, 0, j, o);
#pragma unroll
                for (int i = 0; i < N; ++i) a.x[cell * N + i] = o.x[i];
                a.objective[cell] = o.objective;
                a.q_lb[cell] = o.q_lb;
                a.vertex[cell] = o.vertex;
                a.cell_status[cell] = o.status;
#pragma unroll
                for (int i = 0; i + 1 < N; ++i) { a.threshold[cell * (N - 1) + i] = o.T[i]; thr_s[c][i] = o.T[i]; }
                a.max_level[cell] = o.max_level;
                ml_s[c] = o.max_level;
                ok = o.status == SPROUT_CELL_OK;
            }
            ok_s[c] = ok;
        }
        if (tid == 0) {
            const bool good = s0 >= 0 && s0 <= s1 && s1 <= a.n_requests && (s1 - s0) < (int64_t)0xFFFFFFFFll;
            seg_ok_s = good;
            if (!good) err |= SPROUT_TRACE_BAD_OFFSETS;
        }
        for (int i = tid; i < kClMaxPieces * G * N; i += kClThreads) (&pcnt[0][0])[i] = 0u;
        for (int i = tid; i < G * N; i += kClThreads) ctot[i] = 0u;
        for (int i = tid; i < kClWarps * (NCELL + NSEG); i += kClThreads) (&part64[0][0])[i] = 0ull;
        __syncthreads();
        const bool seg_ok = seg_ok_s;
        bool okc[G];
        uint32_t T[G][N > 1 ? N - 1 : 1];
        int ml[G];
#pragma unroll
        for (int c = 0; c < G; ++c) {
            okc[c] = ok_s[c] != 0 && seg_ok;
            ml[c] = ml_s[c];
#pragma unroll
            for (int i = 0; i + 1 < N; ++i) T[c][i] = thr_s[c][i];
        }
        // pieces of kClPiece requests, 8-aligned in the local index (first_request % 8 == 0)
        const int64_t pstart = seg_ok ? (s0 & ~(int64_t)7) : 0, pend = seg_ok ? s1 : 0;
        const int n_pieces = pend > pstart ? (int)((pend - pstart + kClPiece - 1) / kClPiece) : 0;

        // ---- pass 1: select every request in every chain; the interval's cell and
        // segment sums in registers, per-piece level counts in shared memory ----
        uint32_t cs[G][NCM][N], ts[G][NCM][N];
        uint32_t sm[NCM][N + 2];
#pragma unroll
        for (int c = 0; c < G; ++c)
#pragma unroll
            for (int cc = 0; cc < NCM; ++cc)
#pragma unroll
                for (int L = 0; L < N; ++L) { cs[c][cc][L] = 0u; ts[c][cc][L] = 0u; }
#pragma unroll
        for (int cc = 0; cc < NCM; ++cc)
#pragma unroll
            for (int f = 0; f < N + 2; ++f) sm[cc][f] = 0u;
        // 32-bit sums per thread are folded into part64 every 32 pieces (<= 256 requests per thread)
        auto flush = [&]() {
            int v = 0;
#pragma unroll
            for (int c = 0; c < G; ++c)
#pragma unroll
                for (int cc = 0; cc < NCM; ++cc)
#pragma unroll
                    for (int L = 0; L < N; ++L) {
                        const uint32_t x0 = __reduce_add_sync(0xFFFFFFFFu, cs[c][cc][L]);
                        const uint32_t x1 = __reduce_add_sync(0xFFFFFFFFu, ts[c][cc][L]);
                        if (lane == 0) { part64[warp][v] += x0; part64[warp][v + 1] += x1; }
                        v += 2;
                        cs[c][cc][L] = 0u; ts[c][cc][L] = 0u;
                    }
#pragma unroll
            for (int cc = 0; cc < NCM; ++cc)
#pragma unroll
                for (int f = 0; f < N + 2; ++f) {
                    const uint32_t x = __reduce_add_sync(0xFFFFFFFFu, sm[cc][f]);
                    if (lane == 0) part64[warp][NCELL + cc * (N + 2) + f] += x;
                    sm[cc][f] = 0u;
                }
        };
        for (int pi = 0; pi < n_pieces; ++pi) {
            if (pi > 0 && (pi & 31) == 0) flush();
            prefetch_piece<N>(a, pstart + (int64_t)(pi + 2) * kClPiece, pend, tid);
            const int64_t c0 = pstart + (int64_t)pi * kClPiece + 8 * (int64_t)tid;
            const bool any = c0 + 8 > s0 && c0 < s1;
            Chunk<N> ch;
            load_chunk<N>(a, c0, any, ch);
            uint32_t lc[G][N];
#pragma unroll
            for (int c = 0; c < G; ++c)
#pragma unroll
                for (int L = 0; L < N; ++L) lc[c][L] = 0u;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int64_t g = c0 + k;
                const uint32_t fb = flag_byte(ch.fw, k);
                const uint32_t cls = (fb >> 1) & 3u;
                const bool pinned = fb & 1u;
                const bool inr = any && g >= s0 && g < s1;
                if (inr && cls >= (uint32_t)NC) err |= SPROUT_TRACE_BAD_CLASS;
                if (!(inr && cls < (uint32_t)NC)) continue;
                uint32_t tl[N];
#pragma unroll
                for (int L = 0; L < N; ++L) tl[L] = cl_half(ch.tk[L], k);
                if (seg_writer) {
#pragma unroll
                    for (int cc = 0; cc < NCM; ++cc) {
                        if ((uint32_t)cc != cls) continue;
                        sm[cc][0] += 1u;
                        sm[cc][1] += pinned ? 1u : 0u;
#pragma unroll
                        for (int L = 0; L < N; ++L) sm[cc][2 + L] += tl[L];
                    }
                }
#pragma unroll
                for (int c = 0; c < G; ++c) {
                    if (!okc[c]) continue;
                    const int L = cl_level<N>(ch.w[k], T[c], ml[c], pinned);
#pragma unroll
                    for (int LL = 0; LL < N; ++LL) {
                        const bool hit = LL == L;
                        lc[c][LL] += hit ? 1u : 0u;
#pragma unroll
                        for (int cc = 0; cc < NCM; ++cc) {
                            const bool h2 = hit && (uint32_t)cc == cls;
                            cs[c][cc][LL] += h2 ? 1u : 0u;
                            ts[c][cc][LL] += h2 ? tl[LL] : 0u;
                        }
                    }
                }
            }
#pragma unroll
            for (int c = 0; c < G; ++c)
#pragma unroll
                for (int L = 0; L < N; ++L) {
                    const uint32_t v = __reduce_add_sync(0xFFFFFFFFu, lc[c][L]);
                    if (lane == 0 && v) {
                        atomicAdd(&ctot[c * N + L], v);
                        if (pi < kClMaxPieces) atomicAdd(&pcnt[pi][c * N + L], v);
                    }
                }
        }
        flush();
        __syncthreads();
        // interval totals per (chain, level) and the first piece holding one of the
        // last W requests (the ones that enter the window); pcnt becomes the level-L
        // requests BEFORE each piece
        const bool long_interval = n_pieces > kClMaxPieces;   // (> 2^20 requests: counts re-derived below)
        if (tid < G * N) {
            const uint32_t tot = ctot[tid];
            uint32_t run0 = 0u;
            for (int pi = 0; pi < n_pieces && pi < kClMaxPieces; ++pi) { const uint32_t v = pcnt[pi][tid]; pcnt[pi][tid] = run0; run0 += v; }
            uint32_t first = 0u;
            if (!long_interval) {   // the first piece whose level-L requests reach the window (index >= tot - W)
                const uint32_t need = tot > (uint32_t)W ? tot - (uint32_t)W : 0u;
                first = (uint32_t)n_pieces;
                for (int pi = n_pieces - 1; pi >= 0; --pi) {
                    const uint32_t next = pi + 1 < n_pieces ? pcnt[pi + 1][tid] : tot;
                    if (next > need) first = (uint32_t)pi; else break;
                }
            }
            cfirst[tid] = first;
        }
        __syncthreads();
        // ---- pass 2: the window entries, in request order (a block scan per piece
        // gives every request its forward index among its (chain, level)) ----
        int dn[G][N][NCM], dk[G][N][NCM];
#pragma unroll
        for (int c = 0; c < G; ++c)
#pragma unroll
            for (int L = 0; L < N; ++L)
#pragma unroll
                for (int cc = 0; cc < NCM; ++cc) { dn[c][L][cc] = 0; dk[c][L][cc] = 0; }
        int p_first = n_pieces;
        uint32_t tot_c[G][N];
#pragma unroll
        for (int c = 0; c < G; ++c)
#pragma unroll
            for (int L = 0; L < N; ++L) {
                tot_c[c][L] = ctot[c * N + L];
                if (okc[c] && tot_c[c][L] > 0u) p_first = min(p_first, long_interval ? 0 : (int)cfirst[c * N + L]);
            }
        uint32_t run[G][N];   // long intervals: level-L requests of the pieces already walked
#pragma unroll
        for (int c = 0; c < G; ++c)
#pragma unroll
            for (int L = 0; L < N; ++L) run[c][L] = 0u;
        const int p2 = long_interval ? 0 : p_first;
        prefetch_piece<N>(a, pstart + (int64_t)p2 * kClPiece, pend, tid);
        for (int pi = p2; pi < n_pieces; ++pi) {
            prefetch_piece<N>(a, pstart + (int64_t)(pi + 1) * kClPiece, pend, tid);
            const int64_t c0 = pstart + (int64_t)pi * kClPiece + 8 * (int64_t)tid;
            const bool any = c0 + 8 > s0 && c0 < s1;
            Chunk<N> ch;
            load_chunk<N>(a, c0, any, ch);
            uint32_t lv[G];     // 2-bit... levels of the 8 requests per chain, 4 bits each
            uint32_t lc[G][N];
            uint32_t valid = 0u;
#pragma unroll
            for (int c = 0; c < G; ++c) {
                lv[c] = 0u;
#pragma unroll
                for (int L = 0; L < N; ++L) lc[c][L] = 0u;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int64_t g = c0 + k;
                const uint32_t fb = flag_byte(ch.fw, k);
                const bool v = any && g >= s0 && g < s1 && ((fb >> 1) & 3u) < (uint32_t)NC;
                valid |= v ? (1u << k) : 0u;
                if (!v) continue;
#pragma unroll
                for (int c = 0; c < G; ++c) {
                    const int L = cl_level<N>(ch.w[k], T[c], ml[c], fb & 1u);
                    lv[c] |= (uint32_t)L << (4 * k);
#pragma unroll
                    for (int LL = 0; LL < N; ++LL) lc[c][LL] += LL == L ? 1u : 0u;
                }
            }
            // exclusive scan of the counts over the piece's threads
            uint32_t before[G][N];
#pragma unroll
            for (int c = 0; c < G; ++c)
#pragma unroll
                for (int L = 0; L < N; ++L) {
                    uint32_t x = lc[c][L];
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, d);
                        if (lane >= d) x += y;
                    }
                    before[c][L] = x - lc[c][L];
                    if (lane == 31) wtot[warp][c * N + L] = x;
                }
            __syncthreads();
#pragma unroll
            for (int c = 0; c < G; ++c)
#pragma unroll
                for (int L = 0; L < N; ++L) {
                    uint32_t b = 0u, pt = 0u;
                    for (int w2 = 0; w2 < kClWarps; ++w2) {
                        const uint32_t v = wtot[w2][c * N + L];
                        b += w2 < warp ? v : 0u;
                        pt += v;
                    }
                    const uint32_t base = long_interval ? run[c][L] : pcnt[pi][c * N + L];
                    before[c][L] += base + b;
                    run[c][L] += pt;
                }
            __syncthreads();   // wtot is reused by the next piece
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (!((valid >> k) & 1u)) continue;
                const uint32_t cls = (flag_byte(ch.fw, k) >> 1) & 3u;
#pragma unroll
                for (int c = 0; c < G; ++c) {
                    if (!okc[c]) continue;
                    const int L = (int)((lv[c] >> (4 * k)) & 15u);
                    uint32_t idx = 0u, tot = 0u, tl = 0u;
#pragma unroll
                    for (int LL = 0; LL < N; ++LL)
                        if (LL == L) { idx = before[c][LL]; tot = tot_c[c][LL]; tl = cl_half(ch.tk[LL], k); before[c][LL] += 1u; }
                    if (idx + (uint32_t)W < tot) continue;   // not among the interval's last W of its level
                    // forward index idx goes to slot head + idx (FIFO); the slot's entry from
                    // before the interval leaves the window
                    const int slot = (int)(((uint32_t)head[c][L] + idx) % (uint32_t)W);
                    uint32_t *rp = ring + ((size_t)c * N + L) * W + slot;
                    if (size[c][L] == W || slot < size[c][L]) {
                        const uint32_t old = *rp;
                        const uint32_t oc = old >> 16;
#pragma unroll
                        for (int LL = 0; LL < N; ++LL)
#pragma unroll
                            for (int cc = 0; cc < NCM; ++cc)
                                if (LL == L && (uint32_t)cc == oc) { dn[c][LL][cc] -= 1; dk[c][LL][cc] -= (int)(old & 0xFFFFu); }
                    }
                    *rp = (cls << 16) | tl;
#pragma unroll
                    for (int LL = 0; LL < N; ++LL)
#pragma unroll
                        for (int cc = 0; cc < NCM; ++cc)
                            if (LL == L && (uint32_t)cc == cls) { dn[c][LL][cc] += 1; dk[c][LL][cc] += (int)tl; }
                }
            }
        }
        if (t + 1 < a.T) {   // the next interval's first two pieces into L2 while this one is folded
            const int64_t n0 = a.seg_offsets[sl + 1], n1 = a.seg_offsets[sl + 2];
            if (n0 >= 0 && n0 <= n1 && n1 <= a.n_requests) {
                prefetch_piece<N>(a, n0 & ~(int64_t)7, n1, tid);
                prefetch_piece<N>(a, (n0 & ~(int64_t)7) + kClPiece, n1, tid);
            }
        }
        // ---- fold the interval: window deltas per warp, then one thread per value ----
        {
            int v = 0;
#pragma unroll
            for (int c = 0; c < G; ++c)
#pragma unroll
                for (int L = 0; L < N; ++L)
#pragma unroll
                    for (int cc = 0; cc < NCM; ++cc) {
                        const uint32_t x0 = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)dn[c][L][cc]);
                        const uint32_t x1 = __reduce_add_sync(0xFFFFFFFFu, (uint32_t)dk[c][L][cc]);
                        if (lane == 0) { part[warp][v] = x0; part[warp][v + 1] = x1; }
                        v += 2;
                    }
        }
        __syncthreads();
        __shared__ unsigned long long tot64[NCELL + NSEG];
        for (int v = tid; v < NDELTA; v += kClThreads) {
            long long sum = 0;
            for (int w2 = 0; w2 < kClWarps; ++w2) sum += (long long)(int)part[w2][v];
            unsigned long long *wp = &wsum[0][0][0][0] + v;
            *wp = (unsigned long long)((long long)*wp + sum);
        }
        for (int v = tid; v < NCELL + NSEG; v += kClThreads) {
            unsigned long long sum = 0ull;
            for (int w2 = 0; w2 < kClWarps; ++w2) sum += part64[w2][v];
            tot64[v] = sum;
        }
        if (tid < G * N) {
            const int c = tid / N, L = tid % N;
            const uint32_t tt = okc[c] ? ctot[tid] : 0u;
            head[c][L] = (int)(((uint32_t)head[c][L] + tt) % (uint32_t)W);
            size[c][L] = (int)min((uint32_t)size[c][L] + tt, (uint32_t)W);
        }
        __syncthreads();
        // ---- the interval's outputs: G cells (cell_epilogue's formulas and order) and the segment ----
        const double kp = __dmul_rn(k0_s, a.pue);
        if (tid < G && j0 + tid < a.X) {
            const int c = tid;
            const int64_t cell = sl * a.X + j0 + c;
            const bool okk = ok_s[c] != 0 && seg_ok;
            double E = 0.0, Tm = 0.0, Q = 0.0;
            for (int cc = 0; cc < NC; ++cc) {
#pragma unroll
                for (int L = 0; L < N; ++L) {
                    const int v = ((c * NCM + cc) * N + L) * 2;
                    const unsigned long long cn = okk ? tot64[v] : 0ull, tk2 = okk ? tot64[v + 1] : 0ull;
                    a.cnt[(cell * NC + cc) * N + L] = cn;
                    a.tok[(cell * NC + cc) * N + L] = tk2;
                    const double n_ = (double)cn, t_ = (double)tk2;
                    E += n_ * cost.ef[cc][L] + t_ * cost.et[cc][L];
                    Tm += n_ * cost.pf[cc][L] + t_ * cost.pt[cc][L];
                    Q += n_ * qrow[L];
                }
            }
            a.energy[cell] = E;
            a.time_s[cell] = Tm;
            a.carbon[cell] = okk ? kp * E + a.k1 * Tm : 0.0;
            a.quality[cell] = Q;
        }
        if (seg_writer && tid == G) {   // write_seg_stats' formulas and order (trace_sim.cu)
            const unsigned long long *ss = tot64 + NCELL;   // [NCM][N + 2]
            double bE = 0.0, bT = 0.0, m = 0.0;
            for (int cc = 0; cc < NC; ++cc) {
                const unsigned long long mc = ss[cc * (N + 2)];
                a.seg_count[sl * NC + cc] = mc;
                a.seg_pinned[sl * NC + cc] = ss[cc * (N + 2) + 1];
                for (int L = 0; L < N; ++L) a.seg_tok[(sl * NC + cc) * N + L] = ss[cc * (N + 2) + 2 + L];
                bE += (double)mc * cost.ef[cc][0] + (double)ss[cc * (N + 2) + 2] * cost.et[cc][0];
                bT += (double)mc * cost.pf[cc][0] + (double)ss[cc * (N + 2) + 2] * cost.pt[cc][0];
                m += (double)mc;
            }
            a.seg_base[sl * 4 + 0] = bE;
            a.seg_base[sl * 4 + 1] = bT;
            a.seg_base[sl * 4 + 2] = kp * bE + a.k1 * bT;
            a.seg_base[sl * 4 + 3] = m * qrow[0];
        }
        __syncthreads();
    }
    err = __reduce_or_sync(0xFFFFFFFFu, err);
    if (lane == 0 && err) atomicOr(a.trace_status, err);
}

// chains per CTA: the smallest group that keeps every region's groups on
// distinct SMs (a CTA per SM; more chains per CTA only add per-request work),
// at most kMaxG, one chain per CTA with several classes (the per-thread sums),
// and the group's rings within shared memory
constexpr int kMaxG = 4;
static int pick_group(const ClosedArgs &a, int sms) {
    if (a.NC > 1) return 1;
    int G = 1;
    while (G < kMaxG && (int64_t)a.R_local * ((a.X + G - 1) / G) > sms && (size_t)(G + 1) * a.n * a.W * 4 <= 160 * 1024)
        ++G;
    return G;
}

cudaError_t launch_closed_loop(ClosedArgs &a, cudaStream_t stream, int *launches) {
    if ((int64_t)a.R_local * a.X == 0) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int G = pick_group(a, sms);
    a.n_groups = (a.X + G - 1) / G;
    const int64_t blocks = (int64_t)a.R_local * a.n_groups;
    const size_t smem = (size_t)G * a.n * a.W * 4;
    cudaError_t e = cudaSuccess;
#define CL_LAUNCH(NN, NCM_, GG)                                                                   \
    {                                                                                             \
        auto kern = closed_loop_kernel<NN, NCM_, GG>;                                             \
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);   \
        if (e != cudaSuccess) return e;                                                           \
        kern<<<(unsigned)blocks, kClThreads, smem, stream>>>(a);                                  \
    }
#define CL_G(NN)                                                                                  \
    case NN:                                                                                      \
        if (a.NC > 1) CL_LAUNCH(NN, kMaxClasses, 1)                                               \
        else if (G == 1) CL_LAUNCH(NN, 1, 1)                                                      \
        else if (G == 2) CL_LAUNCH(NN, 1, 2)                                                      \
        else if (G == 3) CL_LAUNCH(NN, 1, 3)                                                      \
        else CL_LAUNCH(NN, 1, 4)                                                                  \
        break;
    switch (a.n) {
        CL_G(1) CL_G(2) CL_G(3) CL_G(4) CL_G(5) CL_G(6) CL_G(7) CL_G(8)
        default: return cudaErrorInvalidValue;
    }
#undef CL_G
#undef CL_LAUNCH
    ++*launches;
    return cudaGetLastError();
}

}  // namespace sprout
