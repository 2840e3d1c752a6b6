// trace_x1.cu -- step 2 of the hot path for ONE cell per segment (X = 1:
// configs C1, C3 and C5, and any single-xi sweep) with n <= 4 levels and
// <= 2 model classes, or n <= 8 levels and one class.  With a single cell the level of a request is the a6 rule
// itself -- level = pinned ? 0 : min(#{i : w >= T_i}, max_level) (P:162,
// P:240; reading L10) -- so no breakpoint merge or histogram is needed: a
// warp owns a segment, each lane takes aligned quads of 4 consecutive
// requests (one Philox4x32-10 call, 8-byte token loads, one 4-byte flags
// load), and accumulates the cell's (class, level) counts and tokens and the
// segment's statistics in 32-bit registers; the warp folds them with
// __reduce_add_sync at the segment's end (in chunks, so no 32-bit sum can
// overflow).  Short segments (C3: 190 requests on average) are bound by
// per-segment overhead, which this keeps to a few dozen instructions instead
// of a histogram readout.  Outputs and fp64 closed forms are those of
// trace_sim.cu's epilogue (same formula order).
#include <cuda_runtime.h>
#include "sprout_device.cuh"
#include "sprout_kernels.cuh"

namespace sprout {

constexpr int kX1Warps = 8;                   // warps per CTA
#ifndef SPROUT_X1_NO_GROUPS
#define SPROUT_X1_NO_GROUPS 0   // A/B only: every segment on trace_x1_kernel (one warp per segment)
#endif
constexpr bool kX1NoGroups = SPROUT_X1_NO_GROUPS;
constexpr int64_t kX1Chunk = (int64_t)1 << 21; // requests per fold: <= 2^16 per lane, token sums <= 2^16 * 65535 < 2^32

template <int N, bool FLAGS, bool NC2, bool VB>
#ifndef SPROUT_X1_MIN_BLOCKS
#define SPROUT_X1_MIN_BLOCKS 3
#endif
__global__ void __launch_bounds__(32 * kX1Warps, SPROUT_X1_MIN_BLOCKS) trace_x1_kernel(const __grid_constant__ SimArgs a) {
    __shared__ CostConst cost;
    // per-warp 64-bit totals of a segment: [0, NC*N) cell counts, [NC*N, 2NC*N) cell tokens,
    // then tokens per level (all classes), class-1 tokens per level, valid requests,
    // class-1 requests, pinned per class
    constexpr int kTot = 2 * (NC2 ? 2 : 1) * N + 2 * N + 2 + 2;   // <= 36 (N <= 4 with 2 classes, N <= 8 with 1)
    __shared__ unsigned long long tot_s[kX1Warps][kTot];
    unsigned long long *tot = tot_s[threadIdx.x >> 5];
    for (int i = threadIdx.x; i < (int)(sizeof(CostConst) / 8); i += blockDim.x)
        reinterpret_cast<double *>(&cost)[i] = reinterpret_cast<const double *>(&a.cost)[i];
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31u;
    const int NC = a.NC;                 // == NCc (dispatch)
    constexpr int NCc = NC2 ? 2 : 1;
    uint32_t err = 0u;
    // Segment pipeline: the next segment's metadata is loaded into registers
    // and its tokens are prefetched into L2 while the current one streams, so
    // a short segment costs one L2 round trip instead of several HBM ones.
    // Queue tickets hand out batches of a.seg_batch segments; lane 0 holds
    // the ticket of the next batch.
    struct Pre {
        int64_t sl, s0, s1;
        int meta, ml;
        bool cell_ok;
        uint32_t T[N > 1 ? N - 1 : 1];
    };
    auto load_pre = [&](int64_t sl) {
        Pre p;
        p.sl = sl;
        p.meta = -3;
        p.s0 = p.s1 = 0;
        p.ml = 0;
        p.cell_ok = false;
#pragma unroll
        for (int i = 0; i + 1 < N; ++i) p.T[i] = 0xFFFFFFFFu;
        if (sl < a.n_segments) {
            p.s0 = a.seg_offsets[sl];
            p.s1 = a.seg_offsets[sl + 1];
            // invalid offsets: prep's verdict, or the same test here when prep did not run
            p.meta = a.seg_meta ? a.seg_meta[sl] : ((p.s0 >= 0 && p.s0 <= p.s1 && p.s1 <= a.n_requests) ? 0 : -2);
            p.cell_ok = a.cell_status[sl] == SPROUT_CELL_OK;
#pragma unroll
            for (int i = 0; i + 1 < N; ++i) p.T[i] = a.threshold[sl * (N - 1) + i];
            p.ml = a.max_level[sl];
        }
        return p;
    };
    // lanes 0..7: the first 8 lines (512 requests) of every plane -- a whole short segment; a long
    // one is prefetched inside its loop (more would evict lines from L2 before they are used)
    auto prefetch_tokens = [&](const Pre &p) {
        if (p.meta < -1 || p.s1 <= p.s0) return;
        const int64_t b0 = (p.s0 * 2) & ~(int64_t)127, b1 = p.s1 * 2;
        const int64_t off = b0 + 128 * (int64_t)lane;
        if (lane < 8 && off < b1) {
#pragma unroll
            for (int i = 0; i < N; ++i)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const uint8_t *>(a.tokens + (size_t)i * a.pitch) + off));
        }
        if (FLAGS) {
            const int64_t f0 = p.s0 & ~(int64_t)127, fo = f0 + 128 * (int64_t)lane;
            if (lane < 4 && fo < p.s1) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.flags + fo));
        }
    };
    const int64_t B = a.seg_batch;
    int64_t it_seg = 0, it_end = 0;
    uint32_t pend = 0u;
    if (lane == 0) pend = atomicAdd(a.queue, 1u);
    auto next_segment = [&]() -> int64_t {
        if (it_seg >= it_end) {
            it_seg = (int64_t)__shfl_sync(0xFFFFFFFFu, pend, 0) * B;
            it_end = min(it_seg + B, a.n_segments);
            if (it_seg >= a.n_segments) return a.n_segments;
            if (lane == 0) pend = atomicAdd(a.queue, 1u);
        }
        return it_seg++;
    };
    Pre cur = load_pre(next_segment());
    prefetch_tokens(cur);
    for (;;) {
        const int64_t sl = cur.sl;
        if (sl >= a.n_segments) break;
        const Pre nxt = load_pre(next_segment());
        const int64_t s = a.first_segment + sl;
        const int meta = cur.meta;
        if (meta == -2) {   // invalid offsets (prep): segment skipped, outputs zero
            err |= SPROUT_TRACE_BAD_OFFSETS;
            if (lane < (uint32_t)(NC * N)) { a.cnt[sl * NC * N + lane] = 0ull; a.tok[sl * NC * N + lane] = 0ull; }
            if (lane < (uint32_t)NC) { a.seg_count[sl * NC + lane] = 0ull; a.seg_pinned[sl * NC + lane] = 0ull; }
            if (lane < (uint32_t)(NC * N)) a.seg_tok[sl * NC * N + lane] = 0ull;
            if (lane < 4) a.seg_base[sl * 4 + lane] = 0.0;
            if (lane == 0) { a.energy[sl] = 0.0; a.time_s[sl] = 0.0; a.carbon[sl] = 0.0; a.quality[sl] = 0.0; }
            cur = nxt;
            prefetch_tokens(cur);
            continue;
        }
        prefetch_tokens(nxt);
        const int64_t s0 = cur.s0, s1 = cur.s1;
        const bool cell_ok = cur.cell_ok;
        uint32_t T[N > 1 ? N - 1 : 1];
#pragma unroll
        for (int i = 0; i + 1 < N; ++i) T[i] = cur.T[i];
        const int ml = cur.ml;
        bool pure = true;
#pragma unroll
        for (int i = 0; i + 1 < N; ++i) pure = pure && (T[i] == 0u || T[i] == 0xFFFFFFFFu);

        constexpr int NCc_N = (NC2 ? 2 : 1) * N;
        constexpr int oCC = 0, oCT = NCc_N, oST = 2 * NCc_N, oST1 = oST + N, oCV = oST1 + N, oC1 = oCV + 1,
                      oSP = oC1 + 1;
        for (int i = lane; i < kTot; i += 32) tot[i] = 0ull;
        __syncwarp();
        for (int64_t c0 = s0; c0 < s1; c0 += kX1Chunk) {
            const int64_t c1 = min(s1, c0 + kX1Chunk);
            uint32_t cc[NCc * N], ct[NCc * N], st[N], st1[N], cv = 0, cl1 = 0, sp[NCc];
#pragma unroll
            for (int k = 0; k < NCc * N; ++k) { cc[k] = 0; ct[k] = 0; }
#pragma unroll
            for (int i = 0; i < N; ++i) { st[i] = 0; st1[i] = 0; }
#pragma unroll
            for (int c = 0; c < NCc; ++c) sp[c] = 0;
            const int64_t gq0 = (int64_t)((a.first_request + (uint64_t)c0) >> 2);   // global quad of c0
            const int64_t gq1 = (int64_t)((a.first_request + (uint64_t)c1 + 3) >> 2);
            // quads in pairs (both quads' loads in flight together), L2 prefetch 8 iterations ahead
            auto quad = [&](int64_t gq, const uint2 (&tw)[N], uint32_t fw, bool valid) {
                const int64_t r4 = gq * 4 - (int64_t)a.first_request;
                // a pure mix (every threshold 0 or saturated) selects the same level for every
                // draw: no draw is needed (warp-uniform)
                Philox4 d;
                if (pure) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) d.v[j] = 0u;
                } else {
                    d = philox4x32_10_rk((uint32_t)gq, (uint32_t)((uint64_t)gq >> 32), 0u, 0u, a.rk0, a.rk1);
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int64_t r = r4 + j;
                    const uint32_t w = d.v[j];
                    uint32_t cls = 0u, pin = 0u;
                    if (FLAGS) {
                        const uint32_t fb = (fw >> (8 * j)) & 0xFFu;
                        pin = fb & 1u;
                        cls = (fb >> 1) & 3u;
                    }
                    const bool inr = valid && (uint64_t)(r - c0) < (uint64_t)(c1 - c0);
                    const bool okc = cls < (uint32_t)NC;
                    if (inr && !okc) err |= SPROUT_TRACE_BAD_CLASS;
                    const bool ok = inr && okc;
                    int L = 0;
#pragma unroll
                    for (int i = 0; i + 1 < N; ++i) L += (w >= T[i]) ? 1 : 0;
                    L = min(L, ml);
                    L = pin ? 0 : L;
                    if (VB && inr) a.levels_out[r] = (ok && cell_ok) ? (uint8_t)L : (uint8_t)0xFF;   // verify mode
                    uint32_t t[N], tL = 0u;
#pragma unroll
                    for (int i = 0; i < N; ++i) {
                        const uint32_t word = (j >> 1) ? tw[i].y : tw[i].x;
                        t[i] = (j & 1) ? (word >> 16) : (word & 0xFFFFu);
                        tL = (L == i) ? t[i] : tL;
                    }
                    const bool is1 = NC2 && cls == 1u;
                    cv += ok ? 1u : 0u;
                    cl1 += (ok && is1) ? 1u : 0u;
#pragma unroll
                    for (int c = 0; c < NCc; ++c) sp[c] += (ok && pin && (int)cls == c) ? 1u : 0u;
#pragma unroll
                    for (int i = 0; i < N; ++i) {
                        st[i] += ok ? t[i] : 0u;
                        if (NC2) st1[i] += (ok && is1) ? t[i] : 0u;
                    }
                    const int idx = L + (is1 ? N : 0);
#pragma unroll
                    for (int k = 0; k < NCc * N; ++k) {
                        const bool hit = ok && idx == k;
                        cc[k] += hit ? 1u : 0u;
                        ct[k] += hit ? tL : 0u;
                    }
                }
            };
            auto load = [&](int64_t gq, uint2 (&tw)[N], uint32_t &fw) {
                const int64_t r4 = gq * 4 - (int64_t)a.first_request;
#pragma unroll
                for (int i = 0; i < N; ++i)
                    tw[i] = __ldcs(reinterpret_cast<const uint2 *>(a.tokens + (size_t)i * a.pitch + r4));
                fw = FLAGS ? __ldcs(reinterpret_cast<const uint32_t *>(a.flags + r4)) : 0u;
                const int64_t rp = r4 + 4 * 32 * 8;
                if (rp < c1) {
#pragma unroll
                    for (int i = 0; i < N; ++i)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.tokens + (size_t)i * a.pitch + rp));
                }
            };
            if (!FLAGS && !NC2 && pure && !VB) {
                // pure mix, no flags: every request is at the same level -- a streaming sum of the
                // token planes (interior quads whole, the two edge quads per request)
                int Lp = 0;
#pragma unroll
                for (int i = 0; i + 1 < N; ++i) Lp += (T[i] == 0u) ? 1 : 0;
                Lp = min(Lp, ml);
                constexpr int U = N <= 3 ? 4 : 2;   // quads in flight per lane (registers)
                for (int64_t base = gq0 + lane; base < gq1; base += 32 * U) {
                    uint2 ta[U][N];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        uint32_t fa;
                        load(min(base + 32 * u, gq1 - 1), ta[u], fa);
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int64_t gq = base + 32 * u;
                        if (gq >= gq1) break;
                        const int64_t r4 = gq * 4 - (int64_t)a.first_request;
                        if (r4 >= c0 && r4 + 4 <= c1) {
#pragma unroll
                            for (int i = 0; i < N; ++i)
                                st[i] += (ta[u][i].x & 0xFFFFu) + (ta[u][i].x >> 16) + (ta[u][i].y & 0xFFFFu) +
                                         (ta[u][i].y >> 16);
                            cv += 4u;
                        } else {
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                if ((uint64_t)(r4 + j - c0) < (uint64_t)(c1 - c0)) {
#pragma unroll
                                    for (int i = 0; i < N; ++i) {
                                        const uint32_t word = (j >> 1) ? ta[u][i].y : ta[u][i].x;
                                        st[i] += (j & 1) ? (word >> 16) : (word & 0xFFFFu);
                                    }
                                    cv += 1u;
                                }
                            }
                        }
                    }
                }
#pragma unroll
                for (int i = 0; i < N; ++i) {
                    cc[i] = (i == Lp) ? cv : 0u;
                    ct[i] = (i == Lp) ? st[i] : 0u;
                }
            } else {
                for (int64_t gq = gq0 + lane; gq < gq1; gq += 32) {
                    uint2 ta[N];
                    uint32_t fa;
                    load(gq, ta, fa);
                    quad(gq, ta, fa, true);
                }
            }
            // fold the chunk into the warp's 64-bit totals
            auto fold = [&](int o, uint32_t v) {
                const uint32_t sum = __reduce_add_sync(0xFFFFFFFFu, v);
                if (lane == 0) tot[o] += sum;
            };
#pragma unroll
            for (int k = 0; k < NCc * N; ++k) { fold(oCC + k, cc[k]); fold(oCT + k, ct[k]); }
#pragma unroll
            for (int i = 0; i < N; ++i) {
                fold(oST + i, st[i]);
                if (NC2) fold(oST1 + i, st1[i]);
            }
            fold(oCV, cv);
            if (NC2) fold(oC1, cl1);
#pragma unroll
            for (int c = 0; c < NCc; ++c) fold(oSP + c, sp[c]);
        }
        __syncwarp();

        // per-class segment statistics and the Base counterfactual (write_seg_stats' order)
        const int64_t qrow_i = a.profile_per_interval ? s
                             : (s < 0xFFFFFFFFll ? (int64_t)a.div_t.div((uint32_t)s) : s / a.T);
        const double *qrow = a.q + qrow_i * N;
        const double kp = a.k0[s] * a.pue;
        if (lane == 0) {
            const unsigned long long c1n = NC2 ? tot[oC1] : 0ull;
            double bE = 0.0, bT = 0.0, m = 0.0;
#pragma unroll
            for (int c = 0; c < NCc; ++c) {
                const unsigned long long mc = c == 0 ? tot[oCV] - c1n : c1n;
                a.seg_count[sl * NCc + c] = mc;
                a.seg_pinned[sl * NCc + c] = tot[oSP + c];
                unsigned long long t0 = 0ull;
#pragma unroll
                for (int i = 0; i < N; ++i) {
                    const unsigned long long t1 = NC2 ? tot[oST1 + i] : 0ull;
                    const unsigned long long tc = c == 0 ? tot[oST + i] - t1 : t1;
                    a.seg_tok[(sl * NCc + c) * N + i] = tc;
                    if (i == 0) t0 = tc;
                }
                bE += (double)mc * cost.ef[c][0] + (double)t0 * cost.et[c][0];
                bT += (double)mc * cost.pf[c][0] + (double)t0 * cost.pt[c][0];
                m += (double)mc;
            }
            a.seg_base[sl * 4 + 0] = bE;
            a.seg_base[sl * 4 + 1] = bT;
            a.seg_base[sl * 4 + 2] = kp * bE + a.k1 * bT;
            a.seg_base[sl * 4 + 3] = m * qrow[0];
            // the cell (cell_epilogue's order)
            double E = 0.0, Tm = 0.0, Q = 0.0;
#pragma unroll
            for (int c = 0; c < NCc; ++c) {
#pragma unroll
                for (int L = 0; L < N; ++L) {
                    const unsigned long long cn = cell_ok ? tot[oCC + c * N + L] : 0ull;
                    const unsigned long long tk = cell_ok ? tot[oCT + c * N + L] : 0ull;
                    a.cnt[(sl * NCc + c) * N + L] = cn;
                    a.tok[(sl * NCc + c) * N + L] = tk;
                    const double n_ = (double)cn, t_ = (double)tk;
                    E += n_ * cost.ef[c][L] + t_ * cost.et[c][L];
                    Tm += n_ * cost.pf[c][L] + t_ * cost.pt[c][L];
                    Q += n_ * qrow[L];
                }
            }
            a.energy[sl] = E;
            a.time_s[sl] = Tm;
            a.carbon[sl] = cell_ok ? kp * E + a.k1 * Tm : 0.0;
            a.quality[sl] = Q;
        }
        __syncwarp();
        cur = nxt;
    }
    err = __reduce_or_sync(0xFFFFFFFFu, err);
    if (lane == 0 && err) atomicOr(a.trace_status, err);
}

// ---------------------------------------------------------------------------
// Short segments (C3: 190 requests on average): G segments per warp, 32/G
// lanes per segment.  The same per-quad selection and accumulation as
// trace_x1_kernel, but the per-segment work -- metadata loads, the register
// folds (__reduce_add_sync over the segment's lane group, all G groups at
// once) and the epilogue (one leader lane per group, all G leaders at once)
// -- is shared by G segments, and a segment's quads keep 32/G lanes busy
// instead of leaving most of 32 idle.  Outputs, formulas and order as
// trace_x1_kernel.
template <int N, bool FLAGS, bool NC2, int G, bool VB>
__global__ void __launch_bounds__(32 * kX1Warps, SPROUT_X1_MIN_BLOCKS) trace_x1g_kernel(const __grid_constant__ SimArgs a) {
    constexpr int LG = 32 / G;                       // lanes per segment
    constexpr int NCc = NC2 ? 2 : 1;
    constexpr int NCc_N = NCc * N;
    constexpr int kTot = 2 * NCc_N + 2 * N + 2 + 2;
    constexpr int64_t kChunk = (int64_t)LG << 16;    // requests per fold: <= 2^16 per lane
    __shared__ CostConst cost;
    __shared__ unsigned long long tot_s[kX1Warps][G][kTot];
    for (int i = threadIdx.x; i < (int)(sizeof(CostConst) / 8); i += blockDim.x)
        reinterpret_cast<double *>(&cost)[i] = reinterpret_cast<const double *>(&a.cost)[i];
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31u;
    const int grp = (int)lane / LG, li = (int)lane % LG;
    unsigned long long *tot = tot_s[threadIdx.x >> 5][grp];
    const int NC = a.NC;
    uint32_t err = 0u;
    constexpr int oCC = 0, oCT = NCc_N, oST = 2 * NCc_N, oST1 = oST + N, oCV = oST1 + N, oC1 = oCV + 1, oSP = oC1 + 1;
    // tickets hand out batches of a.seg_batch * G consecutive segments; group g of the warp
    // takes segment base + g of each G-block
    const int64_t B = (int64_t)a.seg_batch * G;
    int64_t it_seg = 0, it_end = 0;
    uint32_t pend = 0u;
    if (lane == 0) pend = atomicAdd(a.queue, 1u);
    for (;;) {
        if (it_seg >= it_end) {
            it_seg = (int64_t)__shfl_sync(0xFFFFFFFFu, pend, 0) * B;
            it_end = min(it_seg + B, a.n_segments);
            if (it_seg >= a.n_segments) break;
            if (lane == 0) pend = atomicAdd(a.queue, 1u);
        }
        const int64_t sl = it_seg + grp;
        it_seg += G;
        const bool have = sl < it_end;
        int meta = -3;
        int64_t s0 = 0, s1 = 0;
        bool cell_ok = false;
        uint32_t T[N > 1 ? N - 1 : 1];
        int ml = 0;
#pragma unroll
        for (int i = 0; i + 1 < N; ++i) T[i] = 0xFFFFFFFFu;
        if (have) {
            s0 = a.seg_offsets[sl];
            s1 = a.seg_offsets[sl + 1];
            meta = a.seg_meta ? a.seg_meta[sl] : ((s0 >= 0 && s0 <= s1 && s1 <= a.n_requests) ? 0 : -2);
            cell_ok = a.cell_status[sl] == SPROUT_CELL_OK;
#pragma unroll
            for (int i = 0; i + 1 < N; ++i) T[i] = a.threshold[sl * (N - 1) + i];
            ml = a.max_level[sl];
        }
        const bool bad = have && meta == -2;   // invalid offsets (prep): segment skipped, outputs zero
        if (bad) err |= SPROUT_TRACE_BAD_OFFSETS;
        const bool live = have && !bad;
        if (!live) s0 = s1 = 0;
        bool pure = true;
#pragma unroll
        for (int i = 0; i + 1 < N; ++i) pure = pure && (T[i] == 0u || T[i] == 0xFFFFFFFFu);
        if (li < kTot) for (int i = li; i < kTot; i += LG) tot[i] = 0ull;
        __syncwarp();
        // chunks of kChunk requests per segment (one for any segment of <= 2^16 requests per lane)
        const int64_t nch = s1 > s0 ? (s1 - s0 + kChunk - 1) / kChunk : 0;
        int64_t nch_max = nch;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) nch_max = max(nch_max, (int64_t)__shfl_xor_sync(0xFFFFFFFFu, (long long)nch_max, d));
        for (int64_t ci = 0; ci < nch_max; ++ci) {
            const int64_t c0 = s0 + ci * kChunk, c1 = min(s1, c0 + kChunk);
            uint32_t cc[NCc_N], ct[NCc_N], st[N], st1[N], cv = 0, cl1 = 0, sp[NCc];
#pragma unroll
            for (int k = 0; k < NCc_N; ++k) { cc[k] = 0; ct[k] = 0; }
#pragma unroll
            for (int i = 0; i < N; ++i) { st[i] = 0; st1[i] = 0; }
#pragma unroll
            for (int c = 0; c < NCc; ++c) sp[c] = 0;
            if (c0 < c1) {
                const int64_t gq0 = (int64_t)((a.first_request + (uint64_t)c0) >> 2);
                const int64_t gq1 = (int64_t)((a.first_request + (uint64_t)c1 + 3) >> 2);
                // the lane's quads gq0 + li + LG*k; the next quad's loads are issued before the
                // current one is processed (two in flight)
                auto ld = [&](int64_t gq, uint2 (&tw)[N], uint32_t &fw) {
                    const int64_t r4 = gq * 4 - (int64_t)a.first_request;
#pragma unroll
                    for (int i = 0; i < N; ++i)
                        tw[i] = __ldcs(reinterpret_cast<const uint2 *>(a.tokens + (size_t)i * a.pitch + r4));
                    fw = FLAGS ? __ldcs(reinterpret_cast<const uint32_t *>(a.flags + r4)) : 0u;
                };
                uint2 twn[N];
                uint32_t fwn = 0u;
                if (gq0 + li < gq1) ld(gq0 + li, twn, fwn);
                for (int64_t gq = gq0 + li; gq < gq1; gq += LG) {
                    const int64_t r4 = gq * 4 - (int64_t)a.first_request;
                    uint2 tw[N];
#pragma unroll
                    for (int i = 0; i < N; ++i) tw[i] = twn[i];
                    const uint32_t fw = fwn;
                    if (gq + LG < gq1) ld(gq + LG, twn, fwn);
                    Philox4 d;
                    if (pure) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) d.v[j] = 0u;
                    } else {
                        d = philox4x32_10_rk((uint32_t)gq, (uint32_t)((uint64_t)gq >> 32), 0u, 0u, a.rk0, a.rk1);
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int64_t r = r4 + j;
                        const uint32_t w = d.v[j];
                        uint32_t cls = 0u, pin = 0u;
                        if (FLAGS) {
                            const uint32_t fb = (fw >> (8 * j)) & 0xFFu;
                            pin = fb & 1u;
                            cls = (fb >> 1) & 3u;
                        }
                        const bool inr = (uint64_t)(r - c0) < (uint64_t)(c1 - c0);
                        const bool okc = cls < (uint32_t)NC;
                        if (inr && !okc) err |= SPROUT_TRACE_BAD_CLASS;
                        const bool ok = inr && okc;
                        int L = 0;
#pragma unroll
                        for (int i = 0; i + 1 < N; ++i) L += (w >= T[i]) ? 1 : 0;
                        L = min(L, ml);
                        L = pin ? 0 : L;
                        if (VB && inr) a.levels_out[r] = (ok && cell_ok) ? (uint8_t)L : (uint8_t)0xFF;   // verify mode
                        uint32_t t[N], tL = 0u;
#pragma unroll
                        for (int i = 0; i < N; ++i) {
                            const uint32_t word = (j >> 1) ? tw[i].y : tw[i].x;
                            t[i] = (j & 1) ? (word >> 16) : (word & 0xFFFFu);
                            tL = (L == i) ? t[i] : tL;
                        }
                        const bool is1 = NC2 && cls == 1u;
                        cv += ok ? 1u : 0u;
                        cl1 += (ok && is1) ? 1u : 0u;
#pragma unroll
                        for (int c = 0; c < NCc; ++c) sp[c] += (ok && pin && (int)cls == c) ? 1u : 0u;
#pragma unroll
                        for (int i = 0; i < N; ++i) {
                            st[i] += ok ? t[i] : 0u;
                            if (NC2) st1[i] += (ok && is1) ? t[i] : 0u;
                        }
                        const int idx = L + (is1 ? N : 0);
#pragma unroll
                        for (int k = 0; k < NCc_N; ++k) {
                            const bool hit = ok && idx == k;
                            cc[k] += hit ? 1u : 0u;
                            ct[k] += hit ? tL : 0u;
                        }
                    }
                }
            }
            // fold the chunk over the segment's lane group (all groups at once: xor
            // shuffles within aligned groups of LG lanes)
            auto fold = [&](int o, uint32_t v) {
#pragma unroll
                for (int d = 1; d < LG; d <<= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
                if (li == 0) tot[o] += v;
            };
#pragma unroll
            for (int k = 0; k < NCc_N; ++k) { fold(oCC + k, cc[k]); fold(oCT + k, ct[k]); }
#pragma unroll
            for (int i = 0; i < N; ++i) {
                fold(oST + i, st[i]);
                if (NC2) fold(oST1 + i, st1[i]);
            }
            fold(oCV, cv);
            if (NC2) fold(oC1, cl1);
#pragma unroll
            for (int c = 0; c < NCc; ++c) fold(oSP + c, sp[c]);
        }
        __syncwarp();
        if (li == 0 && have) {
            const int64_t s = a.first_segment + sl;
            const int64_t qrow_i = a.profile_per_interval ? s
                                 : (s < 0xFFFFFFFFll ? (int64_t)a.div_t.div((uint32_t)s) : s / a.T);
            const double *qrow = a.q + qrow_i * N;
            const double kp = a.k0[s] * a.pue;
            if (bad) {
#pragma unroll
                for (int k = 0; k < NCc_N; ++k) { a.cnt[sl * NCc_N + k] = 0ull; a.tok[sl * NCc_N + k] = 0ull; a.seg_tok[sl * NCc_N + k] = 0ull; }
#pragma unroll
                for (int c = 0; c < NCc; ++c) { a.seg_count[sl * NCc + c] = 0ull; a.seg_pinned[sl * NCc + c] = 0ull; }
#pragma unroll
                for (int f = 0; f < 4; ++f) a.seg_base[sl * 4 + f] = 0.0;
                a.energy[sl] = 0.0; a.time_s[sl] = 0.0; a.carbon[sl] = 0.0; a.quality[sl] = 0.0;
            } else {
                // per-class segment statistics and the Base counterfactual (write_seg_stats' order)
                const unsigned long long c1n = NC2 ? tot[oC1] : 0ull;
                double bE = 0.0, bT = 0.0, m = 0.0;
#pragma unroll
                for (int c = 0; c < NCc; ++c) {
                    const unsigned long long mc = c == 0 ? tot[oCV] - c1n : c1n;
                    a.seg_count[sl * NCc + c] = mc;
                    a.seg_pinned[sl * NCc + c] = tot[oSP + c];
                    unsigned long long t0 = 0ull;
#pragma unroll
                    for (int i = 0; i < N; ++i) {
                        const unsigned long long t1 = NC2 ? tot[oST1 + i] : 0ull;
                        const unsigned long long tc = c == 0 ? tot[oST + i] - t1 : t1;
                        a.seg_tok[(sl * NCc + c) * N + i] = tc;
                        if (i == 0) t0 = tc;
                    }
                    bE += (double)mc * cost.ef[c][0] + (double)t0 * cost.et[c][0];
                    bT += (double)mc * cost.pf[c][0] + (double)t0 * cost.pt[c][0];
                    m += (double)mc;
                }
                a.seg_base[sl * 4 + 0] = bE;
                a.seg_base[sl * 4 + 1] = bT;
                a.seg_base[sl * 4 + 2] = kp * bE + a.k1 * bT;
                a.seg_base[sl * 4 + 3] = m * qrow[0];
                // the cell (cell_epilogue's order)
                double E = 0.0, Tm = 0.0, Q = 0.0;
#pragma unroll
                for (int c = 0; c < NCc; ++c) {
#pragma unroll
                    for (int L = 0; L < N; ++L) {
                        const unsigned long long cn = cell_ok ? tot[oCC + c * N + L] : 0ull;
                        const unsigned long long tk = cell_ok ? tot[oCT + c * N + L] : 0ull;
                        a.cnt[(sl * NCc + c) * N + L] = cn;
                        a.tok[(sl * NCc + c) * N + L] = tk;
                        const double n_ = (double)cn, t_ = (double)tk;
                        E += n_ * cost.ef[c][L] + t_ * cost.et[c][L];
                        Tm += n_ * cost.pf[c][L] + t_ * cost.pt[c][L];
                        Q += n_ * qrow[L];
                    }
                }
                a.energy[sl] = E;
                a.time_s[sl] = Tm;
                a.carbon[sl] = cell_ok ? kp * E + a.k1 * Tm : 0.0;
                a.quality[sl] = Q;
            }
        }
        __syncwarp();
    }
    err = __reduce_or_sync(0xFFFFFFFFu, err);
    if (lane == 0 && err) atomicOr(a.trace_status, err);
}

template <int N, bool FLAGS, bool NC2, int G>
static cudaError_t launch_x1g_t(SimArgs &a, cudaStream_t stream) {
    auto kern = a.levels_out ? trace_x1g_kernel<N, FLAGS, NC2, G, true> : trace_x1g_kernel<N, FLAGS, NC2, G, false>;
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * kX1Warps, 0);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    const int64_t warps = (int64_t)sms * per_sm * kX1Warps;
    int64_t bsz = a.n_segments / (warps * G * 16);
    a.seg_batch = (int)(bsz < 1 ? 1 : (bsz > 16 ? 16 : bsz));
    int64_t grid = (int64_t)sms * per_sm;
    const int64_t need = (a.n_segments + kX1Warps * G - 1) / (kX1Warps * G);
    if (grid > need) grid = need > 0 ? need : 1;
    kern<<<(unsigned)grid, 32 * kX1Warps, 0, stream>>>(a);
    return cudaGetLastError();
}

template <int N, bool FLAGS, bool NC2>
static cudaError_t launch_x1_t(SimArgs &a, cudaStream_t stream) {
    auto kern = a.levels_out ? trace_x1_kernel<N, FLAGS, NC2, true> : trace_x1_kernel<N, FLAGS, NC2, false>;
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * kX1Warps, 0);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    const int64_t warps = (int64_t)sms * per_sm * kX1Warps;
    int64_t bsz = a.n_segments / (warps * 16);
    a.seg_batch = (int)(bsz < 1 ? 1 : (bsz > 16 ? 16 : bsz));
    int64_t grid = (int64_t)sms * per_sm;
    const int64_t need = (a.n_segments + kX1Warps - 1) / kX1Warps;
    if (grid > need) grid = need > 0 ? need : 1;
    kern<<<(unsigned)grid, 32 * kX1Warps, 0, stream>>>(a);
    return cudaGetLastError();
}

bool trace_x1_supported(int n, int X, int NC) {
    return X == 1 && n >= 1 && ((NC == 2 && n <= 4) || (NC == 1 && n <= 8));
}

cudaError_t launch_trace_x1(SimArgs &a, cudaStream_t stream) {
    const bool fl = a.flags != nullptr, nc2 = a.NC == 2;
    // short segments on average: G = 4 segments per warp (8 lanes each)
    if (!kX1NoGroups && a.n <= 4 && a.n_segments > 0 && a.n_requests <= (int64_t)1024 * a.n_segments) {
#define X1G_CASE(NN)                                                                                          \
    case NN:                                                                                                  \
        return fl ? (nc2 ? launch_x1g_t<NN, true, true, 4>(a, stream) : launch_x1g_t<NN, true, false, 4>(a, stream)) \
                  : (nc2 ? launch_x1g_t<NN, false, true, 4>(a, stream) : launch_x1g_t<NN, false, false, 4>(a, stream));
        switch (a.n) {
            X1G_CASE(1) X1G_CASE(2) X1G_CASE(3) X1G_CASE(4)
            default: break;
        }
#undef X1G_CASE
    }
#define X1_CASE(NN)                                                                                      \
    case NN:                                                                                             \
        return fl ? (nc2 ? launch_x1_t<NN, true, true>(a, stream) : launch_x1_t<NN, true, false>(a, stream)) \
                  : (nc2 ? launch_x1_t<NN, false, true>(a, stream) : launch_x1_t<NN, false, false>(a, stream));
#define X1_CASE1(NN)                                                                                     \
    case NN:                                                                                             \
        return fl ? launch_x1_t<NN, true, false>(a, stream) : launch_x1_t<NN, false, false>(a, stream);
    if (nc2 && a.n > 4) return cudaErrorInvalidValue;
    switch (a.n) {
        X1_CASE(1) X1_CASE(2) X1_CASE(3) X1_CASE(4) X1_CASE1(5) X1_CASE1(6) X1_CASE1(7) X1_CASE1(8)
        default: return cudaErrorInvalidValue;
    }
#undef X1_CASE1
#undef X1_CASE
}

}  // namespace sprout
