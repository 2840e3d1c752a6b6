// trace_sim.cu -- step 2 of the hot path: stream the request trace once,
// select a directive level for every request in every xi cell of its
// segment, and reduce per-cell totals.
//
// Design:
//  * All X cells of a segment share one Philox draw per request (reading
//    L10).  A cell's level is a step function of the draw w with steps at its
//    thresholds, so every cell of the segment is determined by which BIN of
//    the segment's merged, sorted, distinct breakpoints w falls in.  The
//    prep kernel builds that breakpoint list and, per cell, the first bin of
//    each level.  The streaming kernel then only needs, per request, the bin
//    (a branchless binary search over <= X+1 keys) and one add of
//    (1, tok_0..tok_{n-1}) into a histogram; every cell's exact integer
//    statistics are differences of histogram prefix sums (a8), and its fp64
//    energy/time/carbon/quality follow from them in closed form (Eq. 1 is
//    linear in (count, tokens)).
//  * Histograms are lane-private in shared memory (no atomics on the hot
//    path): 16-bit packed fields, two per 32-bit word, with a guard bit that
//    spills a word into 64-bit warp accumulators before it can overflow.
//  * One warp owns one segment at a time (dynamic queue), so segment totals
//    need no cross-CTA reduction and are written with plain stores.
//  * Token planes are read once with 128-bit streaming loads, prefetched
//    two groups ahead.
// Segments the fast path cannot represent (more than kcap distinct
// breakpoints; arbitrary user thresholds) use a generic per-cell path.
#include <cuda_runtime.h>
#include <type_traits>
#include "sprout_device.cuh"
#include "sprout_kernels.cuh"

namespace sprout {

constexpr uint32_t kGuard = 0x80008000u;
constexpr int kPrepWarps = 4;
// warps per trace CTA (one CTA per SM): 8 warps = 2 per SM sub-partition leave 255 registers
// per thread for the 4-deep load rotation and the software pipeline
#ifndef SPROUT_TRACE_WARPS
#define SPROUT_TRACE_WARPS 8
#endif
constexpr int kMaxTraceWarps = SPROUT_TRACE_WARPS;
#ifndef SPROUT_LOOKUP_ORDER
#define SPROUT_LOOKUP_ORDER 0   // A/B only: placement of the next group's table lookups in the body
#endif
#ifndef SPROUT_LD_HINT
#define SPROUT_LD_HINT 0     // A/B only: L2::256B sector-promotion hint on the token loads
#endif
#ifndef SPROUT_NO_PREFETCH
#define SPROUT_NO_PREFETCH 0 // A/B only: no in-loop L2 prefetch
#endif
#ifndef SPROUT_LUT_FIXED
#define SPROUT_LUT_FIXED 0   // A/B only: bucket table over [0, 2^32) (no per-segment range, no clamp)
#endif
#ifndef SPROUT_DISABLE_X1
#define SPROUT_DISABLE_X1 0
#endif
#ifndef SPROUT_RMW_QUAD
#define SPROUT_RMW_QUAD 0   // A/B: read-modify-write four requests per link instead of two
#endif
constexpr bool kDisableX1 = SPROUT_DISABLE_X1;   // A/B only: route X = 1 through the general kernel

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// ---------------------------------------------------------------------------
// prep: one warp per segment.  Validates the segment's offsets, merges the
// nonzero thresholds of its valid cells into sorted distinct keys, and for
// each valid cell the first bin of levels 1..n-1 (count-and-clamp rule).
// E > 0: the (<= 32E) thresholds are sorted in registers, E per lane, by a
// warp bitonic network (shuffles across lanes, register swaps within); E = 0:
// generic shared-memory bitonic sort for larger sets.

// bitonic sort, ascending, of 32E values held E per lane (element i = lane*E + e)
template <int E>
__device__ __forceinline__ void warp_bitonic_sort(uint32_t (&v)[E], uint32_t lane) {
#pragma unroll
    for (int k = 2; k <= 32 * E; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= E) {
                const int lj = j / E;
                const bool lower = (lane & (uint32_t)lj) == 0u;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const uint32_t other = __shfl_xor_sync(0xFFFFFFFFu, v[e], lj);
                    const bool up = (((int)lane * E + e) & k) == 0;
                    v[e] = (lower == up) ? min(v[e], other) : max(v[e], other);
                }
            } else {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    if ((e & j) == 0) {
                        const bool up = (((int)lane * E + e) & k) == 0;
                        const uint32_t lo = min(v[e], v[e ^ j]), hi = max(v[e], v[e ^ j]);
                        v[e] = up ? lo : hi;
                        v[e ^ j] = up ? hi : lo;
                    }
                }
            }
        }
    }
}

template <int E>
__global__ void __launch_bounds__(32 * kPrepWarps) prep_kernel(const __grid_constant__ SimArgs a) {
    extern __shared__ uint32_t prep_smem[];
    const int warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    const int scap = E > 0 ? 32 * E : (a.sort_cap > 0 ? a.sort_cap : 1);
    uint32_t *buf = prep_smem + (size_t)warp * 2 * scap;
    uint32_t *keys = buf + scap;
    const int n = a.n, X = a.X;
    const int nt = n - 1;

    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *a.queue = 0u;
        *a.trace_status = 0u;
    }
    const int64_t gw = (int64_t)blockIdx.x * kPrepWarps + warp;
    const int64_t nwarps = (int64_t)gridDim.x * kPrepWarps;
    for (int64_t sl = gw; sl < a.n_segments; sl += nwarps) {
        const int64_t s0 = a.seg_offsets[sl], s1 = a.seg_offsets[sl + 1];
        if (!(s0 >= 0 && s0 <= s1 && s1 <= a.n_requests && (s1 - s0) < (int64_t)0xFFFFFFFFll)) {
            if (lane == 0) a.seg_meta[sl] = -2;
            continue;
        }
        if (a.kcap < 0 || nt == 0) {
            if (lane == 0) a.seg_meta[sl] = (a.kcap < 0) ? -1 : 0;
            continue;
        }
        const int M = X * nt;
        int K = 0;
        if constexpr (E > 0) {
            // gather nonzero thresholds of valid cells (0 = empty slot)
            uint32_t v[E];
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int idx = (int)lane * E + e;
                v[e] = 0u;
                if (idx < M) {
                    const int64_t cell = sl * X + (int)a.div_nt.div((uint32_t)idx);
                    if (a.cell_status[cell] == SPROUT_CELL_OK) v[e] = a.threshold[sl * M + idx];
                }
            }
            warp_bitonic_sort<E>(v, lane);
            // compact distinct nonzero keys: rank = exclusive count of first occurrences
            const uint32_t prev_last = __shfl_up_sync(0xFFFFFFFFu, v[E - 1], 1);
            uint32_t firsts = 0u;
            int cnt = 0;
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const uint32_t prev = e > 0 ? v[e - 1] : (lane > 0 ? prev_last : 0u);
                const bool first = v[e] != 0u && v[e] != prev;
                firsts |= first ? (1u << e) : 0u;
                cnt += first ? 1 : 0;
            }
            int incl = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(0xFFFFFFFFu, incl, d);
                if ((int)lane >= d) incl += y;
            }
            K = __shfl_sync(0xFFFFFFFFu, incl, 31);
            int r = incl - cnt;
#pragma unroll
            for (int e = 0; e < E; ++e)
                if (firsts & (1u << e)) keys[r++] = v[e];
        } else {
            const int cap = a.sort_cap;
            for (int idx = lane; idx < cap; idx += 32) {
                uint32_t v = 0u;
                if (idx < M) {
                    const int64_t cell = sl * X + idx / nt;
                    if (a.cell_status[cell] == SPROUT_CELL_OK) v = a.threshold[cell * nt + idx % nt];
                }
                buf[idx] = v;
            }
            __syncwarp();
            for (int k = 2; k <= cap; k <<= 1) {
                for (int jj = k >> 1; jj > 0; jj >>= 1) {
                    for (int i = lane; i < cap; i += 32) {
                        const int ixj = i ^ jj;
                        if (ixj > i) {
                            const uint32_t u = buf[i], v = buf[ixj];
                            const bool up = (i & k) == 0;
                            if ((u > v) == up) { buf[i] = v; buf[ixj] = u; }
                        }
                    }
                    __syncwarp();
                }
            }
            for (int base = 0; base < cap; base += 32) {
                const int i = base + lane;
                const uint32_t v = buf[i];
                const bool first = v != 0u && (i == 0 || buf[i - 1] != v);
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, first);
                const int rank = K + __popc(bal & ((1u << lane) - 1u));
                if (first) keys[rank] = v;
                K += __popc(bal);
            }
        }
        __syncwarp();
        if (K > a.kcap) {
            if (lane == 0) a.seg_meta[sl] = -1;
            continue;
        }
        for (int i = lane; i < K; i += 32) a.seg_keys[sl * a.kcap + i] = keys[i] - 1u;
        // per valid cell: first bin of each level L >= 1
        for (int j = lane; j < X; j += 32) {
            const int64_t cell = sl * X + j;
            if (a.cell_status[cell] != SPROUT_CELL_OK) continue;
            const int ml = a.max_level[cell];
            uint32_t pos[kMaxLevels];
            for (int i = 0; i < nt; ++i) {
                const uint32_t t = a.threshold[cell * nt + i];
                uint32_t ps = 0;
                if (t != 0u) {   // 1 + index of t in keys (binary search)
                    int lo = 0, hi = K - 1;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (keys[mid] < t) lo = mid + 1; else hi = mid;
                    }
                    ps = (uint32_t)lo + 1u;
                }
                pos[i] = ps;
            }
            for (int i = 1; i < nt; ++i) {   // insertion sort (nt <= 7)
                const uint32_t v = pos[i];
                int k = i - 1;
                while (k >= 0 && pos[k] > v) { pos[k + 1] = pos[k]; --k; }
                pos[k + 1] = v;
            }
            for (int L = 1; L <= nt; ++L) {
                const uint32_t bnd = (L <= ml) ? pos[L - 1] : (uint32_t)(K + 1);
                a.seg_bnd[cell * nt + (L - 1)] = (uint16_t)bnd;
            }
        }
        __syncwarp();
        if (lane == 0) a.seg_meta[sl] = K;
    }
}

// ---------------------------------------------------------------------------
// streaming kernel
//
// Lane-private histogram entry layout: fields packed two per 32-bit word,
// words grouped in pairs (one 64-bit shared access per pair):
//   word 0 = tok_0 (bits 0-19) | count (bits 20-31);
//   word m >= 1 = tok_{2m-1} (bits 0-15) | tok_{2m} (bits 16-31).
// The top bit of every field is a guard: a row is spilled into the warp's
// 64-bit accumulators ("wide" rows; field 0 = count, 1+i = tok_i) once a
// guard is set, before the next group of 8 requests could overflow it.
constexpr int kW0Shift = 20;                 // count field of word 0
constexpr uint32_t kW0Low = (1u << kW0Shift) - 1u;
constexpr uint32_t kGuard0 = 0x80080000u;    // guards of word 0 (tok_0 >= 2^19, count >= 2^11)

template <int N>
struct Words {
    static constexpr int NW = (N + 2) / 2;   // 32-bit words per entry
    static constexpr int NP = (NW + 1) / 2;  // 64-bit pairs per entry
};

template <int N, bool FLAGS>
struct Group {
    uint4 t[N];
    uint2 f;
};

template <int N, bool FLAGS>
__device__ __forceinline__ void load_group(Group<N, FLAGS> &g, const SimArgs &a, int64_t v) {
#pragma unroll
    for (int i = 0; i < N; ++i)
        g.t[i] = __ldcs(reinterpret_cast<const uint4 *>(a.tokens + (size_t)i * a.pitch) + v);
    if (FLAGS) g.f = __ldcs(reinterpret_cast<const uint2 *>(a.flags) + v);
}

// 32-bit word of level plane i holding requests 2(k/2), 2(k/2)+1 of a group
template <int N, bool FLAGS>
__device__ __forceinline__ uint32_t plane_word(const Group<N, FLAGS> &g, int i, int k) {
    const uint4 &u = g.t[i];
    return (k >> 1) == 0 ? u.x : (k >> 1) == 1 ? u.y : (k >> 1) == 2 ? u.z : u.w;
}

__device__ __forceinline__ uint32_t half16(uint32_t w, int k) { return (k & 1) ? (w >> 16) : (w & 0xFFFFu); }

// packed word m of request k (without the count increment of word 0)
template <int N, bool FLAGS>
__device__ __forceinline__ uint32_t packed_word(const Group<N, FLAGS> &g, int m, int k) {
    if (m == 0) return half16(plane_word<N, FLAGS>(g, 0, k), k);
    const uint32_t lo_src = plane_word<N, FLAGS>(g, 2 * m - 1, k);
    const uint32_t hi_src = (2 * m <= N - 1) ? plane_word<N, FLAGS>(g, 2 * m, k) : 0u;
    return __byte_perm(lo_src, hi_src, (k & 1) ? 0x7632u : 0x5410u);
}

// (low field index, high field index) of word m in the wide rows
__device__ __forceinline__ int word_lo_field(int m) { return m == 0 ? 1 : 2 * m; }
__device__ __forceinline__ int word_hi_field(int m) { return m == 0 ? 0 : 2 * m + 1; }

struct WarpSmem {
    uint2 *hist;                 // [(NC*nb + 1)][np][32] lane-private packed pairs
    unsigned long long *wide;    // [(NC*nb + 1)][n+1] 64-bit per-entry totals
    uint2 *lut;                  // [kLutBuckets] bin lookup table (if a.lut)
    uint32_t *keys;              // [kp] breakpoints - 1, padded with 0xFFFFFFFF
};

__device__ __forceinline__ WarpSmem carve(uint8_t *base, const SimArgs &a) {
    WarpSmem w;
    const int entries = a.NC * a.nb + 1;
    w.wide = reinterpret_cast<unsigned long long *>(base);
    // 16-byte aligned rows: bit 2 of a lane's row address is then free to carry the
    // bucket table's multi-key flag (fix_offsets)
    size_t off = ((size_t)entries * (a.n + 1) * 8 + 15) & ~(size_t)15;
    w.hist = reinterpret_cast<uint2 *>(base + off);
    off += (size_t)entries * a.nw * 32 * 4;          // a.nw = 2 * np words
    w.lut = reinterpret_cast<uint2 *>(base + off);
    if (a.lut) off += (size_t)kLutBuckets * 8;
    w.keys = reinterpret_cast<uint32_t *>(base + off);
    return w;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint2 lds64(uint32_t addr) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void sts64(uint32_t addr, uint2 v) {
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(addr), "r"(v.x), "r"(v.y) : "memory");
}

// bin of draw w = #{keys < w}: branchless binary search over P (power of
// two) padded keys holding (breakpoint - 1)
__device__ __forceinline__ int find_bin(const uint32_t *keys, int P, uint32_t w) {
    int pos = 0;
    for (int step = P >> 1; step > 0; step >>= 1) pos += (keys[pos + step - 1] < w) ? step : 0;
    return pos;
}

// Bucket table of the segment's keys over the draw range [base, 2^32):
// base = the smallest key rounded down to a multiple of the bucket width 2^s,
// s the smallest with (2^32 - 1 - base) >> s < kLutBuckets (0 <= s <= 32 - kLutBits).  A
// draw w is clamped to d = max(w, base) (draws below base are in bin 0) and
// looked up in bucket (d >> s) - (base >> s).  Entry = {the bucket's single
// key (0xFFFFFFFF if none), byte offset of the bin at the bucket start in the
// lane histogram | 4 if the bucket holds >= 2 keys}.  For a bucket with <= 1
// key the histogram row of d is offset + rowbytes * (d > key): one 64-bit
// shared load and one compare per request.  Adapting the range to the keys
// keeps a xi sweep's (uniformly spaced) keys one per bucket even when they
// crowd near 2^32 (low carbon intensity: mixes close to pure L0).
struct LutGeom {
    uint32_t base;      // aligned range start
    int s;              // log2 bucket width
    uint32_t bias;      // shared address of bucket 0 minus (base >> s) * 8
};

__device__ __forceinline__ LutGeom lut_geometry(const WarpSmem &W, int K) {
    LutGeom g;
#if SPROUT_LUT_FIXED
    const uint32_t kmin = 0u;
#else
    const uint32_t kmin = K > 0 ? W.keys[0] : 0u;
#endif
    int s = 0;
    for (;;) {
        const uint32_t b = (s >= 32) ? 0u : (kmin & ~((1u << s) - 1u));
        if (s >= 32 - kLutBits || ((0xFFFFFFFFu - b) >> s) < (uint32_t)kLutBuckets) {
            g.base = b;
            break;
        }
        ++s;
    }
    g.s = s;
    g.bias = smem_u32(W.lut) - ((g.base >> s) << 3);
    return g;
}

// Build: clear the table, scatter the keys (count in .y, key in .x), then an
// exclusive prefix over the bucket counts, 32 buckets per step (lane = bucket
// within the chunk; two ballots of the counts' low bits give the in-chunk
// prefix unless some count is >= 4, then a shuffle scan).
__device__ __forceinline__ void build_lut(const WarpSmem &W, int K, LutGeom g, uint32_t rowbytes) {
    const uint32_t lane = lane_id();
    for (int b = (int)lane; b < kLutBuckets; b += 32) W.lut[b] = make_uint2(0xFFFFFFFFu, 0u);
    __syncwarp();
    for (int j = (int)lane; j < K; j += 32) {
        const uint32_t key = W.keys[j];
        const uint32_t b = (key - g.base) >> g.s;
        atomicAdd(&W.lut[b].y, 1u);
        atomicExch(&W.lut[b].x, key);   // meaningful only when the bucket holds exactly one key (else replaced below)
    }
    __syncwarp();
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t run = 0u;
#pragma unroll 4
    for (int c = 0; c < kLutBuckets / 32; ++c) {
        const int b = c * 32 + (int)lane;
        const uint2 e = W.lut[b];
        const uint32_t cnt = e.y;
        uint32_t excl, total;
        if (__any_sync(0xFFFFFFFFu, cnt >= 4u)) {
            uint32_t x = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, d);
                if ((int)lane >= d) x += y;
            }
            excl = x - cnt;
            total = __shfl_sync(0xFFFFFFFFu, x, 31);
        } else {
            const uint32_t b0 = __ballot_sync(0xFFFFFFFFu, cnt & 1u), b1 = __ballot_sync(0xFFFFFFFFu, cnt & 2u);
            excl = __popc(b0 & lt) + 2u * __popc(b1 & lt);
            total = __popc(b0) + 2u * __popc(b1);
        }
        W.lut[b] = make_uint2(cnt == 1u ? e.x : 0xFFFFFFFFu, (run + excl) * rowbytes | (cnt >= 2u ? 4u : 0u));
        run += total;
    }
    __syncwarp();
}

// histogram entry of request k of a group: draw bin, or the class's pinned
// bin, offset by class; the discard entry for bad classes / masked requests
template <bool FLAGS>
__device__ __forceinline__ int entry_of(int bin, uint2 f, int k, int nb, int NC, bool inr, uint32_t &err) {
    int entry = bin;
    if (FLAGS) {
        const uint32_t fw = (k < 4) ? f.x : f.y;
        const uint32_t fb = (fw >> (8 * (k & 3))) & 0xFFu;
        const int cls = (int)((fb >> 1) & 3u);
        if (fb & 1u) entry = nb - 1;
        entry += cls * nb;
        if (cls >= NC) {
            entry = NC * nb;
            if (inr) err |= SPROUT_TRACE_BAD_CLASS;
        }
    }
    return inr ? entry : NC * nb;
}

// 64-bit accumulator add from several lanes: a native 32-bit shared atomic
// on the low word, and a carry into the high word when it wraps (rare).
// (A 64-bit shared atomicAdd would compile to a CAS loop.)
__device__ __forceinline__ void wide_add(unsigned long long *slot, uint32_t x) {
    uint32_t *w = reinterpret_cast<uint32_t *>(slot);
    const uint32_t old = atomicAdd(w, x);
    if (old + x < old) atomicAdd(w + 1, 1u);
}

// move a lane's packed row into the warp's 64-bit accumulators (rare)
template <int N>
__device__ __forceinline__ void spill_entry(uint2 *hist, unsigned long long *wide, int entry, uint32_t lane) {
    constexpr int NP = Words<N>::NP;
    unsigned long long *wr = wide + (size_t)entry * (N + 1);
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        uint2 *slot = hist + ((size_t)entry * NP + p) * 32 + lane;
        const uint2 v = *slot;
        *slot = make_uint2(0u, 0u);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int m = 2 * p + h;
            if (m >= Words<N>::NW) break;
            const uint32_t x = h ? v.y : v.x;
            wide_add(&wr[word_lo_field(m)], m == 0 ? (x & kW0Low) : (x & 0xFFFFu));
            if (word_hi_field(m) <= N) wide_add(&wr[word_hi_field(m)], m == 0 ? (x >> kW0Shift) : (x >> 16));
        }
    }
}

constexpr int kModeSearch = 0;   // level-synchronous binary search over the padded keys
constexpr int kModeLut = 1;      // bucket table + rare exact search

struct U8x {                     // eight per-request words, passed by value
    uint32_t v[8];
};

// Element k (runtime) of eight registers, and its replacement, as select
// cascades: lets the rare paths run as rolled loops (small code) without
// dynamically indexed -- hence local-memory -- register arrays.
__device__ __forceinline__ uint32_t sel8(const U8x &x, int k) {
    uint32_t r = x.v[0];
#pragma unroll
    for (int j = 1; j < 8; ++j) r = (k == j) ? x.v[j] : r;
    return r;
}
__device__ __forceinline__ void set8(U8x &x, int k, uint32_t val) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x.v[j] = (k == j) ? val : x.v[j];
}

// Selection draws of the 8 requests of group v (local requests 8v..8v+7;
// reading L10: counter (g>>2, 0, 0), word g&3).
__device__ __forceinline__ void group_draws_blk(uint64_t blk, const SimArgs &a, U8x &w) {
    const Philox4 d0 = philox4x32_10_rk((uint32_t)blk, (uint32_t)(blk >> 32), 0u, 0u, a.rk0, a.rk1);
    const Philox4 d1 = philox4x32_10_rk((uint32_t)(blk + 1), (uint32_t)((blk + 1) >> 32), 0u, 0u, a.rk0, a.rk1);
#pragma unroll
    for (int k = 0; k < 4; ++k) { w.v[k] = d0.v[k]; w.v[4 + k] = d1.v[k]; }
}
__device__ __forceinline__ void group_draws(int64_t v, const SimArgs &a, U8x &w) {
    group_draws_blk((a.first_request + (uint64_t)v * 8u) >> 2, a, w);
}

// shared address of the lane's histogram row of one draw, from the bucket
// table (bit 2 of `eor` flags a multi-key bucket)
__device__ __forceinline__ uint32_t lut_offset(uint32_t w, LutGeom geo, uint32_t rowbytes, uint32_t lane_base,
                                               uint32_t &eor) {
#if SPROUT_LUT_FIXED
    const uint32_t d = w;   // fixed geometry: base 0, no clamp
#else
    const uint32_t d = max(w, geo.base);
#endif
    const uint2 e = lds64(geo.bias + ((d >> geo.s) << 3));
    eor |= e.y;
    uint32_t r;   // e.y + lane_base + (d > e.x ? rowbytes : 0): one compare, one select, one 3-input add
    asm("{\n\t.reg .pred p;\n\t.reg .u32 t;\n\t"
        "setp.gt.u32 p, %1, %2;\n\t"
        "selp.u32 t, %3, 0, p;\n\t"
        "add.u32 t, t, %4;\n\t"
        "add.u32 %0, t, %5;\n\t}"
        : "=r"(r) : "r"(d), "r"(e.x), "r"(rowbytes), "r"(e.y), "r"(lane_base));
    return r;
}

// Shared addresses (lane_base + bin * rowbytes) of the histogram rows of the 8 draws.
// Branch-free: in LUT mode the return value has bit 2 set if some draw fell
// in a bucket holding >= 2 keys; the caller repairs those with fix_offsets().
template <int MODE>
__device__ __forceinline__ uint32_t group_offsets(const U8x &w, const WarpSmem &W, int P, LutGeom geo,
                                                  uint32_t rowbytes, uint32_t lane_base, U8x &off) {
    uint32_t eor = 0u;
    if (MODE == kModeLut) {
#pragma unroll
        for (int k = 0; k < 8; ++k) off.v[k] = lut_offset(w.v[k], geo, rowbytes, lane_base, eor);
    } else {
        int bin[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) bin[k] = 0;
        for (int step = P >> 1; step > 0; step >>= 1) {
            const uint32_t *base = W.keys + (step - 1);
#pragma unroll
            for (int k = 0; k < 8; ++k) bin[k] += (base[bin[k]] < w.v[k]) ? step : 0;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) off.v[k] = lane_base + (uint32_t)bin[k] * rowbytes;
    }
    return eor;
}

// exact offsets for the draws that fell in multi-key buckets (rare; inline
// -- a call would make the warp wait for its in-flight prefetch loads -- and
// rolled, to keep the hot loop's code small).  A flagged offset still
// carries bit 2 (lane_base is 8-aligned, rows are multiples of 256 B, and a
// multi-key entry's key is 0xFFFFFFFF so no row step was added), so the
// flagged requests are found from registers, and the bucket's first bin is
// (offset - lane_base) / rowbytes: the exact bin is a short linear scan over
// the bucket's keys from there (keys are padded with 0xFFFFFFFF past K).
__device__ __forceinline__ void fix_offsets(const U8x &w, U8x &off, const uint32_t *keys, int P, LutGeom geo,
                                            uint32_t rowbytes, uint32_t lane_base) {
    uint32_t mask = 0u;
#pragma unroll
    for (int k = 0; k < 8; ++k) mask |= ((off.v[k] >> 2) & 1u) << k;
#pragma unroll 1
    while (mask) {
        const int k = __ffs(mask) - 1;
        mask &= mask - 1u;
        const uint32_t wk = sel8(w, k);
        uint32_t pos = (sel8(off, k) - lane_base) / rowbytes;
#pragma unroll 1
        for (int t = 0; t < 4 && keys[pos] < wk; ++t) ++pos;
        if (keys[pos] < wk) pos = (uint32_t)find_bin(keys, P, wk);   // crowded bucket: full search
        set8(off, k, lane_base + pos * rowbytes);
    }
}

// row byte offset of request k: the draw's bin, or (FLAGS) the class's pinned
// bin, offset by class; the discard row for bad classes
template <bool FLAGS>
__device__ __forceinline__ uint32_t row_of(uint32_t off, uint2 f, int k, uint32_t pin_off, uint32_t class_bytes,
                                           int NC, uint32_t discard_off, uint32_t &err) {
    if (!FLAGS) return off;
    const uint32_t fw = (k < 4) ? f.x : f.y;
    const uint32_t fb = (fw >> (8 * (k & 3))) & 0xFFu;
    const uint32_t cls = (fb >> 1) & 3u;
    uint32_t r = ((fb & 1u) ? pin_off : off) + cls * class_bytes;
    if (cls >= (uint32_t)NC) {
        r = discard_off;
        err |= SPROUT_TRACE_BAD_CLASS;
    }
    return r;
}

// add one request straight into the 64-bit accumulators of its entry
template <int N, bool FLAGS>
__device__ __forceinline__ void add_wide(unsigned long long *wide, const Group<N, FLAGS> &g, int entry, int k) {
    unsigned long long *wr = wide + (size_t)entry * (N + 1);
    wide_add(&wr[0], 1u);
#pragma unroll
    for (int i = 0; i < N; ++i) wide_add(&wr[1 + i], half16(plane_word<N, FLAGS>(g, i, k), k));
}

// packed increment of word m >= 1 of request k: tok_{2m-1} | tok_{2m} << 16
template <int N, bool FLAGS>
__device__ __forceinline__ uint32_t packed_hi(const Group<N, FLAGS> &g, int m, int k) {
    const uint32_t lo_src = plane_word<N, FLAGS>(g, 2 * m - 1, k);
    const uint32_t hi_src = (2 * m <= N - 1) ? plane_word<N, FLAGS>(g, 2 * m, k) : 0u;
    return __byte_perm(lo_src, hi_src, (k & 1) ? 0x7632u : 0x5410u);
}

// OR of every token word of the group (bits 12-15 of a field set <=> a token >= 4096)
template <int N, bool FLAGS>
__device__ __forceinline__ uint32_t group_or(const Group<N, FLAGS> &g) {
    uint32_t big = 0u;
#pragma unroll
    for (int i = 0; i < N; ++i) big |= g.t[i].x | g.t[i].y | g.t[i].z | g.t[i].w;
    return big;
}
constexpr uint32_t kBigTok = 0xF000F000u;

// Fast update of a full group: for each request, one 64-bit shared load,
// packed adds (word 0 += tok_0 + 1<<16, the count; word m += tok_{2m-1} |
// tok_{2m} << 16) and a store per word pair of its lane-private row, with no
// branch (one basic block, so the scheduler can interleave it with the next
// group's Philox rounds).  Every field is below its guard bit before the
// group (guard invariant: 2^15 for 16-bit token fields, 2^19 for tok_0, 2^11
// for the count) and gains at most 8 * 4095 (tokens < 4096) or 8 (count), so
// no field can overflow inside the group; the caller checks the returned
// guard bits of the stored words afterwards, and redoes the group through
// the 64-bit path if it had a token >= 4096.  Stores happen in request
// order, so two requests of the group hitting the same row are serialised
// through shared memory correctly.
// packed increment of word pair p of request k
template <int N, bool FLAGS>
__device__ __forceinline__ uint2 packed_inc(const Group<N, FLAGS> &g, int k, int p) {
    constexpr int NW = Words<N>::NW;
    uint2 inc;
    if (p == 0) {
        const uint32_t w0 = plane_word<N, FLAGS>(g, 0, k);
        inc.x = ((k & 1) ? (w0 >> 16) : (w0 & 0xFFFFu)) + (1u << kW0Shift);
    } else {
        inc.x = packed_hi<N, FLAGS>(g, 2 * p, k);
    }
    inc.y = (2 * p + 1 < NW) ? packed_hi<N, FLAGS>(g, 2 * p + 1, k) : 0u;
    return inc;
}

// Read-modify-write of the rows of requests k, k+1 (k even): both loads issue
// together; if the two requests hit the same row, the second store carries
// both increments (stores stay in request order, so it lands last).
template <int N, bool FLAGS>
__device__ __forceinline__ void rmw_pair(const Group<N, FLAGS> &g, int k, uint32_t ra, uint32_t rb, uint32_t &acc0,
                                         uint32_t &acc) {
    constexpr int NP = Words<N>::NP;
    const bool same = ra == rb;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        uint2 A = lds64(ra + p * 256);
        const uint2 Bl = lds64(rb + p * 256);
        const uint2 ia = packed_inc<N, FLAGS>(g, k, p), ib = packed_inc<N, FLAGS>(g, k + 1, p);
        A.x += ia.x;
        A.y += ia.y;
        uint2 B = same ? A : Bl;
        B.x += ib.x;
        B.y += ib.y;
        sts64(ra + p * 256, A);
        sts64(rb + p * 256, B);
        if (p == 0) { acc0 |= B.x | A.x; acc |= B.y | A.y; } else { acc |= A.x | A.y | B.x | B.y; }
    }
}

// Read-modify-write of the rows of requests k..k+3 (k % 4 == 0): the four loads
// issue together, the increments are folded in registers in request order
// (a later request hitting an earlier one's row starts from that request's
// updated value), and the stores stay in request order, so the last store to
// a row carries every increment.  Half the dependent links of rmw_pair.
template <int N, bool FLAGS>
__device__ __forceinline__ void rmw_quad(const Group<N, FLAGS> &g, int k, uint32_t r0, uint32_t r1, uint32_t r2,
                                         uint32_t r3, uint32_t &acc0, uint32_t &acc) {
    constexpr int NP = Words<N>::NP;
    const bool e10 = r1 == r0, e20 = r2 == r0, e21 = r2 == r1, e30 = r3 == r0, e31 = r3 == r1, e32 = r3 == r2;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        uint2 A0 = lds64(r0 + p * 256);
        const uint2 L1 = lds64(r1 + p * 256), L2 = lds64(r2 + p * 256), L3 = lds64(r3 + p * 256);
        const uint2 i0 = packed_inc<N, FLAGS>(g, k, p), i1 = packed_inc<N, FLAGS>(g, k + 1, p);
        const uint2 i2 = packed_inc<N, FLAGS>(g, k + 2, p), i3 = packed_inc<N, FLAGS>(g, k + 3, p);
        A0.x += i0.x; A0.y += i0.y;
        uint2 A1 = e10 ? A0 : L1;
        A1.x += i1.x; A1.y += i1.y;
        uint2 A2 = e21 ? A1 : (e20 ? A0 : L2);
        A2.x += i2.x; A2.y += i2.y;
        uint2 A3 = e32 ? A2 : (e31 ? A1 : (e30 ? A0 : L3));
        A3.x += i3.x; A3.y += i3.y;
        sts64(r0 + p * 256, A0);
        sts64(r1 + p * 256, A1);
        sts64(r2 + p * 256, A2);
        sts64(r3 + p * 256, A3);
        if (p == 0) { acc0 |= A0.x | A1.x | A2.x | A3.x; acc |= A0.y | A1.y | A2.y | A3.y; }
        else { acc |= A0.x | A0.y | A1.x | A1.y | A2.x | A2.y | A3.x | A3.y; }
    }
}

// The read-modify-write chain of a group (a request's load may alias an
// earlier request's store, so updates are serialised through shared memory,
// two requests per link) interleaved, in program order, with the
// bucket-table lookups of the lane's next group: each lookup issues right
// behind a store and its result is only needed in the next iteration, so it
// fills the chain's load-latency gaps instead of running before it.
// Returns the guard bits.
template <int N, bool FLAGS, int MODE>
__device__ __forceinline__ uint32_t update_fast(const Group<N, FLAGS> &g, const U8x &row, uint32_t lane_base,
                                                const U8x &wn, const WarpSmem &W, int P, LutGeom geo,
                                                uint32_t rowbytes, U8x &on, uint32_t &en) {
    uint32_t acc0 = 0u, acc = 0u;
    if (MODE == kModeLut) {
#if SPROUT_LOOKUP_ORDER == 1
        // A/B: the next group's lookups first, then the read-modify-write chain
#pragma unroll
        for (int k = 0; k < 8; ++k) on.v[k] = lut_offset(wn.v[k], geo, rowbytes, lane_base, en);
#pragma unroll
        for (int k = 0; k < 8; k += 2) rmw_pair<N, FLAGS>(g, k, row.v[k], row.v[k + 1], acc0, acc);
#elif SPROUT_LOOKUP_ORDER == 2
        // A/B: four lookups ahead of each pair
#pragma unroll
        for (int k = 0; k < 4; ++k) on.v[k] = lut_offset(wn.v[k], geo, rowbytes, lane_base, en);
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
            rmw_pair<N, FLAGS>(g, k, row.v[k], row.v[k + 1], acc0, acc);
            if (k + 4 < 8) {
                on.v[k + 4] = lut_offset(wn.v[k + 4], geo, rowbytes, lane_base, en);
                on.v[k + 5] = lut_offset(wn.v[k + 5], geo, rowbytes, lane_base, en);
            }
        }
#elif SPROUT_RMW_QUAD
#pragma unroll
        for (int k = 0; k < 8; k += 4) {
            rmw_quad<N, FLAGS>(g, k, row.v[k], row.v[k + 1], row.v[k + 2], row.v[k + 3], acc0, acc);
#pragma unroll
            for (int u = 0; u < 4; ++u) on.v[k + u] = lut_offset(wn.v[k + u], geo, rowbytes, lane_base, en);
        }
#else
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
            rmw_pair<N, FLAGS>(g, k, row.v[k], row.v[k + 1], acc0, acc);
            on.v[k] = lut_offset(wn.v[k], geo, rowbytes, lane_base, en);
            on.v[k + 1] = lut_offset(wn.v[k + 1], geo, rowbytes, lane_base, en);
        }
#endif
    } else {
#pragma unroll
        for (int k = 0; k < 8; k += 2) rmw_pair<N, FLAGS>(g, k, row.v[k], row.v[k + 1], acc0, acc);
        en = group_offsets<MODE>(wn, W, P, geo, rowbytes, lane_base, on);
    }
    return (acc0 & kGuard0) | (acc & kGuard);
}

// token of request k (runtime) at level i
template <int N, bool FLAGS>
__device__ __forceinline__ uint32_t token_rt(const Group<N, FLAGS> &g, int i, int k) {
    const uint4 &u = g.t[i];
    const int h = k >> 1;
    const uint32_t wd = h == 0 ? u.x : h == 1 ? u.y : h == 2 ? u.z : u.w;
    return (k & 1) ? (wd >> 16) : (wd & 0xFFFFu);
}

// packed word m of one request from its tokens tk[0..N-1] (word 0 with the
// count increment; see the row layout above)
template <int N>
__device__ __forceinline__ uint32_t word_of_tokens(const uint32_t (&tk)[N], int m) {
    if (m == 0) return tk[0] + (1u << kW0Shift);
    const uint32_t lo = tk[2 * m - 1];
    const uint32_t hi = (2 * m <= N - 1) ? tk[2 * m] : 0u;
    return lo | (hi << 16);
}

// Rare paths, inline (a call would make the warp wait for its in-flight
// prefetch loads) and rolled over the 8 requests (small code).
// Revert a fast update (exact: 32-bit word arithmetic is modular) and add the
// group's requests into the 64-bit accumulators instead ...
template <int N, bool FLAGS>
__device__ __forceinline__ void redo_wide(const Group<N, FLAGS> &g, const U8x &row, uint32_t lane_base,
                                          unsigned long long *wide, uint32_t rowbytes, uint32_t discard_off) {
    constexpr int NW = Words<N>::NW;
    constexpr int NP = Words<N>::NP;
#pragma unroll 1
    for (int k = 0; k < 8; ++k) {
        const uint32_t r = sel8(row, k);
        uint32_t tk[N];
#pragma unroll
        for (int i = 0; i < N; ++i) tk[i] = token_rt<N, FLAGS>(g, i, k);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            uint2 cur = lds64(r + p * 256);
            cur.x -= word_of_tokens<N>(tk, 2 * p);
            if (2 * p + 1 < NW) cur.y -= word_of_tokens<N>(tk, 2 * p + 1);
            sts64(r + p * 256, cur);
        }
        if (r != lane_base + discard_off) {
            unsigned long long *wr = wide + (size_t)((r - lane_base) / rowbytes) * (N + 1);
            wide_add(&wr[0], 1u);
#pragma unroll
            for (int i = 0; i < N; ++i) wide_add(&wr[1 + i], tk[i]);
        }
    }
}

// ... and spill every row of the group with a guard bit set
template <int N>
__device__ __forceinline__ void spill_group(const U8x &row, uint2 *hist, unsigned long long *wide, uint32_t lane,
                                            uint32_t rowbytes, uint32_t lane_base) {
    constexpr int NP = Words<N>::NP;
#pragma unroll 1
    for (int k = 0; k < 8; ++k) {
        const int entry = (int)((sel8(row, k) - lane_base) / rowbytes);
        uint32_t acc = 0u;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const uint2 v = hist[((size_t)entry * NP + p) * 32 + lane];
            acc |= (p == 0 ? (v.x & kGuard0) : (v.x & kGuard)) | (v.y & kGuard);
        }
        if (acc) spill_entry<N>(hist, wide, entry, lane);
    }
}

// One partial group (requests outside [lo, hi) belong to another segment) --
// the careful 64-bit path, used at segment ends.
template <int N, bool FLAGS, int MODE>
__device__ __forceinline__ void process_partial(const Group<N, FLAGS> &g, int64_t v, int lo, int hi,
                                                const SimArgs &a, const WarpSmem &W, int P, LutGeom geo,
                                                uint32_t &err) {
    const uint32_t rowbytes = Words<N>::NP * 256;
    U8x w, off;
    group_draws(v, a, w);
    const uint32_t eor = group_offsets<MODE>(w, W, P, geo, rowbytes, 0u, off);
    if (MODE == kModeLut && (eor & 4u)) fix_offsets(w, off, W.keys, P, geo, rowbytes, 0u);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const bool inr = k >= lo && k < hi;
        const int entry = entry_of<FLAGS>((int)(off.v[k] / rowbytes), g.f, k, a.nb, a.NC, inr, err);
        if (entry != a.NC * a.nb) add_wide<N, FLAGS>(W.wide, g, entry, k);
    }
}

// Generic path: per request, per cell, compare the draw with the cell's
// thresholds (count-and-clamp rule) and add into the global per-cell
// counters with atomics; segment stats go to wide rows [c*nb] / [c*nb+1].
template <int N, bool FLAGS>
__device__ __forceinline__ void slow_segment(const SimArgs &a, const WarpSmem &W, int64_t sl, int64_t s0, int64_t s1,
                                          uint32_t &err) {
    const uint32_t lane = lane_id();
    const int X = a.X, NC = a.NC;
    const int64_t cell0 = sl * X;
    for (int64_t i = lane; i < (int64_t)X * NC * N; i += 32) {
        a.cnt[cell0 * NC * N + i] = 0ull;
        a.tok[cell0 * NC * N + i] = 0ull;
    }
    __syncwarp();
    for (int64_t r = s0 + lane; r < s1; r += 32) {
        const uint64_t gidx = a.first_request + (uint64_t)r;
        const uint64_t blk = gidx >> 2;
        const Philox4 d = philox4x32_10((uint32_t)blk, (uint32_t)(blk >> 32), 0u, 0u, (uint32_t)a.seed,
                                        (uint32_t)(a.seed >> 32));
        const uint32_t w = d.v[gidx & 3u];
        int cls = 0;
        bool pinned = false;
        if (FLAGS) {
            const uint8_t f = a.flags[r];
            pinned = f & 1u;
            cls = (f >> 1) & 3;
        }
        if (cls >= NC) {
            err |= SPROUT_TRACE_BAD_CLASS;
            continue;
        }
        unsigned long long *wr = W.wide + (size_t)(cls * a.nb) * (N + 1);
        atomicAdd(&wr[0], 1ull);
        for (int i = 0; i < N; ++i) atomicAdd(&wr[1 + i], (unsigned long long)a.tokens[(size_t)i * a.pitch + r]);
        if (pinned) atomicAdd(&W.wide[(size_t)(cls * a.nb + 1) * (N + 1)], 1ull);
        for (int j = 0; j < X; ++j) {
            const int64_t cell = cell0 + j;
            if (a.cell_status[cell] != SPROUT_CELL_OK) continue;
            int L = 0;
            if (!pinned) {
                int c = 0;
                for (int i = 0; i + 1 < N; ++i) c += (w >= a.threshold[cell * (N - 1) + i]) ? 1 : 0;
                const int ml = a.max_level[cell];
                L = c < ml ? c : ml;
            }
            atomicAdd(reinterpret_cast<unsigned long long *>(&a.cnt[(cell * NC + cls) * N + L]), 1ull);
            atomicAdd(reinterpret_cast<unsigned long long *>(&a.tok[(cell * NC + cls) * N + L]),
                      (unsigned long long)a.tokens[(size_t)L * a.pitch + r]);
        }
    }
    err |= SPROUT_TRACE_SLOW_PATH;
    __syncwarp();
}

// Segment statistics and the Base counterfactual (every request at L0,
// P:366): counts and token sums per class, fp64 Base energy/time/carbon
// (Eq. 1) and quality.  Fast path: totals = row `tot_row` (prefix total) +
// the pinned row; slow path: totals in row 0, pinned count in row 1.
template <int N>
__device__ __forceinline__ void write_seg_stats(const SimArgs &a, const WarpSmem &W, int64_t sl, double kp, double q0,
                                             int tot_row, int pin_row, bool fast, const CostConst &cost) {
    if (lane_id() == 0) {
    const int NC = a.NC, nb = a.nb;
    double bE = 0.0, bT = 0.0, m = 0.0;
    for (int c = 0; c < NC; ++c) {
        const unsigned long long *tr = W.wide + (size_t)(c * nb + tot_row) * (N + 1);
        const unsigned long long *pr = W.wide + (size_t)(c * nb + pin_row) * (N + 1);
        const unsigned long long mc = tr[0] + (fast ? pr[0] : 0ull);
        a.seg_count[sl * NC + c] = mc;
        a.seg_pinned[sl * NC + c] = pr[0];
        unsigned long long t0 = 0;
        for (int i = 0; i < N; ++i) {
            const unsigned long long t = tr[1 + i] + (fast ? pr[1 + i] : 0ull);
            a.seg_tok[(sl * NC + c) * N + i] = t;
            if (i == 0) t0 = t;
        }
        bE += (double)mc * cost.ef[c][0] + (double)t0 * cost.et[c][0];
        bT += (double)mc * cost.pf[c][0] + (double)t0 * cost.pt[c][0];
        m += (double)mc;
    }
    a.seg_base[sl * 4 + 0] = bE;
    a.seg_base[sl * 4 + 1] = bT;
    a.seg_base[sl * 4 + 2] = kp * bE + a.k1 * bT;
    a.seg_base[sl * 4 + 3] = m * q0;
    }
}

__device__ __forceinline__ void zero_cell(const SimArgs &a, int64_t cell, int NCN) {
    for (int i = 0; i < NCN; ++i) { a.cnt[cell * NCN + i] = 0ull; a.tok[cell * NCN + i] = 0ull; }
    a.energy[cell] = 0.0; a.time_s[cell] = 0.0; a.carbon[cell] = 0.0; a.quality[cell] = 0.0;
}

// Per-cell integer statistics (from the histogram prefix sums, or from the
// slow path's global counters) and the closed-form fp64 totals of Eq. 1.
// `pre` (N <= 3, X <= 64): the status and packed level boundaries of the
// lane's cells lane and lane + 32 were loaded one segment ahead (SegCells).
struct SegCells {
    uint32_t st[2];    // cell_status
    uint32_t bw[2];    // seg_bnd of levels 1..N-1, packed u16 (N <= 3)
};

template <int N>
__device__ __forceinline__ void cell_epilogue(const SimArgs &a, const WarpSmem &W, int64_t sl, int K, double kp,
                                           const double *qrow, bool fast, const CostConst &cost, bool pre,
                                           const SegCells &sc) {
    const int NC = a.NC, nb = a.nb;
    int t = 0;
    for (int j = lane_id(); j < a.X; j += 32, ++t) {
        const int64_t cell = sl * a.X + j;
        // status and level boundaries are loaded together (independent loads, one round trip)
        int bnd[N + 1];
        bnd[0] = 0;
        bnd[N] = K + 1;
        if (fast) {
            if (N <= 3 && pre) {
                const uint32_t bw = t == 0 ? sc.bw[0] : sc.bw[1];
#pragma unroll
                for (int L = 1; L < N; ++L) bnd[L] = (int)((bw >> (16 * (L - 1))) & 0xFFFFu);
            } else {
#pragma unroll
                for (int L = 1; L < N; ++L) bnd[L] = a.seg_bnd[cell * (N - 1) + (L - 1)];
            }
        }
        const uint32_t st = pre ? (t == 0 ? sc.st[0] : sc.st[1]) : a.cell_status[cell];
        if (st != SPROUT_CELL_OK) {
            zero_cell(a, cell, NC * N);
            continue;
        }
        double E = 0.0, T = 0.0, Q = 0.0;
        for (int c = 0; c < NC; ++c) {
            const unsigned long long *pre = W.wide + (size_t)(c * nb) * (N + 1);
            const unsigned long long *pin = W.wide + (size_t)(c * nb + nb - 1) * (N + 1);
#pragma unroll
            for (int L = 0; L < N; ++L) {
                unsigned long long cn, tk;
                uint64_t *pc = &a.cnt[(cell * NC + c) * N + L];
                uint64_t *pt = &a.tok[(cell * NC + c) * N + L];
                if (fast) {
                    cn = pre[(size_t)bnd[L + 1] * (N + 1)] - pre[(size_t)bnd[L] * (N + 1)];
                    tk = pre[(size_t)bnd[L + 1] * (N + 1) + 1 + L] - pre[(size_t)bnd[L] * (N + 1) + 1 + L];
                    if (L == 0) { cn += pin[0]; tk += pin[1]; }
                    *pc = cn;
                    *pt = tk;
                } else {
                    cn = __ldcg(reinterpret_cast<const unsigned long long *>(pc));
                    tk = __ldcg(reinterpret_cast<const unsigned long long *>(pt));
                }
                const double n_ = (double)cn, t_ = (double)tk;
                E += n_ * cost.ef[c][L] + t_ * cost.et[c][L];
                T += n_ * cost.pf[c][L] + t_ * cost.pt[c][L];
                Q += n_ * qrow[L];
            }
        }
        a.energy[cell] = E;
        a.time_s[cell] = T;
        a.carbon[cell] = kp * E + a.k1 * T;
        a.quality[cell] = Q;
    }
}

// Lane-private slots -> 64-bit per-entry totals, then the exclusive prefix
// over draw bins 0..K+1 per (class, field).
template <int N>
__device__ __forceinline__ void readout(const SimArgs &a, const WarpSmem &W, int K) {
    constexpr int NW = Words<N>::NW;
    constexpr int NP = Words<N>::NP;
    const uint32_t lane = lane_id();
    const int NC = a.NC, nb = a.nb;
    const int used = K + 2;   // draw bins 0..K and the pinned bin
    {
        for (int e = lane; e < NC * used; e += 32) {
            int c = 0, b = e;   // (class, bin) of entry e without a division (NC <= 4)
            while (b >= used) { b -= used; ++c; }
            {
                const int entry = c * nb + (b <= K ? b : nb - 1);
                unsigned long long *wr = W.wide + (size_t)entry * (N + 1);
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    uint2 *row = W.hist + ((size_t)entry * NP + p) * 32;
                    uint32_t sv[4] = {0u, 0u, 0u, 0u};
#pragma unroll 8
                    for (int q = 0; q < 32; ++q) {
                        const int idx = (q + (int)lane) & 31;   // rotated: conflict-free
                        const uint2 val = row[idx];
                        row[idx] = make_uint2(0u, 0u);
                        sv[0] += p == 0 ? (val.x & kW0Low) : (val.x & 0xFFFFu);
                        sv[1] += p == 0 ? (val.x >> kW0Shift) : (val.x >> 16);
                        sv[2] += val.y & 0xFFFFu;
                        sv[3] += val.y >> 16;
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int m = 2 * p + h;
                        if (m >= NW) break;
                        wr[word_lo_field(m)] += sv[2 * h];
                        if (word_hi_field(m) <= N) wr[word_hi_field(m)] += sv[2 * h + 1];
                    }
                }
            }
        }
    }
    for (int i = lane; i < NP * 32; i += 32) W.hist[(size_t)(NC * nb) * NP * 32 + i] = make_uint2(0u, 0u);  // discard
    for (int i = lane; i < N + 1; i += 32) W.wide[(size_t)(NC * nb) * (N + 1) + i] = 0ull;
    __syncwarp();
    for (int e = lane; e < NC * (N + 1); e += 32) {
        const int c = e / (N + 1), f = e % (N + 1);
        unsigned long long run = 0ull;
        for (int b = 0; b <= K + 1; ++b) {
            unsigned long long *pt = &W.wide[(size_t)(c * nb + b) * (N + 1) + f];
            const unsigned long long v2 = *pt;
            *pt = run;
            run += v2;
        }
    }
    __syncwarp();
}

// The requests of a segment outside its whole groups of 8 (head: up to the
// first 8-aligned index, tail: after the last), at most 14, one per lane:
// each lane draws its request's word, finds its bin and adds it into its own
// lane-private row (tokens >= 4096 go to the 64-bit accumulators).  All lanes
// work at once, so a short segment does not serialise on two lanes.
template <int N, bool FLAGS, int MODE, bool VB>
__device__ __forceinline__ void process_ends(const SimArgs &a, const WarpSmem &W, int64_t s0, int64_t s1, int P,
                                             LutGeom geo, uint32_t &err) {
    constexpr int NW = Words<N>::NW;
    constexpr int NP = Words<N>::NP;
    constexpr uint32_t rowbytes = NP * 256;
    const uint32_t lane = lane_id();
    const int64_t h_end = min(s1, (s0 + 7) & ~(int64_t)7);
    const int64_t t_beg = max(h_end, s1 & ~(int64_t)7);
    const int n_head = (int)(h_end - s0), n_tail = (int)(s1 - t_beg);
    int64_t r = -1;
    if ((int)lane < n_head) r = s0 + lane;
    else if (lane >= 8 && (int)lane < 8 + n_tail) r = t_beg + (lane - 8);
    if (r < 0) return;
    const uint64_t gidx = a.first_request + (uint64_t)r;
    const uint64_t blk = gidx >> 2;
    const Philox4 d = philox4x32_10_rk((uint32_t)blk, (uint32_t)(blk >> 32), 0u, 0u, a.rk0, a.rk1);
    const uint32_t k3 = (uint32_t)(gidx & 3u);
    const uint32_t w = k3 == 0 ? d.v[0] : k3 == 1 ? d.v[1] : k3 == 2 ? d.v[2] : d.v[3];
    int bin;
    if (MODE == kModeLut) {
        const uint32_t dd = max(w, geo.base);
        const uint2 e = lds64(geo.bias + ((dd >> geo.s) << 3));
        bin = (e.y & 4u) ? find_bin(W.keys, P, w) : (int)(e.y / rowbytes) + (dd > e.x ? 1 : 0);
    } else {
        bin = find_bin(W.keys, P, w);
    }
    if (VB) a.bins_out[r] = (uint8_t)bin;   // verify mode: the bin this kernel found
    int entry = bin;
    if (FLAGS) {
        const uint32_t fb = a.flags[r];
        const int cls = (int)((fb >> 1) & 3u);
        if (fb & 1u) entry = a.nb - 1;
        entry += cls * a.nb;
        if (cls >= a.NC) {
            err |= SPROUT_TRACE_BAD_CLASS;
            return;
        }
    }
    uint32_t tk[N];
    uint32_t big = 0u;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        tk[i] = a.tokens[(size_t)i * a.pitch + r];
        big |= tk[i];
    }
    if (big >= 4096u) {
        unsigned long long *wr = W.wide + (size_t)entry * (N + 1);
        wide_add(&wr[0], 1u);
#pragma unroll
        for (int i = 0; i < N; ++i) wide_add(&wr[1 + i], tk[i]);
        return;
    }
    const uint32_t addr = smem_u32(W.hist) + lane * 8u + (uint32_t)entry * rowbytes;
    uint32_t guard = 0u;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        uint2 cur = lds64(addr + p * 256);
        cur.x += word_of_tokens<N>(tk, 2 * p);
        if (2 * p + 1 < NW) cur.y += word_of_tokens<N>(tk, 2 * p + 1);
        sts64(addr + p * 256, cur);
        guard |= (p == 0 ? (cur.x & kGuard0) : (cur.x & kGuard)) | (cur.y & kGuard);
    }
    if (guard) spill_entry<N>(W.hist, W.wide, entry, lane);
}

// L2 prefetch distance of the streaming loop, in warp iterations (one
// iteration = 32 groups = 512 contiguous bytes per token plane)
#ifndef SPROUT_PREFETCH_ITERS
#define SPROUT_PREFETCH_ITERS 3
#endif
constexpr int kPrefetchIters = SPROUT_PREFETCH_ITERS;

__device__ __forceinline__ void prefetch_l2(const void *p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Stream a segment's requests [s0, s1).  Lane l takes the full groups
// gf + l, gf + l + 32, ... (warp iteration i covers groups gf + 32i ..
// gf + 32i + 31: every 128-bit load of the warp reads 512 contiguous bytes
// of a plane).  Memory-level parallelism comes from L2 prefetches of the
// lane's group kPrefetchIters iterations ahead (one per plane, no
// registers held), so the register loads -- one group ahead, ping-pong --
// hit L2; this keeps the unrolled loop to two bodies (instruction-cache
// footprint).  Software pipeline: while
// group v's tokens are added into the histogram, the Philox draws and
// histogram rows of the lane's next group v+32 are computed in the same
// basic block (they do not depend on token data), so the scheduler overlaps
// the integer rounds with the shared-memory read-modify-write chain.  The
// (at most two) partial groups at the segment's ends take the careful
// 64-bit path.
template <int N, bool FLAGS, int MODE, bool VB>
__device__ __forceinline__ void stream_segment(const SimArgs &a, const WarpSmem &W, int64_t s0, int64_t s1, int P,
                                               LutGeom geo, uint32_t &err) {
    if (s1 <= s0) return;
    const uint32_t lane = lane_id();
    const int64_t gf = (s0 + 7) >> 3;       // first full group
    const int64_t ge = s1 >> 3;             // one past the last full group
    auto prefetch_group = [&](int64_t v) {
#pragma unroll
        for (int i = 0; i < N; ++i) prefetch_l2(reinterpret_cast<const uint4 *>(a.tokens + (size_t)i * a.pitch) + v);
    };
    for (int it = 1; it < kPrefetchIters; ++it)
        if (gf + lane + 32 * it < ge) prefetch_group(gf + lane + 32 * it);
    process_ends<N, FLAGS, MODE, VB>(a, W, s0, s1, P, geo, err);
    constexpr uint32_t rowbytes = Words<N>::NP * 256;
    const uint32_t lane_base = smem_u32(W.hist) + lane * 8u;
    const uint32_t discard_row = lane_base + (uint32_t)(a.NC * a.nb) * rowbytes;
    const uint32_t pin_row = lane_base + (uint32_t)(a.nb - 1) * rowbytes;
    const uint32_t class_bytes = (uint32_t)a.nb * rowbytes;
    const int64_t v0 = gf + lane;
    const uint32_t n_mine = v0 < ge ? (uint32_t)((ge - v0 + 31) >> 5) : 0u;   // this lane's groups
    if (n_mine == 0) return;
    // Per-lane cursors advanced by one warp iteration (32 groups) per body:
    // one pointer per token plane at the lane's current group (so the next
    // group's load and the prefetch are immediate offsets), flags, and the
    // Philox block of the group two iterations ahead.
    const uint8_t *qp[N];
#pragma unroll
    for (int q = 0; q < N; ++q) qp[q] = reinterpret_cast<const uint8_t *>(a.tokens + (size_t)q * a.pitch) + (size_t)v0 * 16u;
    const uint8_t *fp = FLAGS ? a.flags + (size_t)v0 * 8u : nullptr;
    uint64_t blk = ((a.first_request + (uint64_t)v0 * 8u) >> 2) + 128u;
    auto load_at = [&](Group<N, FLAGS> &g, int it) {   // group of iteration (current + it)
#pragma unroll
        for (int q = 0; q < N; ++q) {
#if SPROUT_LD_HINT
            const uint4 *src = reinterpret_cast<const uint4 *>(qp[q]) + 32 * it;
            asm volatile("ld.global.cs.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(g.t[q].x), "=r"(g.t[q].y), "=r"(g.t[q].z), "=r"(g.t[q].w) : "l"(src));
#else
            g.t[q] = __ldcs(reinterpret_cast<const uint4 *>(qp[q]) + 32 * it);
#endif
        }
        if (FLAGS) g.f = __ldcs(reinterpret_cast<const uint2 *>(fp) + 32 * it);
    };

    // Pipeline state (ping-pong names, so no register copies): body b works
    // on group v with rows oc[b]; it looks up the rows of v+32 (into
    // oc[b^1]) from the draws wq[b] computed one body earlier, and draws
    // for v+64 (into wq[b^1]).  The three chains -- Philox rounds, table
    // lookups, histogram read-modify-writes -- are mutually independent
    // inside a body.  All rare work (a token >= 4096, a guard bit, a
    // multi-key bucket) sits behind one branch per body; the prefetch and
    // the next load are predicated, and the loop runs whole body pairs with
    // a one-body tail, so a body has no other branch.
    Group<N, FLAGS> g[2];
    U8x oc[2], wq[2];
    load_at(g[0], 0);
    {
        U8x w;
        group_draws_blk(blk - 128u, a, w);
        const uint32_t e = group_offsets<MODE>(w, W, P, geo, rowbytes, lane_base, oc[0]);
        if (MODE == kModeLut && (e & 4u)) fix_offsets(w, oc[0], W.keys, P, geo, rowbytes, lane_base);
        group_draws_blk(blk - 64u, a, wq[0]);
    }
    auto body = [&](auto bc, uint32_t i) {
        constexpr int b = decltype(bc)::value;
#if !SPROUT_NO_PREFETCH
        {
            const uint32_t pf = (i + kPrefetchIters < n_mine) ? 1u : 0u;
#pragma unroll
            for (int q = 0; q < N; ++q)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %0, 0;\n\t@p prefetch.global.L2 [%1];\n\t}"
                             ::"r"(pf), "l"(qp[q] + 512 * kPrefetchIters));
        }
#endif
        if (i + 1 < n_mine) load_at(g[b ^ 1], 1);
        group_draws_blk(blk, a, wq[b ^ 1]);
        U8x row;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            row.v[k] = row_of<FLAGS>(oc[b].v[k], g[b].f, k, pin_row, class_bytes, a.NC, discard_row, err);
        if (VB) {   // verify mode: the eight draw bins this kernel looked up, one 8-byte store
            uint32_t lo8 = 0u, hi8 = 0u;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                lo8 |= ((oc[b].v[k] - lane_base) / rowbytes) << (8 * k);
                hi8 |= ((oc[b].v[4 + k] - lane_base) / rowbytes) << (8 * k);
            }
            reinterpret_cast<uint2 *>(a.bins_out)[v0 + 32 * (int64_t)i] = make_uint2(lo8, hi8);
        }
        uint32_t en = 0u;
        const uint32_t acc =
            update_fast<N, FLAGS, MODE>(g[b], row, lane_base, wq[b], W, P, geo, rowbytes, oc[b ^ 1], en);
        const uint32_t big = group_or<N, FLAGS>(g[b]) & kBigTok;
        if (big | acc | (MODE == kModeLut ? (en & 4u) : 0u)) {
            if (big) redo_wide<N, FLAGS>(g[b], row, lane_base, W.wide, rowbytes, discard_row - lane_base);
            if (acc) spill_group<N>(row, W.hist, W.wide, lane, rowbytes, lane_base);
            if (MODE == kModeLut && (en & 4u)) fix_offsets(wq[b], oc[b ^ 1], W.keys, P, geo, rowbytes, lane_base);
        }
#pragma unroll
        for (int q = 0; q < N; ++q) qp[q] += 512;
        if (FLAGS) fp += 256;
        blk += 64u;
    };
    uint32_t i = 0;
    for (; i + 2 <= n_mine; i += 2) {
        body(std::integral_constant<int, 0>{}, i);
        body(std::integral_constant<int, 1>{}, i + 1);
    }
    if (i < n_mine) body(std::integral_constant<int, 0>{}, i);
}

// A segment without breakpoints (K = 0: every valid cell's mix is pure, so
// each cell's level is the same for every draw -- e.g. CO2_Opt, or an LP
// whose floor is inactive) and without flags: every request is in draw bin
// 0 whatever its draw, so no draw is needed and the bin-0 statistics are the
// segment's request count and token sums.  Lanes sum the tokens of their
// groups per level in registers (4 groups of 8 requests in flight per lane),
// the warp reduces them, and lane 0 adds them to the 64-bit row of bin 0;
// the epilogue then runs unchanged.
template <int N>
__device__ __forceinline__ void stream_segment_k0(const SimArgs &a, const WarpSmem &W, int64_t s0, int64_t s1) {
    const uint32_t lane = lane_id();
    uint64_t acc[N];
#pragma unroll
    for (int q = 0; q < N; ++q) acc[q] = 0ull;
    const int64_t gf = (s0 + 7) >> 3, ge = s1 >> 3;   // full groups [gf, ge)
    // head / tail requests (at most 7 each), one per lane
    {
        const int64_t h_end = min(s1, (s0 + 7) & ~(int64_t)7);
        const int64_t t_beg = max(h_end, s1 & ~(int64_t)7);
        int64_t r = -1;
        if ((int64_t)lane < h_end - s0) r = s0 + lane;
        else if (lane >= 8 && (int64_t)(lane - 8) < s1 - t_beg) r = t_beg + (lane - 8);
        if (r >= 0) {
#pragma unroll
            for (int q = 0; q < N; ++q) acc[q] += a.tokens[(size_t)q * a.pitch + r];
        }
    }
    auto half_sum = [](uint4 t) -> uint32_t {   // sum of the 8 u16 tokens of a 16-byte group (< 2^19)
        return (t.x & 0xFFFFu) + (t.x >> 16) + (t.y & 0xFFFFu) + (t.y >> 16) + (t.z & 0xFFFFu) + (t.z >> 16) +
               (t.w & 0xFFFFu) + (t.w >> 16);
    };
    constexpr int U = 4;   // groups in flight per lane
    int64_t v = gf + lane;
    for (; v + 32 * (U - 1) < ge; v += 32 * U) {
        uint4 t[U][N];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int q = 0; q < N; ++q)
                t[u][q] = __ldcs(reinterpret_cast<const uint4 *>(a.tokens + (size_t)q * a.pitch) + v + 32 * u);
#pragma unroll
        for (int q = 0; q < N; ++q) {
            uint32_t sq = 0u;   // < 4 * 2^19
#pragma unroll
            for (int u = 0; u < U; ++u) sq += half_sum(t[u][q]);
            acc[q] += sq;
        }
    }
    for (; v < ge; v += 32) {
#pragma unroll
        for (int q = 0; q < N; ++q)
            acc[q] += half_sum(__ldcs(reinterpret_cast<const uint4 *>(a.tokens + (size_t)q * a.pitch) + v));
    }
#pragma unroll
    for (int q = 0; q < N; ++q)
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) acc[q] += __shfl_xor_sync(0xFFFFFFFFu, acc[q], d);
    if (lane == 0) {
        unsigned long long *wr = W.wide;   // class 0, bin 0
        wr[0] += (unsigned long long)(s1 - s0);
#pragma unroll
        for (int q = 0; q < N; ++q) wr[1 + q] += acc[q];
    }
    __syncwarp();
}

template <int N, bool FLAGS, bool VB>
__global__ void __launch_bounds__(32 * kMaxTraceWarps, 1) trace_kernel(const __grid_constant__ SimArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ CostConst cost;   // per-launch coefficients (dynamic [class][level] indexing)
    const int warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    const WarpSmem W = carve(smem + (size_t)warp * a.warp_smem, a);
    const int NC = a.NC, nb = a.nb, X = a.X;
    const int entries = NC * nb + 1;
    for (int i = threadIdx.x; i < (int)(sizeof(CostConst) / 8); i += blockDim.x)
        reinterpret_cast<double *>(&cost)[i] = reinterpret_cast<const double *>(&a.cost)[i];
    for (int i = lane; i < entries * Words<N>::NP * 32; i += 32) W.hist[i] = make_uint2(0u, 0u);
    for (int i = lane; i < entries * (N + 1); i += 32) W.wide[i] = 0ull;
    __syncthreads();

    uint32_t err = 0u;
    // Segment pipeline (hides the per-segment global round trips, which
    // dominate for short segments): the queue ticket for the segment after
    // next is taken while the current one is processed (lane 0 holds it until
    // needed), and the next segment's metadata and keys are loaded into
    // registers one segment ahead.
    constexpr int kKeyRegs = 4;   // keys prefetched per lane (kcap <= 128)
    struct SegPre {
        int64_t sl, s0, s1;
        int meta;
        double k0;
        uint32_t key[kKeyRegs];
        SegCells sc;
    };
    const bool pre_cells = N <= 3 && X <= 64;
    auto load_pre = [&](int64_t sl) {
        SegPre p;
        p.sl = sl;
        p.meta = -3;
        p.s0 = p.s1 = 0;
        p.k0 = 0.0;
#pragma unroll
        for (int t = 0; t < kKeyRegs; ++t) p.key[t] = 0xFFFFFFFFu;
        p.sc.st[0] = p.sc.st[1] = 0xFFu;
        p.sc.bw[0] = p.sc.bw[1] = 0u;
        if (sl < a.n_segments) {
            p.meta = a.seg_meta[sl];
            p.s0 = a.seg_offsets[sl];
            p.s1 = a.seg_offsets[sl + 1];
            p.k0 = a.k0[a.first_segment + sl];
            if (pre_cells) {
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    const int j = (int)lane + 32 * t;
                    if (j < X) {
                        const int64_t cell = sl * X + j;
                        p.sc.st[t] = a.cell_status[cell];
                        p.sc.bw[t] = N == 3 ? *reinterpret_cast<const uint32_t *>(a.seg_bnd + cell * 2)
                                   : N == 2 ? (uint32_t)a.seg_bnd[cell] : 0u;
                    }
                }
            }
            if (a.kcap > 0 && a.kcap <= 32 * kKeyRegs) {
#pragma unroll
                for (int t = 0; t < kKeyRegs; ++t) {
                    const int i = (int)lane + 32 * t;
                    if (i < a.kcap) p.key[t] = a.seg_keys[sl * a.kcap + i];
                }
            }
        }
        return p;
    };
    // Queue tickets hand out batches of a.seg_batch consecutive segments (one
    // atomic per batch: with many short segments a per-segment atomic on a
    // single counter serialises in L2).  Lane 0 holds the ticket of the
    // batch after the current one until it is needed.
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
    SegPre cur = load_pre(next_segment());
    for (;;) {
        const int64_t sl = cur.sl;
        if (sl >= a.n_segments) break;
        const SegPre nxt = load_pre(next_segment());
        const int64_t s = a.first_segment + sl;
        const int meta = cur.meta;
        const double *qrow =
            a.q + (a.profile_per_interval ? s : (s < 0xFFFFFFFFll ? (int64_t)a.div_t.div((uint32_t)s) : s / a.T)) * N;
        const double kp = cur.k0 * a.pue;

        if (meta == -2) {   // invalid offsets: segment skipped, outputs zero
            err |= SPROUT_TRACE_BAD_OFFSETS;
            for (int j = lane; j < X; j += 32) zero_cell(a, sl * X + j, NC * N);
            for (int i = lane; i < NC; i += 32) { a.seg_count[sl * NC + i] = 0ull; a.seg_pinned[sl * NC + i] = 0ull; }
            for (int i = lane; i < NC * N; i += 32) a.seg_tok[sl * NC * N + i] = 0ull;
            if (lane < 4) a.seg_base[sl * 4 + lane] = 0.0;
            cur = nxt;
            continue;
        }
        const int64_t s0 = cur.s0, s1 = cur.s1;
        if (meta == -1) {
            slow_segment<N, FLAGS>(a, W, sl, s0, s1, err);
            cell_epilogue<N>(a, W, sl, 0, kp, qrow, false, cost, false, cur.sc);
            __syncwarp();
            write_seg_stats<N>(a, W, sl, kp, qrow[0], 0, 1, false, cost);
            __syncwarp();
            for (int e = lane; e < NC * 2 * (N + 1); e += 32) {
                const int c = e / (2 * (N + 1)), rem = e % (2 * (N + 1));
                W.wide[(size_t)(c * nb + rem / (N + 1)) * (N + 1) + rem % (N + 1)] = 0ull;
            }
            __syncwarp();
            cur = nxt;
            continue;
        }
        const int K = meta;
        int P = 1;
        while (P < K + 1) P <<= 1;
        if (a.kcap <= 32 * kKeyRegs) {
#pragma unroll
            for (int t = 0; t < kKeyRegs; ++t) {
                const int i = (int)lane + 32 * t;
                if (i < P) W.keys[i] = i < K ? cur.key[t] : 0xFFFFFFFFu;
            }
        } else {
            for (int i = lane; i < P; i += 32) W.keys[i] = i < K ? a.seg_keys[sl * a.kcap + i] : 0xFFFFFFFFu;
        }
        __syncwarp();
        if (!FLAGS && K == 0) {
            stream_segment_k0<N>(a, W, s0, s1);
        } else if (a.lut && K >= kLutMinKeys && s1 - s0 >= kLutMinRequests) {
            const LutGeom geo = lut_geometry(W, K);
            build_lut(W, K, geo, Words<N>::NP * 256);
            stream_segment<N, FLAGS, kModeLut, VB>(a, W, s0, s1, P, geo, err);
        } else {
            stream_segment<N, FLAGS, kModeSearch, VB>(a, W, s0, s1, P, LutGeom{0u, 32 - kLutBits, 0u}, err);
        }
        __syncwarp();
        // the next segment's first groups into L2 while this one's epilogue
        // runs, so that its first loads hit L2 instead of HBM: a short
        // segment's first and last 16 groups, a long one's first
        // kPrefetchIters warp iterations and its last group
        if (nxt.sl < a.n_segments && nxt.meta >= -1 && nxt.s1 > nxt.s0) {
            const int64_t g0 = nxt.s0 >> 3, g1 = (nxt.s1 - 1) >> 3;
            if (nxt.s1 - nxt.s0 < 2048) {
                const int64_t v = (lane < 16) ? g0 + lane : g1 - (int64_t)(lane - 16);
                if (v >= g0 && v <= g1) {
#pragma unroll
                    for (int i = 0; i < N; ++i)
                        prefetch_l2(reinterpret_cast<const uint4 *>(a.tokens + (size_t)i * a.pitch) + v);
                    if (FLAGS) prefetch_l2(a.flags + (size_t)v * 8);
                }
            } else {
#pragma unroll 1
                for (int it = 0; it <= kPrefetchIters; ++it) {
                    const int64_t v = it < kPrefetchIters ? g0 + lane + 32 * it : g1;
#pragma unroll
                    for (int i = 0; i < N; ++i)
                        prefetch_l2(reinterpret_cast<const uint4 *>(a.tokens + (size_t)i * a.pitch) + v);
                    if (FLAGS) prefetch_l2(a.flags + (size_t)v * 8);
                }
            }
        }
        if (!pre_cells) {   // the epilogue's per-cell metadata into L2 (the lines of the two byte ranges)
            const int64_t c0 = sl * X;
            const uintptr_t a0 = reinterpret_cast<uintptr_t>(a.cell_status + c0) & ~(uintptr_t)127;
            const uintptr_t a1 = reinterpret_cast<uintptr_t>(a.cell_status + c0 + X);
            const uintptr_t b0 = reinterpret_cast<uintptr_t>(a.seg_bnd + c0 * (N - 1)) & ~(uintptr_t)127;
            const uintptr_t b1 = reinterpret_cast<uintptr_t>(a.seg_bnd + (c0 + X) * (N - 1));
            const int64_t na = (int64_t)((a1 - a0 + 127) / 128), nbl = (int64_t)((b1 - b0 + 127) / 128);
            for (int64_t ln = lane; ln < na + nbl; ln += 32)
                prefetch_l2(reinterpret_cast<const void *>(ln < na ? a0 + 128 * ln : b0 + 128 * (ln - na)));
        }
        readout<N>(a, W, K);
        cell_epilogue<N>(a, W, sl, K, kp, qrow, true, cost, pre_cells, cur.sc);
        __syncwarp();
        write_seg_stats<N>(a, W, sl, kp, qrow[0], K + 1, nb - 1, true, cost);
        __syncwarp();
        // clear the rows used by this segment: draw bins 0..K+1 and the pinned bin
        for (int c = 0; c < NC; ++c)
            for (int b = lane; b < K + 3; b += 32) {
                unsigned long long *wr = W.wide + (size_t)(c * nb + (b <= K + 1 ? b : nb - 1)) * (N + 1);
#pragma unroll
                for (int f = 0; f < N + 1; ++f) wr[f] = 0ull;
            }
        __syncwarp();
        cur = nxt;
    }
    err = __reduce_or_sync(0xFFFFFFFFu, err);
    if (lane == 0 && err) atomicOr(a.trace_status, err);
}

// ---------------------------------------------------------------------------
// trace_wide_kernel -- A/B EXPERIMENT, off by default (SPROUT_ENABLE_WIDE=1
// to build it in): measured 2.62 ms (mbarrier ring, token loads from global)
// and 3.88 ms (token planes TMA-staged through the ring) against
// trace_kernel's 2.08 ms on C4 (profiles/r02_c4_experiments.md).  A
// streaming kernel for n = 3 levels, one model class
// and no flags plane (the C4 xi sweep, the Sprout_Sta grid sweep).  Same
// method, histogram row format and epilogue as trace_kernel (a5-a8: one
// draw per request shared by the segment's cells, reading L10; the bin
// histogram; per-cell statistics from its prefix sums and Eq. 1 in closed
// form), warp-specialised:
//  * a TEAM of two warps owns one segment at a time.  The PRODUCER warp
//    computes each request's Philox word and its histogram row (bucket
//    table over the fixed range [0, 2^32), exact bin by binary search for the
//    rare draws in buckets holding several keys) and writes the rows into a
//    ring of shared-memory stages; the CONSUMER warp streams the token planes
//    (128-bit loads, L2 prefetch) and does the serial read-modify-writes of
//    its lane-private rows.  mbarriers (full / empty per stage) pace the ring.
//    The producer holds no histogram, so 8 teams (16 warps, 4 per scheduler)
//    fit in shared memory where trace_kernel fits 8 warps: the consumers'
//    load-latency-bound chains interleave with the producers' integer rounds;
//  * rows whose guard bits are set spill into a per-team 64-bit scratch in
//    global memory (rare); after the stream the table space holds the 64-bit
//    rows that the shared epilogue (cell_epilogue, write_seg_stats) reads;
//  * Philox rounds 0-2 are specialised on the counter's constant words
//    (c1 = H, constant over the launch; c2 = c3 = 0).
#ifndef SPROUT_WIDE_TEAMS
#define SPROUT_WIDE_TEAMS 7
#endif
#ifndef SPROUT_WIDE_LB
#define SPROUT_WIDE_LB 9
#endif
#ifndef SPROUT_WIDE_STAGES
#define SPROUT_WIDE_STAGES 4
#endif
#ifndef SPROUT_ENABLE_WIDE
#define SPROUT_ENABLE_WIDE 0   // A/B only: measured slower than trace_kernel on C4 (profiles/r02_c4_experiments.md)
#endif
#ifndef SPROUT_WIDE_AB_NOPHILOX
#define SPROUT_WIDE_AB_NOPHILOX 0   // A/B timing only (wrong results)
#endif
#ifndef SPROUT_WIDE_PREFETCH
#define SPROUT_WIDE_PREFETCH 3
#endif
constexpr int kWideTeams = SPROUT_WIDE_TEAMS;
constexpr int kWideLB = SPROUT_WIDE_LB;
constexpr int kWideBuckets = 1 << kWideLB;
constexpr int kWideShift = 32 - kWideLB;
constexpr int kWideStages = SPROUT_WIDE_STAGES;
constexpr int kWideMaxSMs = 256;   // the spill scratch is sized for this many SMs
// the table space must also hold the epilogue's 64-bit rows: (kcap + 3) * 4 * 8 <= kWideBuckets * 8
constexpr int kWideMaxKeys = (kWideBuckets / 4 - 3) < 253 ? (kWideBuckets / 4 - 3) : 253;
constexpr int kWideCtl = (16 * SPROUT_WIDE_STAGES + 48 + 127) / 128 * 128;   // per team: mbarriers full[S], empty[S], the segment record
// a ring stage: 256 u32 histogram row addresses (16-byte chunks h*32 + lane), then the
// iteration's three token planes (512 B each, copied by TMA bulk copies)
constexpr int kWideStageBytes = 1024 + 3 * 512;
#ifndef SPROUT_WIDE_L2PF
#define SPROUT_WIDE_L2PF 4   // bulk L2 prefetch distance of the token planes, in iterations beyond the ring
#endif

__host__ __device__ inline size_t wide_team_bytes(int kcap, int kp) {
    return (size_t)kWideCtl + (size_t)kWideStages * kWideStageBytes + (size_t)(kcap + 1) * 256 +
           (size_t)kWideBuckets * 8 + (size_t)kp * 4;
}

struct WideSeg {       // the team's current segment (written by the consumer before the team barrier)
    long long sl, s0, s1;
    int meta, P;
};

struct WideSmem {
    uint32_t bar_s;     // shared address of full[0] (full[i] = bar_s + 8i, empty[i] = bar_s + 8(S + i))
    WideSeg *seg;
    uint32_t ring_s;    // [S] stages of kWideStageBytes
    uint2 *hist;        // [(kcap + 1) rows][32 lanes] packed rows
    uint2 *lut;         // [kWideBuckets] {key, row offset}; after the stream: 64-bit rows [nb][4]
    uint32_t *keys;     // [kp] sorted keys, padded with 0xFFFFFFFF
    uint32_t hist_s, lut_s;
};

__device__ __forceinline__ void mbar_init(uint32_t addr, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(addr), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t addr) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t addr, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(done) : "r"(addr), "r"(parity) : "memory");
    } while (!done);
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t addr, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(addr),
                 "r"(bytes) : "memory");
}
// TMA bulk copy global -> shared (1D, 16-byte aligned, size a multiple of 16),
// completing `bytes` of the transaction count of mbarrier `mbar`
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void team_sync(int team) {
    asm volatile("bar.sync %0, 64;" ::"r"(team + 1) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr)
                 : "memory");
    return v;
}

// Philox4x32-10 of the counter (lo, H, 0, 0), H the launch's constant high
// word (reading L10: counter (g >> 2 lo32, g >> 2 hi32, 0, 0)).  Round 0's
// second product is 0 and its first output word H ^ k0[0] = ph_a is
// constant, so round 1's first product M0 * ph_a and round 2's c3 are launch
// constants (host-computed ph_d, ph_e).  Bit-identical to philox4x32_10_rk.
__device__ __forceinline__ Philox4 philox_lo(uint32_t lo, const SimArgs &a) {
    uint64_t p0 = (uint64_t)0xD2511F53u * lo;                // round 0
    uint32_t c2 = (uint32_t)(p0 >> 32) ^ a.rk1[0];
    uint32_t c3 = (uint32_t)p0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;               // round 1 (c0 = ph_a, c1 = 0)
    uint32_t c0 = (uint32_t)(p1 >> 32) ^ a.rk0[1];
    uint32_t c1 = (uint32_t)p1;
    c2 = c3 ^ a.ph_d;
    p0 = (uint64_t)0xD2511F53u * c0;                         // round 2 (c3 = lo32(M0 * ph_a))
    p1 = (uint64_t)0xCD9E8D57u * c2;
    c0 = (uint32_t)(p1 >> 32) ^ c1 ^ a.rk0[2];
    c2 = (uint32_t)(p0 >> 32) ^ a.ph_e;
    c1 = (uint32_t)p1;
    c3 = (uint32_t)p0;
#pragma unroll
    for (int r = 3; r < 10; ++r) {
        p0 = (uint64_t)0xD2511F53u * c0;
        p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ a.rk0[r];
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ a.rk1[r];
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
    }
    Philox4 o;
    o.v[0] = c0; o.v[1] = c1; o.v[2] = c2; o.v[3] = c3;
    return o;
}

struct WTok {
    uint4 t[3];
};

// 32-bit word h (0..3) of a 128-bit group load (runtime h: select cascade)
__device__ __forceinline__ uint32_t wword(const uint4 &u, int h) {
    return h == 0 ? u.x : h == 1 ? u.y : h == 2 ? u.z : u.w;
}
// packed increments of request k of a group: word 0 = tok_0 + 1 << 20, word 1 = tok_1 | tok_2 << 16
__device__ __forceinline__ uint2 wide_inc(const WTok &g, int k) {
    const uint32_t w0 = wword(g.t[0], k >> 1), w1 = wword(g.t[1], k >> 1), w2 = wword(g.t[2], k >> 1);
    return make_uint2(((k & 1) ? (w0 >> 16) : (w0 & 0xFFFFu)) + (1u << kW0Shift),
                      __byte_perm(w1, w2, (k & 1) ? 0x7632u : 0x5410u));
}

// Bucket table over [0, 2^32) for the segment's K sorted keys: clear, scatter
// the keys (count in .y, key in .x), then an exclusive prefix over the bucket
// counts, 32 buckets per step.  Entry = {key, first bin * 256} for a bucket
// with one key, {0xFFFFFFFF, first bin * 256} for none, {0xFFFFFFFF, 1} (odd:
// the producer searches the keys) for two or more.
__device__ __forceinline__ void wide_build_lut(const WideSmem &S, int K) {
    const uint32_t lane = lane_id();
    for (int b = (int)lane; b < kWideBuckets; b += 32) S.lut[b] = make_uint2(0xFFFFFFFFu, 0u);
    __syncwarp();
    for (int j = (int)lane; j < K; j += 32) {
        const uint32_t key = S.keys[j];
        const uint32_t b = key >> kWideShift;
        atomicAdd(&S.lut[b].y, 1u);
        atomicExch(&S.lut[b].x, key);   // meaningful only when the bucket holds exactly one key
    }
    __syncwarp();
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t run = 0u;
#pragma unroll 4
    for (int c = 0; c < kWideBuckets / 32; ++c) {
        const int b = c * 32 + (int)lane;
        const uint2 e = S.lut[b];
        const uint32_t cnt = e.y;
        uint32_t excl, total;
        if (__any_sync(0xFFFFFFFFu, cnt >= 4u)) {
            uint32_t x = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, d);
                if ((int)lane >= d) x += y;
            }
            excl = x - cnt;
            total = __shfl_sync(0xFFFFFFFFu, x, 31);
        } else {
            const uint32_t b0 = __ballot_sync(0xFFFFFFFFu, cnt & 1u), b1 = __ballot_sync(0xFFFFFFFFu, cnt & 2u);
            excl = __popc(b0 & lt) + 2u * __popc(b1 & lt);
            total = __popc(b0) + 2u * __popc(b1);
        }
        S.lut[b] = cnt >= 2u ? make_uint2(0xFFFFFFFFu, 1u)
                             : make_uint2(cnt == 1u ? e.x : 0xFFFFFFFFu, (run + excl) * 256u);
        run += total;
    }
    __syncwarp();
}

// 64-bit add of a packed row (or of one request's exact fields) into the spill scratch
__device__ __forceinline__ void wide_spill_add(unsigned long long *scr, int bin, uint32_t cnt, uint32_t t0,
                                               uint32_t t1, uint32_t t2) {
    unsigned long long *r = scr + (size_t)bin * 4;
    if (cnt) atomicAdd(&r[0], (unsigned long long)cnt);
    if (t0) atomicAdd(&r[1], (unsigned long long)t0);
    if (t1) atomicAdd(&r[2], (unsigned long long)t1);
    if (t2) atomicAdd(&r[3], (unsigned long long)t2);
}

// the eight histogram rows (c0 = the consumer lane's slot) of a group's draws;
// draws in buckets holding several keys take the exact bin by binary search
__device__ __forceinline__ void wide_rows(const SimArgs &a, const WideSmem &S, const U8x &w, uint32_t c0,
                                          uint32_t c1, int P, U8x &row) {
    uint32_t odd = 0u;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint2 e = lds64(S.lut_s + ((w.v[k] >> kWideShift) << 3));
        row.v[k] = e.y + (w.v[k] > e.x ? c1 : c0);
        odd |= row.v[k];
    }
    if (odd & 1u) {   // rare: draws in multi-key buckets (odd row), exact bin by binary search
        uint32_t m = 0u;
#pragma unroll
        for (int k = 0; k < 8; ++k) m |= (row.v[k] & 1u) << k;
#pragma unroll 1
        while (m) {
            const int k = __ffs(m) - 1;
            m &= m - 1u;
            set8(row, k, c0 + (uint32_t)find_bin(S.keys, P, sel8(w, k)) * 256u);
        }
    }
}

// One ring stage: wait until it is free, start the TMA bulk copies of the
// iteration's token planes (lane 0; the full barrier expects their bytes),
// write the rows, then the second arrival on the full barrier.
__device__ __forceinline__ void wide_put(const SimArgs &a, const WideSmem &S, const U8x &row, int64_t gi,
                                         int64_t ge, uint32_t &cnt) {
    const uint32_t lane = lane_id();
    const uint32_t s = cnt % kWideStages, ph = (cnt / kWideStages) & 1u;
    const uint32_t st = S.ring_s + s * (uint32_t)kWideStageBytes;
    const uint32_t full = S.bar_s + 8u * s;
    mbar_wait(S.bar_s + 8u * (kWideStages + s), ph ^ 1u);   // stage free
    if (lane == 0) {
        const int64_t ng = min((int64_t)32, ge - gi);        // whole groups of this iteration
        const uint32_t bytes = (uint32_t)ng * 16u;
        mbar_arrive_expect_tx(full, 3u * bytes);
#pragma unroll
        for (int q = 0; q < 3; ++q)
            bulk_g2s(st + 1024u + 512u * q, a.tokens + (size_t)q * a.pitch + (size_t)gi * 8, bytes, full);
        const int64_t gp = gi + 32 * (int64_t)(kWideStages + SPROUT_WIDE_L2PF);   // further ahead into L2
        if (gp < ge) {
            const uint32_t pb = (uint32_t)min((int64_t)32, ge - gp) * 16u;
#pragma unroll
            for (int q = 0; q < 3; ++q) bulk_prefetch_l2(a.tokens + (size_t)q * a.pitch + (size_t)gp * 8, pb);
        }
    }
    if (gi + (int64_t)lane < ge) {
        sts128(st + lane * 16u, make_uint4(row.v[0], row.v[1], row.v[2], row.v[3]));
        sts128(st + 512u + lane * 16u, make_uint4(row.v[4], row.v[5], row.v[6], row.v[7]));
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(full);
    ++cnt;
}

// Producer: per warp iteration i, lane l's group v = gf + l + 32i: its two
// Philox calls, the eight rows (c0 = the consumer lane's slot), the exact
// bin for draws in multi-key buckets, and the rows into ring stage cnt % S.
// Two iterations at a time (four independent Philox chains in flight).
__device__ __forceinline__ void wide_produce(const SimArgs &a, const WideSmem &S, int64_t gf, int64_t ge, int P,
                                             uint32_t &cnt) {
    const uint32_t lane = lane_id();
    const uint32_t n_iter = ge > gf ? (uint32_t)((ge - gf + 31) >> 5) : 0u;
    const uint32_t c0 = S.hist_s + lane * 8u, c1 = c0 + 256u;
    const int64_t v0 = gf + lane;
    uint32_t lo = (uint32_t)((a.first_request >> 2) + 2u * (uint64_t)v0);
    if (lane < 3u * (kWideStages + SPROUT_WIDE_L2PF)) {   // the first iterations' planes into L2
        const int64_t gp = gf + 32 * (int64_t)(lane / 3u);
        if (gp < ge)
            bulk_prefetch_l2(a.tokens + (size_t)(lane % 3u) * a.pitch + (size_t)gp * 8,
                             (uint32_t)min((int64_t)32, ge - gp) * 16u);
    }
    uint32_t i = 0;
#pragma unroll 1
    for (; i + 2 <= n_iter; i += 2, lo += 128u) {
        U8x w0, w1, r0, r1;
#if SPROUT_WIDE_AB_NOPHILOX   // A/B timing only (wrong results): a cheap hash instead of Philox
#pragma unroll
        for (int k = 0; k < 8; ++k) { w0.v[k] = (lo + k) * 0x9E3779B9u; w1.v[k] = (lo + 64u + k) * 0x9E3779B9u; }
#else
        const Philox4 d0 = philox_lo(lo, a), d1 = philox_lo(lo + 1u, a);
        const Philox4 d2 = philox_lo(lo + 64u, a), d3 = philox_lo(lo + 65u, a);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            w0.v[k] = d0.v[k]; w0.v[4 + k] = d1.v[k];
            w1.v[k] = d2.v[k]; w1.v[4 + k] = d3.v[k];
        }
#endif
        wide_rows(a, S, w0, c0, c1, P, r0);
        wide_rows(a, S, w1, c0, c1, P, r1);
        wide_put(a, S, r0, gf + 32 * (int64_t)i, ge, cnt);
        wide_put(a, S, r1, gf + 32 * (int64_t)(i + 1), ge, cnt);
    }
    if (i < n_iter) {
        U8x w0, r0;
        const Philox4 d0 = philox_lo(lo, a), d1 = philox_lo(lo + 1u, a);
#pragma unroll
        for (int k = 0; k < 4; ++k) { w0.v[k] = d0.v[k]; w0.v[4 + k] = d1.v[k]; }
        wide_rows(a, S, w0, c0, c1, P, r0);
        wide_put(a, S, r0, gf + 32 * (int64_t)i, ge, cnt);
    }
}

// Consumer rare work of a group (inline, rolled): big -- some token >= 4096,
// so a 16-bit field may have wrapped: the group's eight increments are
// reverted (exact: 32-bit word arithmetic is modular) and its requests added
// exactly into the 64-bit scratch; then rows with a guard bit set spill.
__device__ __forceinline__ void wide_rare(const WTok &g, const U8x &rows, uint32_t big, uint32_t c0,
                                          unsigned long long *scr, uint32_t &spilled) {
    if (big) {
#pragma unroll 1
        for (int k = 0; k < 8; ++k) {
            const uint32_t r = sel8(rows, k);
            const uint2 inc = wide_inc(g, k);
            uint2 A = lds64(r);
            A.x -= inc.x;
            A.y -= inc.y;
            sts64(r, A);
        }
#pragma unroll 1
        for (int k = 0; k < 8; ++k) {
            const uint32_t w0 = wword(g.t[0], k >> 1), w1 = wword(g.t[1], k >> 1), w2 = wword(g.t[2], k >> 1);
            const int sh = (k & 1) * 16;
            wide_spill_add(scr, (int)((sel8(rows, k) - c0) >> 8), 1u, (w0 >> sh) & 0xFFFFu, (w1 >> sh) & 0xFFFFu,
                           (w2 >> sh) & 0xFFFFu);
        }
        spilled = 1u;
        return;
    }
#pragma unroll 1
    for (int k = 0; k < 8; ++k) {
        const uint32_t r = sel8(rows, k);
        const uint2 A = lds64(r);
        if ((A.x & kGuard0) | (A.y & kGuard)) {
            wide_spill_add(scr, (int)((r - c0) >> 8), A.x >> kW0Shift, A.x & kW0Low, A.y & 0xFFFFu, A.y >> 16);
            sts64(r, make_uint2(0u, 0u));
            spilled = 1u;
        }
    }
}

// Consumer: lane l's groups gf + l + 32i; per iteration it waits for the
// stage (rows written, token planes landed), reads its eight rows and its
// three 16-byte token words, releases the stage, then does the serial
// read-modify-writes and one test for the rare work.
__device__ __forceinline__ void wide_consume(const SimArgs &a, const WideSmem &S, int64_t gf, int64_t ge,
                                             unsigned long long *scr, uint32_t &spilled, uint32_t &cnt) {
    const uint32_t lane = lane_id();
    const uint32_t n_iter = ge > gf ? (uint32_t)((ge - gf + 31) >> 5) : 0u;
    const int64_t v0 = gf + lane;
    const uint32_t n_mine = v0 < ge ? (uint32_t)((ge - v0 + 31) >> 5) : 0u;
    const uint32_t c0 = S.hist_s + lane * 8u;
#pragma unroll 1
    for (uint32_t i = 0; i < n_iter; ++i) {
        const uint32_t s = cnt % kWideStages, ph = (cnt / kWideStages) & 1u;
        const uint32_t st = S.ring_s + s * (uint32_t)kWideStageBytes + lane * 16u;
        mbar_wait(S.bar_s + 8u * s, ph);   // rows written and token planes landed
        U8x row;
        WTok g;
        {
            const uint4 r0 = lds128(st), r1 = lds128(st + 512u);
            row.v[0] = r0.x; row.v[1] = r0.y; row.v[2] = r0.z; row.v[3] = r0.w;
            row.v[4] = r1.x; row.v[5] = r1.y; row.v[6] = r1.z; row.v[7] = r1.w;
#pragma unroll
            for (int q = 0; q < 3; ++q) g.t[q] = lds128(st + 1024u + 512u * q);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(S.bar_s + 8u * (kWideStages + s));   // stage free again
        ++cnt;
        if (i < n_mine) {
            uint32_t acc0 = 0u, acc1 = 0u;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint2 inc = wide_inc(g, k);
                uint2 A = lds64(row.v[k]);
                A.x += inc.x;
                A.y += inc.y;
                sts64(row.v[k], A);
                acc0 |= A.x;
                acc1 |= A.y;
            }
            const uint32_t big = (g.t[0].x | g.t[0].y | g.t[0].z | g.t[0].w | g.t[1].x | g.t[1].y | g.t[1].z |
                                  g.t[1].w | g.t[2].x | g.t[2].y | g.t[2].z | g.t[2].w) & kBigTok;
            if ((acc0 & kGuard0) | (acc1 & kGuard) | big) wide_rare(g, row, big, c0, scr, spilled);
        }
    }
}

// the requests outside the segment's whole groups (at most 7 at each end),
// one per lane, added exactly into the spill scratch
__device__ __forceinline__ void wide_ends(const SimArgs &a, const WideSmem &S, int64_t s0, int64_t s1, int P,
                                          unsigned long long *scr, uint32_t &spilled) {
    const uint32_t lane = lane_id();
    const int64_t h_end = min(s1, (s0 + 7) & ~(int64_t)7);
    const int64_t t_beg = max(h_end, s1 & ~(int64_t)7);
    int64_t r = -1;
    if ((int64_t)lane < h_end - s0) r = s0 + lane;
    else if (lane >= 8 && (int64_t)(lane - 8) < s1 - t_beg) r = t_beg + (lane - 8);
    if (r < 0) return;
    const uint64_t gidx = a.first_request + (uint64_t)r;
    const Philox4 d = philox_lo((uint32_t)(gidx >> 2), a);
    const uint32_t k3 = (uint32_t)(gidx & 3u);
    const uint32_t w = k3 == 0 ? d.v[0] : k3 == 1 ? d.v[1] : k3 == 2 ? d.v[2] : d.v[3];
    wide_spill_add(scr, find_bin(S.keys, P, w), 1u, a.tokens[r], a.tokens[(size_t)a.pitch + r],
                   a.tokens[2 * (size_t)a.pitch + r]);
    spilled = 1u;
}

// lane histograms (+ the spill scratch) -> 64-bit rows 0..K of the table
// space, rows K+1 and the pinned row cleared, then the exclusive prefix over
// bins 0..K+1 per field (the layout cell_epilogue / write_seg_stats read)
__device__ __forceinline__ void wide_readout(const SimArgs &a, const WideSmem &S, int K, bool spilled,
                                             unsigned long long *scr) {
    const uint32_t lane = lane_id();
    unsigned long long *wide = reinterpret_cast<unsigned long long *>(S.lut);
    for (int bn = (int)lane; bn <= K; bn += 32) {
        uint2 *row = S.hist + (size_t)bn * 32;
        uint32_t sv[4] = {0u, 0u, 0u, 0u};
#pragma unroll 8
        for (int q = 0; q < 32; ++q) {
            const int idx = (q + (int)lane) & 31;   // rotated: conflict-free
            const uint2 val = row[idx];
            row[idx] = make_uint2(0u, 0u);
            sv[0] += val.x >> kW0Shift;
            sv[1] += val.x & kW0Low;
            sv[2] += val.y & 0xFFFFu;
            sv[3] += val.y >> 16;
        }
        unsigned long long f[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) f[j] = sv[j];
        if (spilled) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                f[j] += scr[(size_t)bn * 4 + j];
                scr[(size_t)bn * 4 + j] = 0ull;
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) wide[(size_t)bn * 4 + j] = f[j];
    }
    if (lane < 4) {
        wide[(size_t)(K + 1) * 4 + lane] = 0ull;
        wide[(size_t)(a.nb - 1) * 4 + lane] = 0ull;
    }
    __syncwarp();
    if (lane < 4) {
        unsigned long long run = 0ull;
        for (int bn = 0; bn <= K + 1; ++bn) {
            unsigned long long *pt = &wide[(size_t)bn * 4 + lane];
            const unsigned long long v2 = *pt;
            *pt = run;
            run += v2;
        }
    }
    __syncwarp();
}

__global__ void __launch_bounds__(64 * kWideTeams, 1) trace_wide_kernel(const __grid_constant__ SimArgs a) {
    constexpr int N = 3;
    constexpr int kExit = -9;
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ CostConst cost;
    const int warp = threadIdx.x >> 5;
    const int team = warp >> 1;
    const bool producer = (warp & 1) != 0;
    const uint32_t lane = lane_id();
    const int X = a.X, nb = a.nb, kcap = a.kcap;
    WideSmem S;
    {
        uint8_t *base = smem + (size_t)team * a.warp_smem;
        S.bar_s = smem_u32(base);
        S.seg = reinterpret_cast<WideSeg *>(base + 16 * kWideStages);
        S.ring_s = smem_u32(base + kWideCtl);
        uint8_t *h = base + kWideCtl + (size_t)kWideStages * kWideStageBytes;
        S.hist = reinterpret_cast<uint2 *>(h);
        S.lut = reinterpret_cast<uint2 *>(h + (size_t)(kcap + 1) * 256);
        S.keys = reinterpret_cast<uint32_t *>(h + (size_t)(kcap + 1) * 256 + (size_t)kWideBuckets * 8);
        S.hist_s = smem_u32(S.hist);
        S.lut_s = smem_u32(S.lut);
    }
    for (int i = threadIdx.x; i < (int)(sizeof(CostConst) / 8); i += blockDim.x)
        reinterpret_cast<double *>(&cost)[i] = reinterpret_cast<const double *>(&a.cost)[i];
    if (!producer) {
        for (int i = lane; i < (kcap + 1) * 32; i += 32) S.hist[i] = make_uint2(0u, 0u);
        if (lane < 2 * kWideStages) mbar_init(S.bar_s + 8u * lane, lane < kWideStages ? 2u : 1u);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");   // visible to the TMA unit
    }
    __syncthreads();
    uint32_t cnt = 0u;   // ring iterations so far (both warps of a team count the same)

    if (producer) {
        for (;;) {
            team_sync(team);
            const WideSeg sg = *S.seg;
            if (sg.meta == kExit) break;
            if (sg.meta >= 1) wide_produce(a, S, (sg.s0 + 7) >> 3, sg.s1 >> 3, sg.P, cnt);
        }
        return;
    }

    // consumer
    WarpSmem W;   // the view the shared epilogue and the K = 0 / slow paths use
    W.hist = S.hist;
    W.wide = reinterpret_cast<unsigned long long *>(S.lut);
    W.lut = S.lut;
    W.keys = S.keys;
    unsigned long long *scr = a.wide_scratch + ((size_t)blockIdx.x * kWideTeams + team) * (size_t)(kcap + 1) * 4;
    for (int i = lane; i < (kcap + 1) * 4; i += 32) scr[i] = 0ull;
    uint32_t err = 0u;
    constexpr int kKeyRegs = 4;   // keys prefetched per lane (kcap <= 128), else read at use
    struct SegPre {
        int64_t sl, s0, s1;
        int meta;
        double k0;
        uint32_t key[kKeyRegs];
        SegCells sc;
    };
    const bool pre_cells = X <= 64;
    auto load_pre = [&](int64_t sl) {
        SegPre p;
        p.sl = sl;
        p.meta = -3;
        p.s0 = p.s1 = 0;
        p.k0 = 0.0;
#pragma unroll
        for (int t = 0; t < kKeyRegs; ++t) p.key[t] = 0xFFFFFFFFu;
        p.sc.st[0] = p.sc.st[1] = 0xFFu;
        p.sc.bw[0] = p.sc.bw[1] = 0u;
        if (sl < a.n_segments) {
            p.meta = a.seg_meta[sl];
            p.s0 = a.seg_offsets[sl];
            p.s1 = a.seg_offsets[sl + 1];
            p.k0 = a.k0[a.first_segment + sl];
            if (pre_cells) {
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    const int j = (int)lane + 32 * t;
                    if (j < X) {
                        const int64_t cell = sl * X + j;
                        p.sc.st[t] = a.cell_status[cell];
                        p.sc.bw[t] = *reinterpret_cast<const uint32_t *>(a.seg_bnd + cell * 2);
                    }
                }
            }
            if (kcap <= 32 * kKeyRegs) {
#pragma unroll
                for (int t = 0; t < kKeyRegs; ++t) {
                    const int i = (int)lane + 32 * t;
                    if (i < kcap) p.key[t] = a.seg_keys[sl * kcap + i];
                }
            }
        }
        return p;
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
    auto zero_wide = [&](int rows) {   // 64-bit rows 0..rows-1 and the pinned row
        for (int i = lane; i < rows * (N + 1); i += 32) W.wide[i] = 0ull;
        if (lane < N + 1) W.wide[(size_t)(nb - 1) * (N + 1) + lane] = 0ull;
        __syncwarp();
    };
    SegPre cur = load_pre(next_segment());
    for (;;) {
        const int64_t sl = cur.sl;
        if (sl >= a.n_segments) {
            if (lane == 0) S.seg->meta = kExit;
            team_sync(team);
            break;
        }
        const SegPre nxt = load_pre(next_segment());
        const int64_t s = a.first_segment + sl;
        const int meta = cur.meta;
        const double *qrow =
            a.q + (a.profile_per_interval ? s : (s < 0xFFFFFFFFll ? (int64_t)a.div_t.div((uint32_t)s) : s / a.T)) * N;
        const double kp = cur.k0 * a.pue;
        const int64_t s0 = cur.s0, s1 = cur.s1;
        const int K = meta;
        int P = 1;
        while (P < K + 1) P <<= 1;
        if (meta >= 0) {
            if (kcap <= 32 * kKeyRegs) {
#pragma unroll
                for (int t = 0; t < kKeyRegs; ++t) {
                    const int i = (int)lane + 32 * t;
                    if (i < P) S.keys[i] = i < K ? cur.key[t] : 0xFFFFFFFFu;
                }
            } else {
                for (int i = lane; i < P; i += 32) S.keys[i] = i < K ? a.seg_keys[sl * kcap + i] : 0xFFFFFFFFu;
            }
            __syncwarp();
            if (K >= 1) wide_build_lut(S, K);
        }
        if (lane == 0) {
            S.seg->sl = sl; S.seg->s0 = s0; S.seg->s1 = s1;
            S.seg->meta = meta; S.seg->P = P;
        }
        team_sync(team);   // the producer may start on this segment
        if (meta == -2) {   // invalid offsets: segment skipped, outputs zero
            err |= SPROUT_TRACE_BAD_OFFSETS;
            for (int j = lane; j < X; j += 32) zero_cell(a, sl * X + j, N);
            if (lane == 0) { a.seg_count[sl] = 0ull; a.seg_pinned[sl] = 0ull; }
            if (lane < N) a.seg_tok[sl * N + lane] = 0ull;
            if (lane < 4) a.seg_base[sl * 4 + lane] = 0.0;
            cur = nxt;
            continue;
        }
        if (meta == -1) {
            zero_wide(2);
            slow_segment<N, false>(a, W, sl, s0, s1, err);
            cell_epilogue<N>(a, W, sl, 0, kp, qrow, false, cost, false, cur.sc);
            __syncwarp();
            write_seg_stats<N>(a, W, sl, kp, qrow[0], 0, 1, false, cost);
            __syncwarp();
            cur = nxt;
            continue;
        }
        if (K == 0) {
            zero_wide(2);
            stream_segment_k0<N>(a, W, s0, s1);
            __syncwarp();
            if (lane < N + 1) {   // exclusive prefix over bins 0..1
                const unsigned long long v0 = W.wide[lane];
                W.wide[lane] = 0ull;
                W.wide[(N + 1) + lane] = v0;
            }
            __syncwarp();
        } else {
            uint32_t spilled = 0u;
            wide_ends(a, S, s0, s1, P, scr, spilled);
            wide_consume(a, S, (s0 + 7) >> 3, s1 >> 3, scr, spilled, cnt);
            __syncwarp();
            __threadfence_block();
            const bool any_spill = __any_sync(0xFFFFFFFFu, spilled != 0u);
            wide_readout(a, S, K, any_spill, scr);
        }
        // the next segment's first groups into L2 while this one's epilogue runs
        if (nxt.sl < a.n_segments && nxt.meta >= -1 && nxt.s1 > nxt.s0) {
            const int64_t g0 = nxt.s0 >> 3, g1 = (nxt.s1 - 1) >> 3;
            if (nxt.s1 - nxt.s0 < 2048) {
                const int64_t v = (lane < 16) ? g0 + lane : g1 - (int64_t)(lane - 16);
                if (v >= g0 && v <= g1) {
#pragma unroll
                    for (int i = 0; i < N; ++i)
                        prefetch_l2(reinterpret_cast<const uint4 *>(a.tokens + (size_t)i * a.pitch) + v);
                }
            } else {
#pragma unroll 1
                for (int it = 0; it <= SPROUT_WIDE_PREFETCH; ++it) {
                    const int64_t v = it < SPROUT_WIDE_PREFETCH ? g0 + lane + 32 * it : g1;
#pragma unroll
                    for (int i = 0; i < N; ++i)
                        prefetch_l2(reinterpret_cast<const uint4 *>(a.tokens + (size_t)i * a.pitch) + v);
                }
            }
        }
        cell_epilogue<N>(a, W, sl, K, kp, qrow, true, cost, pre_cells, cur.sc);
        __syncwarp();
        write_seg_stats<N>(a, W, sl, kp, qrow[0], K + 1, nb - 1, true, cost);
        __syncwarp();
        cur = nxt;
    }
    err = __reduce_or_sync(0xFFFFFFFFu, err);
    if (lane == 0 && err) atomicOr(a.trace_status, err);
}

// ---------------------------------------------------------------------------
// verify mode (levels_out): the level of every request in every cell of its
// segment, from the same draw, the same breakpoint keys and the same
// per-cell bin boundaries the streaming kernel aggregates over (or, for
// slow segments, directly from the thresholds).  One warp per segment.
template <int N>
__global__ void __launch_bounds__(256) levels_kernel(const __grid_constant__ SimArgs a) {
    const uint32_t lane = lane_id();
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t sl = gw; sl < a.n_segments; sl += nw) {
        const int meta = a.seg_meta[sl];
        if (meta == -2) continue;
        const int64_t s0 = a.seg_offsets[sl], s1 = a.seg_offsets[sl + 1];
        for (int64_t r = s0 + lane; r < s1; r += 32) {
            const uint64_t gidx = a.first_request + (uint64_t)r;
            const uint64_t blk = gidx >> 2;
            const Philox4 d = philox4x32_10((uint32_t)blk, (uint32_t)(blk >> 32), 0u, 0u, (uint32_t)a.seed,
                                            (uint32_t)(a.seed >> 32));
            const uint32_t w = d.v[gidx & 3u];
            bool pinned = false, bad = false;
            if (a.flags) {
                const uint8_t f = a.flags[r];
                pinned = f & 1u;
                bad = ((f >> 1) & 3) >= a.NC;
            }
            int bin = 0;
            if (meta > 0 && a.bins_ready) {
                bin = a.bins_out[r];   // the bin the streaming kernel found (pinned requests: unused)
            } else if (meta >= 0) {
                const uint32_t *keys = a.seg_keys + sl * a.kcap;
                for (int k = 0; k < meta; ++k) bin += (keys[k] < w) ? 1 : 0;
            }
            for (int j = 0; j < a.X; ++j) {
                const int64_t cell = sl * a.X + j;
                uint8_t L = 0xFF;
                if (!bad && a.cell_status[cell] == SPROUT_CELL_OK) {
                    L = 0;
                    if (!pinned) {
                        if (meta >= 0) {
                            for (int l = 1; l < N; ++l)
                                if ((int)a.seg_bnd[cell * (N - 1) + (l - 1)] <= bin) L = (uint8_t)l;
                        } else {
                            int c = 0;
                            for (int i = 0; i + 1 < N; ++i) c += (w >= a.threshold[cell * (N - 1) + i]) ? 1 : 0;
                            const int ml = a.max_level[cell];
                            L = (uint8_t)(c < ml ? c : ml);
                        }
                    }
                }
                a.levels_out[(size_t)j * a.pitch + r] = L;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// host side

// breakpoint slots per segment in the workspace: the fast path's nominal
// capacity (independent of the class count and of the shared-memory fit)
static int nominal_kcap(int n, int X) {
    const long M = (long)X * (n - 1);
    return (n == 1) ? 0 : (int)((M < (long)X + 1) ? M : (long)X + 1);
}

bool make_sim_plan(int n, int X, int NC, SimPlan *plan, int max_keys) {
    SimPlan p{};
    p.n = n; p.X = X; p.NC = NC;
    p.nw = 2 * (((n + 2) / 2 + 1) / 2);   // words allocated per entry: whole 64-bit pairs
    const long M = (long)X * (n - 1);
    int kcap = nominal_kcap(n, X);
    if (max_keys > 0 && max_keys < kcap) kcap = max_keys;   // caller's bound (e.g. a static grid sweep)
    p.sort_cap = 0;
    if (M > 0) {
        long c = 1;
        while (c < M) c <<= 1;
        p.sort_cap = (int)(c < 32 ? 32 : c);
    }
    if (p.sort_cap > 4096) {              // too many thresholds to merge per warp: generic path
        kcap = -1;                        // (prep then only marks segments generic: no sort buffer)
        p.sort_cap = 0;
    }
    auto per_warp = [&](int kc, int *nb_out, int *kp_out) {
        const int kk = kc < 0 ? 0 : kc;
        const int nb = kk + 3;
        int kp = 1;
        while (kp < kk + 1) kp <<= 1;
        const size_t entries = (size_t)NC * nb + 1;
        const bool lut = kc >= kLutMinKeys && kc <= kLutMaxKeys;
        size_t bytes = ((entries * (n + 1) * 8 + 15) & ~(size_t)15) + entries * p.nw * 32 * 4 + (size_t)kp * 4 +
                       (lut ? (size_t)kLutBuckets * 8 : 0);
        *nb_out = nb;
        *kp_out = kp;
        return (bytes + 15) & ~(size_t)15;
    };
    const size_t smem_cap = 227 * 1024 - 2048;   // leave room for the static cost table
    int nb, kp;
    size_t bytes = per_warp(kcap, &nb, &kp);
    if (kcap >= 0 && bytes > smem_cap) {
        kcap = -1;
        p.sort_cap = 0;
        bytes = per_warp(kcap, &nb, &kp);
    }
    p.kcap = kcap;
    p.lut = (kcap >= kLutMinKeys && kcap <= kLutMaxKeys) ? 1 : 0;
    p.nb = nb;
    p.kp = kp;
    p.warp_smem = bytes;
    int wpc = (int)(smem_cap / bytes);
    if (wpc > kMaxTraceWarps) wpc = kMaxTraceWarps;
    if (wpc < 1) return false;
    p.warps_per_cta = wpc;
    *plan = p;
    return true;
}

// spill scratch of trace_wide_kernel (n = 3): [kWideMaxSMs * kWideTeams][kcap + 1][4] u64
static size_t wide_scratch_bytes(const SimPlan &p) {
    if (!SPROUT_ENABLE_WIDE || p.n != 3) return 0;
    const int kc = nominal_kcap(p.n, p.X);
    return ((size_t)kWideMaxSMs * kWideTeams * (size_t)(kc + 1) * 4 * 8 + 255) & ~(size_t)255;
}

size_t sim_workspace_bytes(const SimPlan &p, int64_t n_segments) {
    const int kc = nominal_kcap(p.n, p.X);
    size_t b = 256;                                             // queue
    b += ((size_t)n_segments * 4 + 255) & ~(size_t)255;         // seg_meta
    b += ((size_t)n_segments * kc * 4 + 255) & ~(size_t)255;   // seg_keys
    const size_t cells = (size_t)n_segments * p.X;
    b += (cells * (p.n > 1 ? p.n - 1 : 0) * 2 + 255) & ~(size_t)255;  // seg_bnd
    b += wide_scratch_bytes(p);
    return b;
}

// trace_wide_kernel applies: n = 3, one class, no flags plane, X > 1, a
// breakpoint bound that fits its table space, and a launch whose Philox
// blocks share one high counter word
static bool wide_applies(const SimArgs &a, const SimPlan &plan) {
    if (!SPROUT_ENABLE_WIDE || plan.n != 3 || a.flags || a.NC != 1 || a.X <= 1) return false;
    if (plan.kcap < 1 || plan.kcap > kWideMaxKeys) return false;
    if (a.n_requests > 0 && (a.first_request >> 34) != ((a.first_request + (uint64_t)a.n_requests - 1) >> 34))
        return false;
    int kp = 1;
    while (kp < plan.kcap + 1) kp <<= 1;
    return (size_t)kWideTeams * ((wide_team_bytes(plan.kcap, kp) + 15) & ~(size_t)15) <= (227 * 1024 - 2048);
}

static cudaError_t launch_trace_wide(SimArgs &a, const SimPlan &plan, cudaStream_t stream) {
    int kp = 1;
    while (kp < plan.kcap + 1) kp <<= 1;
    a.warp_smem = (wide_team_bytes(plan.kcap, kp) + 15) & ~(size_t)15;   // per team
    if ((size_t)kWideTeams * a.warp_smem > 227 * 1024 - 2048) return cudaErrorInvalidConfiguration;
    const int threads = kWideTeams * 64;
    const size_t smem = a.warp_smem * kWideTeams;
    cudaError_t e = cudaFuncSetAttribute(trace_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t grid = sms < kWideMaxSMs ? sms : kWideMaxSMs;   // one CTA per SM (the spill scratch covers them)
    const int64_t need = (a.n_segments + kWideTeams - 1) / kWideTeams;
    if (grid > need) grid = need > 0 ? need : 1;
    trace_wide_kernel<<<(unsigned)grid, threads, smem, stream>>>(a);
    return cudaGetLastError();
}

template <int N, bool FLAGS>
static cudaError_t launch_trace_t(SimArgs &a, const SimPlan &plan, cudaStream_t stream) {
    const int threads = plan.warps_per_cta * 32;
    const size_t smem = plan.warp_smem * plan.warps_per_cta;
    auto kern = a.bins_out ? trace_kernel<N, FLAGS, true> : trace_kernel<N, FLAGS, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    int64_t grid = (int64_t)sms * per_sm;
    const int64_t need = (a.n_segments + plan.warps_per_cta - 1) / plan.warps_per_cta;
    if (grid > need) grid = need > 0 ? need : 1;
    kern<<<(unsigned)grid, threads, smem, stream>>>(a);
    return cudaGetLastError();
}

template <int N>
static cudaError_t launch_n(SimArgs &a, const SimPlan &plan, cudaStream_t stream, int *launches) {
    const bool x1 = !kDisableX1 && trace_x1_supported(N, a.X, a.NC);
    // verify mode on the breakpoint-histogram kernel: it writes every request's bin
    // into row 0 of levels_out, and levels_kernel derives the levels from those bins
    a.bins_out = (a.levels_out && !x1 && !(N == 3 && a.wide) && plan.kcap <= 254) ? a.levels_out : nullptr;
    a.bins_ready = a.bins_out ? 1 : 0;
    cudaError_t e = x1 ? launch_trace_x1(a, stream)
                  : (N == 3 && a.wide) ? launch_trace_wide(a, plan, stream)
                  : a.flags ? launch_trace_t<N, true>(a, plan, stream) : launch_trace_t<N, false>(a, plan, stream);
    if (e != cudaSuccess) return e;
    ++*launches;
    if (a.levels_out && !x1) {   // (the one-cell kernels write their requests' levels themselves)
        int64_t blocks = (a.n_segments * 32 + 255) / 256;
        if (blocks > 148 * 32) blocks = 148 * 32;
        levels_kernel<N><<<(unsigned)blocks, 256, 0, stream>>>(a);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        ++*launches;
    }
    return cudaSuccess;
}

cudaError_t launch_simulate(SimArgs &a, const SimPlan &plan, void *ws, cudaStream_t stream, int *launches) {
    uint8_t *w = static_cast<uint8_t *>(ws);
    a.queue = reinterpret_cast<uint32_t *>(w);
    size_t off = 256;
    a.seg_meta = reinterpret_cast<int32_t *>(w + off);
    off += ((size_t)a.n_segments * 4 + 255) & ~(size_t)255;
    a.seg_keys = reinterpret_cast<uint32_t *>(w + off);
    const int kc = nominal_kcap(plan.n, plan.X);
    off += ((size_t)a.n_segments * kc * 4 + 255) & ~(size_t)255;
    a.seg_bnd = reinterpret_cast<uint16_t *>(w + off);
    off += ((size_t)a.n_segments * plan.X * (plan.n > 1 ? plan.n - 1 : 0) * 2 + 255) & ~(size_t)255;
    a.wide_scratch = reinterpret_cast<unsigned long long *>(w + off);
    a.kcap = plan.kcap;   // -1 (all slow) or the plan's bound <= kc (the seg_keys stride)
    a.nb = plan.nb;
    a.nw = plan.nw;
    a.kp = plan.kp;
    a.sort_cap = plan.sort_cap;
    a.warp_smem = plan.warp_smem;
    a.lut = plan.lut;
    a.div_nt = FastDiv((uint32_t)(plan.n > 1 ? plan.n - 1 : 1));
    a.div_t = FastDiv(a.T < (int64_t)0xFFFFFFFFll ? (uint32_t)a.T : 1u);
    {   // about 64 tickets per warp: one per segment for few long segments,
        // batches of up to 32 for many short ones
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int64_t warps = (int64_t)sms * plan.warps_per_cta;
        int64_t bsz = a.n_segments / (warps * 64);
        a.seg_batch = (int)(bsz < 1 ? 1 : (bsz > 8 ? 8 : bsz));
    }
    {
        uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32);
        for (int r = 0; r < 10; ++r) {
            a.rk0[r] = k0; a.rk1[r] = k1;
            k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
        }
        // philox_lo's launch constants for the counter high word H of the launch's blocks
        const uint32_t H = (uint32_t)(a.first_request >> 34);
        a.ph_a = H ^ a.rk0[0];
        const uint64_t B = (uint64_t)0xD2511F53u * a.ph_a;
        a.ph_blo = (uint32_t)B;
        a.ph_d = (uint32_t)(B >> 32) ^ a.rk1[1];
        a.ph_e = (uint32_t)B ^ a.rk1[2];
    }
    a.wide = wide_applies(a, plan) ? 1 : 0;

    // prep (also resets the queue and trace_status).  The one-cell kernels need no
    // breakpoints and check the offsets themselves: without verify mode they only
    // need the two counters reset
    if (!kDisableX1 && trace_x1_supported(plan.n, a.X, a.NC)) {
        cudaError_t e = cudaMemsetAsync(a.queue, 0, 4, stream);
        if (e == cudaSuccess) e = cudaMemsetAsync(a.trace_status, 0, 4, stream);
        if (e != cudaSuccess) return e;
        a.seg_meta = nullptr;
    } else {
        int64_t blocks = (a.n_segments + kPrepWarps - 1) / kPrepWarps;
        if (blocks > 148 * 32) blocks = 148 * 32;
        if (blocks < 1) blocks = 1;
        const int E = plan.sort_cap <= 32 ? 1 : plan.sort_cap <= 64 ? 2 : plan.sort_cap <= 128 ? 4 : 0;
        const int scap = E > 0 ? 32 * E : (plan.sort_cap > 0 ? plan.sort_cap : 1);
        const size_t smem = (size_t)kPrepWarps * 2 * scap * 4;
        auto kern = E == 1 ? prep_kernel<1> : E == 2 ? prep_kernel<2> : E == 4 ? prep_kernel<4> : prep_kernel<0>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        kern<<<(unsigned)blocks, 32 * kPrepWarps, smem, stream>>>(a);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        ++*launches;
    }
    if (a.n_segments == 0) return cudaSuccess;
    switch (a.n) {
        case 1: return launch_n<1>(a, plan, stream, launches);
        case 2: return launch_n<2>(a, plan, stream, launches);
        case 3: return launch_n<3>(a, plan, stream, launches);
        case 4: return launch_n<4>(a, plan, stream, launches);
        case 5: return launch_n<5>(a, plan, stream, launches);
        case 6: return launch_n<6>(a, plan, stream, launches);
        case 7: return launch_n<7>(a, plan, stream, launches);
        case 8: return launch_n<8>(a, plan, stream, launches);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace sprout
