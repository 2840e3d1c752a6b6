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
constexpr int kClPiece = 8192;   // requests per piece (a multiple of 4 * 32 * kClWarps)

template <int N, int NCM>   // NCM: class bound (1, or kMaxClasses)
__global__ void __launch_bounds__(kClThreads) closed_loop_kernel(const __grid_constant__ ClosedArgs a) {
    extern __shared__ uint32_t ring[];                      // [N][W] (class << 16 | tokens), then buf
    uint32_t *buf = ring + N * a.W;                         // [kClPiece] (level << 24 | class << 16 | tokens)
    __shared__ unsigned long long wsum[N][NCM][2];  // window: requests, tokens per (level, class)
    __shared__ unsigned long long csum[NCM][N][2];  // the interval's cell: requests, tokens
    __shared__ int head[N], size[N];
    __shared__ uint32_t thr_s[N > 1 ? N - 1 : 1];
    __shared__ int ml_s, ok_s;
    __shared__ int wcount[kClWarps][N];
    __shared__ uint32_t slots[kClWarps][NCM * N * 4];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int chain = blockIdx.x;
    const int r = a.r0 + chain / a.X, j = chain % a.X;   // this call's regions: [r0, r0 + R_local)
    const int W = a.W, NC = a.NC;
    const CostConst &cost = a.cost;
    if (tid < N) { head[tid] = 0; size[tid] = 0; }
    for (int i = tid; i < N * NCM * 2; i += kClThreads) (&wsum[0][0][0])[i] = 0ull;
    __syncthreads();
    uint32_t err = 0u;
    // the chain is latency-bound on its serial part, so everything an interval
    // reads from global memory besides its requests is loaded one interval
    // ahead: k0, the segment's offsets; the region's constants once
    double q_r[N], e_r[N], p_r[N];
#pragma unroll
    for (int L = 0; L < N; ++L) {
        q_r[L] = a.q[(int64_t)r * N + L];
        e_r[L] = a.e[(int64_t)r * N + L];
        p_r[L] = a.p[(int64_t)r * N + L];
    }
    const double kmin_r = a.kmin[r], kmax_r = a.kmax[r], xi_j = a.xi[j];
    const int64_t sl_first = (int64_t)r * a.T - a.first_segment;
    double k0_nxt = a.k0[(int64_t)r * a.T];
    int64_t off_nxt0 = a.seg_offsets[sl_first], off_nxt1 = a.seg_offsets[sl_first + 1];
    for (int64_t t = 0; t < a.T; ++t) {
        const int64_t s = (int64_t)r * a.T + t;                  // global segment (k0, profiles)
        const int64_t sl = s - a.first_segment;                  // local segment (offsets, outputs)
        const int64_t cell = sl * a.X + j;
        const double k0_s = k0_nxt;
        const int64_t s0 = off_nxt0, s1 = off_nxt1;
        if (t + 1 < a.T) {
            k0_nxt = a.k0[s + 1];
            off_nxt0 = s1;
            off_nxt1 = a.seg_offsets[sl + 2];
        }
        if (tid == 0) {
            double e[N], p[N], q[N];
#pragma unroll
            for (int L = 0; L < N; ++L) {
                q[L] = q_r[L];
                unsigned long long m = 0;
                for (int c = 0; c < NC; ++c) m += wsum[L][c][0];
                if (m == 0) {
                    e[L] = e_r[L];
                    p[L] = p_r[L];
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
            lp_cell<N>(k0_s, kmin_r, kmax_r, xi_j, e, p, q, a.k1, a.pue, 0, 0, j, o);
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
        for (int i = tid; i < NCM * N * 2; i += kClThreads) (&csum[0][0][0])[i] = 0ull;
        __syncthreads();
        const bool cell_ok = ok_s;
        uint32_t T[N > 1 ? N - 1 : 1];
#pragma unroll
        for (int i = 0; i + 1 < N; ++i) T[i] = thr_s[i];
        const int ml = ml_s;
        uint32_t cc[NCM][N], ct[NCM][N];
#pragma unroll
        for (int c = 0; c < NCM; ++c)
#pragma unroll
            for (int L = 0; L < N; ++L) { cc[c][L] = 0u; ct[c][L] = 0u; }
        if (cell_ok) {
            // Pieces of up to kClPiece requests, aligned on global quads (4 requests per Philox
            // call).  Pass A: warp w takes a contiguous run of the piece's quads, 128 requests per
            // step (lane l draws quad l of the step and hands the words out by shuffles), selects
            // every request's level, accumulates the cell and stores (level, class, tokens) in
            // shared memory, counting its level-L requests.  One barrier; then every warp knows
            // how many level-L requests precede its run (request order), and pass B re-walks the
            // run to write the last W of each level into the ring.
            const uint64_t gs0 = a.first_request + (uint64_t)s0, gs1 = a.first_request + (uint64_t)s1;
            const uint64_t q0 = gs0 >> 2, q1 = (gs1 + 3) >> 2;
            for (uint64_t pq = q0; pq < q1; pq += kClPiece / 4) {
                const uint64_t pq1 = min(q1, pq + kClPiece / 4);
                const uint64_t nq = pq1 - pq;
                const uint64_t per_w = ((nq + kClWarps * 32 - 1) / (kClWarps * 32)) * 32;   // quads per warp
                const uint64_t wq0 = min(pq1, pq + per_w * warp), wq1 = min(pq1, wq0 + per_w);
                int cntL[N];
                int dn[N][NCM], dk[N][NCM];   // this lane's window deltas in the piece
#pragma unroll
                for (int L = 0; L < N; ++L) {
                    cntL[L] = 0;
#pragma unroll
                    for (int c = 0; c < NCM; ++c) { dn[L][c] = 0; dk[L][c] = 0; }
                }
                for (uint64_t qb = wq0; qb < wq1; qb += 32) {
                    // the block's tokens at every level and its flags are loaded first (independent,
                    // coalesced loads in flight together; the level only selects among them)
                    uint32_t tk4[4][N], fb4[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint64_t g = qb * 4 + 32 * k + lane;
                        const bool ld = g >= gs0 && g < gs1;
                        const int64_t rq = (int64_t)(g - a.first_request);
#pragma unroll
                        for (int L = 0; L < N; ++L) tk4[k][L] = ld ? (uint32_t)__ldcs(a.tokens + (size_t)L * a.pitch + rq) : 0u;
                        fb4[k] = (ld && a.flags) ? (uint32_t)__ldcs(a.flags + rq) : 0u;
                    }
                    const uint64_t myq = qb + lane;
                    Philox4 d = philox4x32_10_rk((uint32_t)myq, (uint32_t)(myq >> 32), 0u, 0u, a.rk0, a.rk1);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int src = 8 * k + (lane >> 2);
                        const uint32_t v0 = __shfl_sync(0xFFFFFFFFu, d.v[0], src);
                        const uint32_t v1 = __shfl_sync(0xFFFFFFFFu, d.v[1], src);
                        const uint32_t v2 = __shfl_sync(0xFFFFFFFFu, d.v[2], src);
                        const uint32_t v3 = __shfl_sync(0xFFFFFFFFu, d.v[3], src);
                        const uint32_t sel = lane & 3u;
                        const uint32_t w = sel == 0 ? v0 : sel == 1 ? v1 : sel == 2 ? v2 : v3;
                        const uint64_t g = qb * 4 + 32 * k + lane;
                        const bool qin = qb + (uint64_t)(8 * k + (lane >> 2)) < wq1;   // quad of this warp
                        const bool inr = qin && g >= gs0 && g < gs1;
                        const int64_t rq = (int64_t)(g - a.first_request);
                        int lev = -1;
                        uint32_t cls = 0u, tl = 0u;
                        if (inr) {
                            const uint32_t pin = fb4[k] & 1u;
                            cls = (fb4[k] >> 1) & 3u;
                            if (cls >= (uint32_t)NC) {
                                err |= SPROUT_TRACE_BAD_CLASS;
                            } else {
                                int L = 0;
#pragma unroll
                                for (int i = 0; i + 1 < N; ++i) L += (w >= T[i]) ? 1 : 0;
                                L = pin ? 0 : min(L, ml);
                                lev = L;
                                tl = tk4[k][0];
#pragma unroll
                                for (int LL = 1; LL < N; ++LL) tl = L == LL ? tk4[k][LL] : tl;
#pragma unroll
                                for (int c = 0; c < NCM; ++c)
#pragma unroll
                                    for (int LL = 0; LL < N; ++LL) {
                                        const bool hit = (uint32_t)c == cls && LL == L;
                                        cc[c][LL] += hit ? 1u : 0u;
                                        ct[c][LL] += hit ? tl : 0u;
                                    }
                            }
                        }
                        const uint64_t pos = (qb - pq) * 4 + 32 * k + lane;   // piece-relative slot
                        if (qin) buf[pos] = lev < 0 ? 0xFF000000u : ((uint32_t)lev << 24) | (cls << 16) | tl;
#pragma unroll
                        for (int L = 0; L < N; ++L) cntL[L] += __popc(__ballot_sync(0xFFFFFFFFu, lev == L));
                    }
                }
                if (lane < N) {
                    int v = cntL[0];
#pragma unroll
                    for (int L = 1; L < N; ++L) v = lane == L ? cntL[L] : v;
                    wcount[warp][lane] = v;
                }
                __syncthreads();
                int before[N], total[N];
#pragma unroll
                for (int L = 0; L < N; ++L) {
                    before[L] = 0;
                    total[L] = 0;
                    for (int w2 = 0; w2 < kClWarps; ++w2) {
                        before[L] += w2 < warp ? wcount[w2][L] : 0;
                        total[L] += wcount[w2][L];
                    }
                }
                // only the last W requests of each level in the piece enter the ring: a warp
                // whose run ends before them has nothing to write
                bool any = false;
#pragma unroll
                for (int L = 0; L < N; ++L) {
                    int mine = 0;
                    for (int w2 = 0; w2 < kClWarps; ++w2) mine += w2 == warp ? wcount[w2][L] : 0;
                    any = any || (before[L] + mine > total[L] - W && mine > 0);
                }
                for (uint64_t qb = wq0; any && qb < wq1; qb += 32) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint64_t pos = (qb - pq) * 4 + 32 * k + lane;
                        const bool qin = qb + (uint64_t)(8 * k + (lane >> 2)) < wq1;
                        const uint32_t v = qin ? buf[pos] : 0xFF000000u;
                        const int lev = (int)(v >> 24);
#pragma unroll
                        for (int L = 0; L < N; ++L) {
                            const uint32_t bl = __ballot_sync(0xFFFFFFFFu, lev == L);
                            if (lev == L) {
                                const int rank = before[L] + __popc(bl & ((1u << lane) - 1u));
                                if (rank >= total[L] - W) {
                                    // the slot's previous entry (from before this piece) leaves the
                                    // window: occupied iff the ring was full or the slot is below its fill
                                    const int slot = (int)(((int64_t)head[L] + rank) % W);
                                    if (size[L] == W || slot < size[L]) {
                                        const uint32_t old = ring[L * W + slot];
                                        const int oc = (int)(old >> 16);
#pragma unroll
                                        for (int c = 0; c < NCM; ++c)
                                            if (c == oc) { dn[L][c] -= 1; dk[L][c] -= (int)(old & 0xFFFFu); }
                                    }
                                    ring[L * W + slot] = v & 0x00FFFFFFu;
#pragma unroll
                                    for (int c = 0; c < NCM; ++c)
                                        if ((uint32_t)c == ((v >> 16) & 0xFFu)) { dn[L][c] += 1; dk[L][c] += (int)(v & 0xFFFFu); }
                                }
                            }
                            before[L] += __popc(bl);
                        }
                    }
                }
                // fold the piece: per-warp sums into slots, then one thread per value adds the
                // 8 warps (no shared atomics; every sum is an exact integer)
#pragma unroll
                for (int c = 0; c < NCM; ++c) {
                    if (c >= NC) break;
#pragma unroll
                    for (int L = 0; L < N; ++L) {
                        const uint32_t sc = __reduce_add_sync(0xFFFFFFFFu, cc[c][L]);
                        const uint32_t st = __reduce_add_sync(0xFFFFFFFFu, ct[c][L]);
                        const int sn = (int)__reduce_add_sync(0xFFFFFFFFu, (uint32_t)dn[L][c]);
                        const int sk = (int)__reduce_add_sync(0xFFFFFFFFu, (uint32_t)dk[L][c]);
                        if (lane == 0) {
                            const int v = (c * N + L) * 4;
                            slots[warp][v + 0] = sc; slots[warp][v + 1] = st;
                            slots[warp][v + 2] = (uint32_t)sn; slots[warp][v + 3] = (uint32_t)sk;
                        }
                        cc[c][L] = 0u; ct[c][L] = 0u;
                    }
                }
                __syncthreads();
                if (tid < N) {
                    int tt = total[0];
#pragma unroll
                    for (int L = 1; L < N; ++L) tt = tid == L ? total[L] : tt;
                    head[tid] = (int)(((int64_t)head[tid] + tt) % W);
                    size[tid] = min(size[tid] + tt, W);
                }
                for (int v = tid; v < NC * N; v += kClThreads) {
                    const int c = v / N, L = v % N;
                    unsigned long long sc = 0, st = 0;
                    long long sn = 0, sk = 0;
                    for (int w2 = 0; w2 < kClWarps; ++w2) {
                        sc += slots[w2][v * 4 + 0]; st += slots[w2][v * 4 + 1];
                        sn += (int)slots[w2][v * 4 + 2]; sk += (int)slots[w2][v * 4 + 3];
                    }
                    csum[c][L][0] += sc; csum[c][L][1] += st;
                    wsum[L][c][0] = (unsigned long long)((long long)wsum[L][c][0] + sn);
                    wsum[L][c][1] = (unsigned long long)((long long)wsum[L][c][1] + sk);
                }
                __syncthreads();
            }
        }
        __syncthreads();
        if (tid == 0) {   // cell_epilogue's formulas and order
            const double kp = k0_s * a.pue;
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
                    Q += n_ * q_r[L];
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
    const int64_t chains = (int64_t)a.R_local * a.X;
    if (chains == 0) return cudaSuccess;
    const size_t smem = ((size_t)a.n * a.W + kClPiece) * 4;
    cudaError_t e = cudaSuccess;
#define CL_CASE(NN)                                                                                  \
    case NN: {                                                                                       \
        auto kern = a.NC == 1 ? closed_loop_kernel<NN, 1> : closed_loop_kernel<NN, kMaxClasses>;     \
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
