// fp64_check.cu -- the per-request fp64 accounting mode (SURVEY 8(a) a7/a8,
// "the literal north_star structure"): every request's Eq. 1 energy, time
// and carbon (E = ef + et*tok, T = pf + pt*tok, reading L11;
// C = k0*PUE*E + k1*T, reading L2) and its quality q[level] (reading L15),
// at the level the a6 rule gives from its Philox word (reading L10), summed
// per cell in fp64 with warp-shuffle and block tree reductions.  It is a
// cross-check of sprout_simulate_trace's closed form (exact integer
// statistics, then Eq. 1 once per (class, level)), not the timed path: the
// level is taken straight from the cell's thresholds (no breakpoint bins),
// so it shares nothing with the streaming kernel but the draw.
#include <cuda_runtime.h>
#include "sprout_device.cuh"
#include "sprout_kernels.cuh"

namespace sprout {

constexpr int kF64Threads = 256;

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xFFFFFFFFu, v, d));
    return v;   // lane 0: the warp's sum (a fixed tree)
}

// One CTA per segment; the segment's cells one after the other (every cell
// re-reads the segment's requests: verification mode).  Thread t sums the
// requests s0 + t, s0 + t + 256, ... in order; the 256 partial sums are then
// reduced by a fixed tree (warp shuffles, then warp 0 over the 8 warp sums),
// so the result is deterministic.
__global__ void __launch_bounds__(kF64Threads) fp64_cells_kernel(const __grid_constant__ F64Args a) {
    __shared__ double part[kF64Threads / 32][4];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int N = a.n;
    for (int64_t sl = blockIdx.x; sl < a.n_segments; sl += gridDim.x) {
        const int64_t s = a.first_segment + sl;
        const int64_t s0 = a.seg_offsets[sl], s1 = a.seg_offsets[sl + 1];
        const bool seg_ok = s0 >= 0 && s0 <= s1 && s1 <= a.n_requests;
        const double kp = __dmul_rn(a.k0[s], a.pue);
        const double *qrow = a.q + (a.profile_per_interval ? s : s / a.T) * N;
        for (int j = 0; j < a.X; ++j) {
            const int64_t cell = sl * a.X + j;
            const bool ok = seg_ok && a.cell_status[cell] == SPROUT_CELL_OK;
            double E = 0.0, T = 0.0, Cg = 0.0, Q = 0.0;
            if (ok) {
                uint32_t thr[kMaxLevels];
                for (int i = 0; i + 1 < N; ++i) thr[i] = a.threshold[cell * (N - 1) + i];
                const int ml = a.max_level[cell];
                for (int64_t r = s0 + tid; r < s1; r += kF64Threads) {
                    int cls = 0;
                    bool pinned = false;
                    if (a.flags) {
                        const uint8_t f = a.flags[r];
                        pinned = f & 1u;
                        cls = (f >> 1) & 3;
                    }
                    if (cls >= a.NC) continue;
                    int L = 0;
                    if (!pinned) {
                        const uint64_t g = a.first_request + (uint64_t)r;
                        const Philox4 d = philox4x32_10_rk((uint32_t)(g >> 2), (uint32_t)(g >> 34), 0u, 0u, a.rk0, a.rk1);
                        const uint32_t w = d.v[g & 3u];
                        int c = 0;
                        for (int i = 0; i + 1 < N; ++i) c += (w >= thr[i]) ? 1 : 0;
                        L = c < ml ? c : ml;
                    }
                    const double tok = (double)a.tokens[(size_t)L * a.pitch + r];
                    const double Er = __dadd_rn(a.cost.ef[cls][L], __dmul_rn(a.cost.et[cls][L], tok));
                    const double Tr = __dadd_rn(a.cost.pf[cls][L], __dmul_rn(a.cost.pt[cls][L], tok));
                    E = __dadd_rn(E, Er);
                    T = __dadd_rn(T, Tr);
                    Cg = __dadd_rn(Cg, __dadd_rn(__dmul_rn(kp, Er), __dmul_rn(a.k1, Tr)));
                    Q = __dadd_rn(Q, qrow[L]);
                }
            }
            E = warp_sum_f64(E);
            T = warp_sum_f64(T);
            Cg = warp_sum_f64(Cg);
            Q = warp_sum_f64(Q);
            if (lane == 0) { part[warp][0] = E; part[warp][1] = T; part[warp][2] = Cg; part[warp][3] = Q; }
            __syncthreads();
            if (warp == 0) {
                double v[4];
#pragma unroll
                for (int f = 0; f < 4; ++f) {
                    v[f] = lane < kF64Threads / 32 ? part[lane][f] : 0.0;
#pragma unroll
                    for (int d = 4; d > 0; d >>= 1) v[f] = __dadd_rn(v[f], __shfl_down_sync(0xFFFFFFFFu, v[f], d));
                }
                if (lane == 0) {
                    a.energy[cell] = v[0];
                    a.time_s[cell] = v[1];
                    a.carbon[cell] = v[2];
                    a.quality[cell] = v[3];
                }
            }
            __syncthreads();
        }
    }
}

cudaError_t launch_fp64_cells(const F64Args &a, cudaStream_t stream, int *launches) {
    if (a.n_segments == 0) return cudaSuccess;
    int64_t grid = a.n_segments < 148 * 16 ? a.n_segments : 148 * 16;
    fp64_cells_kernel<<<(unsigned)grid, kF64Threads, 0, stream>>>(a);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace sprout
