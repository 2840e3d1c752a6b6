// reduce.cu -- step 3 (local part of a9): per (region, xi) and per xi group
// totals of the cell statistics, in a fixed order (deterministic):
//   stage 1: block = (region, chunk of intervals); thread = (xi column,
//            interval phase q); each thread sums its column over the chunk's
//            intervals t = q, q + Q, ... in order, then the Q phases are
//            combined in order through shared memory;
//   stage 2: per region, 8 warps sum the chunk partials (warp w: chunks
//            w, w + 8, ..., lanes = consecutive (xi, stat) outputs, coalesced)
//            and warp 0 combines the 8 in order;
//   stage 3: the global row, one warp per (xi, stat): lanes over regions in
//            order, then a fixed butterfly.
// Conservation holds exactly for the integer statistics (carried in
// fp64, exact below 2^53).  The cross-GPU SUM is the caller's NCCL allreduce.
#include "sprout_device.cuh"
#include "sprout_kernels.cuh"

namespace sprout {

constexpr int kRedThreads = 256;
#ifndef SPROUT_RED_PER_THREAD
#define SPROUT_RED_PER_THREAD 4
#endif
constexpr int kRedPerThread = SPROUT_RED_PER_THREAD;   // intervals per thread per chunk

// column tile width (power of two >= X, <= 256) and interval phases per block
static inline __host__ __device__ int red_xp(int X) {
    int xp = 1;
    while (xp < X && xp < kRedThreads) xp <<= 1;
    return xp;
}

template <int N>
__global__ void __launch_bounds__(kRedThreads, 4) reduce_stage1(const __grid_constant__ ReduceArgs a) {
    constexpr int K = 11 + 2 * N;
    __shared__ double red[kRedThreads];
    const int xp = red_xp(a.X), Q = kRedThreads / xp;
    const int q = threadIdx.x / xp, jl = threadIdx.x % xp;
    const int64_t r = a.r_lo + blockIdx.y;
    const int chunk = blockIdx.x;
    const int64_t t_lo = (int64_t)chunk * a.chunk;
    int64_t t_hi = t_lo + a.chunk;
    if (t_hi > a.T) t_hi = a.T;
    const int64_t seg_lo = a.first_segment, seg_hi = a.first_segment + a.n_segments;
    const int NC = a.NC;
    for (int jt = 0; jt * xp < a.X; ++jt) {
        const int j = jt * xp + jl;
        double acc[K];
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] = 0.0;
        if (j < a.X) {
            for (int64_t t = t_lo + q; t < t_hi; t += Q) {
                const int64_t s = r * a.T + t;
                if (s < seg_lo || s >= seg_hi) continue;
                const int64_t sl = s - seg_lo;
                const int64_t cell = sl * a.X + j;
                double m = 0.0, pin = 0.0;
                for (int c = 0; c < NC; ++c) {
                    m += (double)a.seg_count[sl * NC + c];
                    pin += (double)a.seg_pinned[sl * NC + c];
                }
                acc[0] += m;
                acc[1] += pin;
#pragma unroll
                for (int k = 0; k < 4; ++k) acc[6 + k] += a.seg_base[sl * 4 + k];
                if (a.cell_status[cell] != SPROUT_CELL_OK) continue;
                acc[2] += a.energy[cell];
                acc[3] += a.time_s[cell];
                acc[4] += a.carbon[cell];
                acc[5] += a.quality[cell];
                acc[10] += m * a.objective[cell];
#pragma unroll
                for (int L = 0; L < N; ++L) {
                    uint64_t cn = 0, tk = 0;
                    for (int c = 0; c < NC; ++c) {
                        cn += a.cnt[(cell * NC + c) * N + L];
                        tk += a.tok[(cell * NC + c) * N + L];
                    }
                    acc[11 + L] += (double)cn;
                    acc[11 + N + L] += (double)tk;
                }
            }
        }
        // combine the Q phases in order (q = 0, 1, ...): deterministic
        double *out = a.partials + (((size_t)blockIdx.y * a.n_chunks + chunk) * a.X + j) * K;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            red[threadIdx.x] = acc[k];
            __syncthreads();
            if (q == 0 && j < a.X) {
                double v = 0.0;
                for (int qq = 0; qq < Q; ++qq) v += red[qq * xp + jl];
                out[k] = v;
            }
            __syncthreads();
        }
    }
}

// regional rows: out[r][jk] = sum over chunks (rows outside the shard: 0)
__global__ void __launch_bounds__(kRedThreads) reduce_stage2(const __grid_constant__ ReduceArgs a) {
    __shared__ double part[kRedThreads / 32][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t per_row = (int64_t)a.X * a.K;
    const int64_t jk = (int64_t)blockIdx.x * 32 + lane;
    const int64_t r = blockIdx.y;
    double v = 0.0;
    if (jk < per_row && r >= a.r_lo && r < a.r_hi) {
        // only the chunks holding intervals of the shard: the others' partials are exact
        // zeros (stage 1 skips foreign intervals), so the sum is the same bit for bit
        const int64_t t_lo = max((int64_t)0, a.first_segment - r * a.T);
        const int64_t t_hi = min(a.T, a.first_segment + a.n_segments - r * a.T);
        const int c_lo = (int)(t_lo / a.chunk), c_hi = (int)((t_hi + a.chunk - 1) / a.chunk);
        const double *p = a.partials + (size_t)(r - a.r_lo) * a.n_chunks * per_row + jk;
        int c = c_lo + warp;
        // two accumulators interleaved would change the order; keep one, with the loads unrolled ahead
#pragma unroll 8
        for (; c < c_hi; c += kRedThreads / 32) v += p[(size_t)c * per_row];
    }
    part[warp][lane] = v;
    __syncthreads();
    if (warp == 0 && jk < per_row) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < kRedThreads / 32; ++w) t += part[w][lane];
        a.out[r * per_row + jk] = t;
    }
}

// global row: out[R][jk] = sum over regions of out[r][jk]
__global__ void __launch_bounds__(kRedThreads) reduce_stage3(const __grid_constant__ ReduceArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t per_row = (int64_t)a.X * a.K;
    const int64_t jk = (int64_t)blockIdx.x * (kRedThreads / 32) + (threadIdx.x >> 5);
    if (jk >= per_row) return;
    double v = 0.0;
    for (int64_t r = lane; r < a.R; r += 32) v += a.out[r * per_row + jk];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
    if (lane == 0) a.out[(int64_t)a.R * per_row + jk] = v;
}

static void reduce_geometry(int X, int64_t T, int64_t first_segment, int64_t n_segments, int64_t *r_lo,
                            int64_t *r_hi, int *chunk, int *n_chunks) {
    *chunk = kRedPerThread * (kRedThreads / red_xp(X));
    *n_chunks = (int)((T + *chunk - 1) / *chunk);
    if (n_segments <= 0) {
        *r_lo = *r_hi = 0;
        return;
    }
    *r_lo = first_segment / T;
    *r_hi = (first_segment + n_segments - 1) / T + 1;
}

size_t reduce_workspace_bytes(int n, int X, int R, int64_t T, int64_t first_segment, int64_t n_segments) {
    (void)R;
    int64_t r_lo, r_hi;
    int chunk, n_chunks;
    reduce_geometry(X, T, first_segment, n_segments, &r_lo, &r_hi, &chunk, &n_chunks);
    const int K = 11 + 2 * n;
    return (size_t)(r_hi - r_lo) * n_chunks * X * K * sizeof(double) + 256;
}

cudaError_t launch_reduce(ReduceArgs &a, void *ws, cudaStream_t stream, int *launches) {
    reduce_geometry(a.X, a.T, a.first_segment, a.n_segments, &a.r_lo, &a.r_hi, &a.chunk, &a.n_chunks);
    a.K = 11 + 2 * a.n;
    a.partials = static_cast<double *>(ws);
    if (a.r_hi > a.r_lo) {
        dim3 grid((unsigned)a.n_chunks, (unsigned)(a.r_hi - a.r_lo));
        switch (a.n) {
#define RD_CASE(NN) case NN: reduce_stage1<NN><<<grid, kRedThreads, 0, stream>>>(a); break;
            RD_CASE(1) RD_CASE(2) RD_CASE(3) RD_CASE(4) RD_CASE(5) RD_CASE(6) RD_CASE(7) RD_CASE(8)
#undef RD_CASE
            default: return cudaErrorInvalidValue;
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        ++*launches;
    }
    const int64_t per_row = (int64_t)a.X * a.K;
    dim3 g2((unsigned)((per_row + 31) / 32), (unsigned)a.R);
    reduce_stage2<<<g2, kRedThreads, 0, stream>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    ++*launches;
    const int64_t wpb = kRedThreads / 32;
    reduce_stage3<<<(unsigned)((per_row + wpb - 1) / wpb), kRedThreads, 0, stream>>>(a);
    ++*launches;
    return cudaGetLastError();
}

// worst cell status
__global__ void check_cells_kernel(const uint8_t *status, int64_t n, uint32_t *out) {
    uint32_t worst = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t s = status[i];
        worst |= (s == SPROUT_CELL_INVALID) ? 1u : (s == SPROUT_CELL_INFEASIBLE ? 2u : (s ? 4u : 0u));
    }
    worst = __reduce_or_sync(0xFFFFFFFFu, worst);
    if ((threadIdx.x & 31) == 0 && worst) atomicOr(out, worst);
}

cudaError_t launch_check_cells(const uint8_t *status, int64_t n_cells, uint32_t *out, cudaStream_t stream,
                               int *launches) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(uint32_t), stream);
    if (e != cudaSuccess) return e;
    if (n_cells == 0) return cudaSuccess;
    int64_t blocks = (n_cells + 255) / 256;
    if (blocks > 1024) blocks = 1024;
    check_cells_kernel<<<(unsigned)blocks, 256, 0, stream>>>(status, n_cells, out);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace sprout
