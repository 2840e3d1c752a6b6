// reduce.cu -- step 3 (local part of a9): per (region, xi) and per xi group
// totals of the cell statistics, in a fixed order (deterministic):
//   stage 1: block (region, chunk of intervals), thread = xi column; each
//            thread sums its column over the chunk's segments in order;
//   stage 2: one thread per output (row, xi, stat) sums the chunks in order
//            (and, for the global row, the regions in order).
// Conservation holds exactly for the integer statistics (carried in
// fp64, exact below 2^53).  The cross-GPU SUM is the caller's NCCL allreduce.
#include "sprout_device.cuh"
#include "sprout_kernels.cuh"

namespace sprout {

template <int N>
__global__ void __launch_bounds__(256) reduce_stage1(const __grid_constant__ ReduceArgs a) {
    constexpr int K = 11 + 2 * N;
    const int64_t r = a.r_lo + blockIdx.y;
    const int chunk = blockIdx.x;
    const int64_t t_lo = (int64_t)chunk * a.chunk;
    int64_t t_hi = t_lo + a.chunk;
    if (t_hi > a.T) t_hi = a.T;
    int64_t s_lo = r * a.T + t_lo, s_hi = r * a.T + t_hi;
    if (s_lo < a.first_segment) s_lo = a.first_segment;
    if (s_hi > a.first_segment + a.n_segments) s_hi = a.first_segment + a.n_segments;
    const int NC = a.NC;
    for (int j = threadIdx.x; j < a.X; j += blockDim.x) {
        double acc[K];
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] = 0.0;
        for (int64_t s = s_lo; s < s_hi; ++s) {
            const int64_t sl = s - a.first_segment;
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
        double *out = a.partials + (((size_t)blockIdx.y * a.n_chunks + chunk) * a.X + j) * K;
#pragma unroll
        for (int k = 0; k < K; ++k) out[k] = acc[k];
    }
}

__global__ void reduce_stage2(const __grid_constant__ ReduceArgs a) {
    const int K = a.K;
    const int64_t per_row = (int64_t)a.X * K;
    const int64_t total = (int64_t)(a.R + 1) * per_row;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / per_row;
        const int64_t jk = i % per_row;
        double v = 0.0;
        if (row < a.R) {
            if (row >= a.r_lo && row < a.r_hi) {
                const double *p = a.partials + (size_t)(row - a.r_lo) * a.n_chunks * per_row + jk;
                for (int c = 0; c < a.n_chunks; ++c) v += p[(size_t)c * per_row];
            }
        } else {
            for (int64_t r = a.r_lo; r < a.r_hi; ++r) {
                const double *p = a.partials + (size_t)(r - a.r_lo) * a.n_chunks * per_row + jk;
                double rv = 0.0;
                for (int c = 0; c < a.n_chunks; ++c) rv += p[(size_t)c * per_row];
                v += rv;
            }
        }
        a.out[i] = v;
    }
}

static void reduce_geometry(int64_t T, int64_t first_segment, int64_t n_segments, int64_t *r_lo, int64_t *r_hi,
                            int *chunk, int *n_chunks) {
    *chunk = 32;
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
    reduce_geometry(T, first_segment, n_segments, &r_lo, &r_hi, &chunk, &n_chunks);
    const int K = 11 + 2 * n;
    return (size_t)(r_hi - r_lo) * n_chunks * X * K * sizeof(double) + 256;
}

cudaError_t launch_reduce(ReduceArgs &a, void *ws, cudaStream_t stream, int *launches) {
    reduce_geometry(a.T, a.first_segment, a.n_segments, &a.r_lo, &a.r_hi, &a.chunk, &a.n_chunks);
    a.K = 11 + 2 * a.n;
    a.partials = static_cast<double *>(ws);
    if (a.r_hi > a.r_lo) {
        dim3 grid((unsigned)a.n_chunks, (unsigned)(a.r_hi - a.r_lo));
        int threads = a.X < 256 ? ((a.X + 31) / 32) * 32 : 256;
        switch (a.n) {
#define RD_CASE(NN) case NN: reduce_stage1<NN><<<grid, threads, 0, stream>>>(a); break;
            RD_CASE(1) RD_CASE(2) RD_CASE(3) RD_CASE(4) RD_CASE(5) RD_CASE(6) RD_CASE(7) RD_CASE(8)
#undef RD_CASE
            default: return cudaErrorInvalidValue;
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        ++*launches;
    }
    const int64_t total = (int64_t)(a.R + 1) * a.X * a.K;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    reduce_stage2<<<(unsigned)blocks, 256, 0, stream>>>(a);
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
