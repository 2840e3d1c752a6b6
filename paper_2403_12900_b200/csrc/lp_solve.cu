// lp_solve.cu -- step 1 of the hot path: one thread per (region, interval, xi)
// cell solves the directive LP of Eqs. 4-7 exactly by vertex
// enumeration, in registers, in fp64.
//
// Every floating-point operation is an explicit __d*_rn intrinsic so nvcc can
// never contract it into an FMA (reading L7): the result is the IEEE-754
// binary64 round-to-nearest value of the formula in the stated order, which
// the CPU oracle computes independently with -ffp-contract=off.
#include "sprout_device.cuh"
#include "sprout_kernels.cuh"
#include "lp_cell.cuh"

namespace sprout {

template <int N>
__global__ void __launch_bounds__(256) lp_solve_kernel(LpArgs a) {
    const int64_t n_cells = a.n_segments * (int64_t)a.X;
    for (int64_t cell = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; cell < n_cells;
         cell += (int64_t)gridDim.x * blockDim.x) {
        int64_t s, r;
        int j;
        if (a.small) {
            const uint32_t c32 = (uint32_t)cell, sl = a.div_x.div(c32);
            j = (int)(c32 - sl * a.div_x.d);
            s = a.first_segment + sl;
            r = a.div_t.div((uint32_t)s);
        } else {
            s = a.first_segment + cell / a.X;
            j = (int)(cell % a.X);
            r = s / a.T;
        }
        const int64_t row = a.profile_per_interval ? s : r;

        const double k0 = a.k0[s], kmin = a.kmin[r], kmax = a.kmax[r];
        const double xi = a.scheme == 0 ? a.xi[j] : 0.0;   // the other schemes have no xi
        double e[N], p[N], q[N];
#pragma unroll
        for (int i = 0; i < N; ++i) {
            e[i] = a.e[row * N + i];
            p[i] = a.p[row * N + i];
            q[i] = a.q[row * N + i];
        }

        LpCell<N> o;
        lp_cell<N>(k0, kmin, kmax, xi, e, p, q, a.k1, a.pue, a.scheme, a.grid_den, j, o);
#pragma unroll
        for (int i = 0; i < N; ++i) a.x[cell * N + i] = o.x[i];
        a.objective[cell] = o.objective;
        a.q_lb[cell] = o.q_lb;
        a.vertex[cell] = o.vertex;
        a.cell_status[cell] = o.status;
#pragma unroll
        for (int i = 0; i + 1 < N; ++i) a.threshold[cell * (N - 1) + i] = o.T[i];
        a.max_level[cell] = o.max_level;
    }
}

cudaError_t launch_lp_solve(const LpArgs &args, cudaStream_t stream, int *launches) {
    LpArgs a = args;
    const int64_t n_cells = a.n_segments * (int64_t)a.X;
    a.small = (n_cells < (int64_t)0xFFFFFFFFll && a.first_segment + a.n_segments < (int64_t)0xFFFFFFFFll &&
               a.T < (int64_t)0xFFFFFFFFll) ? 1 : 0;
    a.div_x = FastDiv((uint32_t)a.X);
    a.div_t = FastDiv(a.T < (int64_t)0xFFFFFFFFll ? (uint32_t)a.T : 1u);
    if (n_cells == 0) return cudaSuccess;
    const int threads = 256;
    int64_t blocks = (n_cells + threads - 1) / threads;
    if (blocks > 148 * 64) blocks = 148 * 64;
    switch (a.n) {
#define LP_CASE(NN) case NN: lp_solve_kernel<NN><<<(unsigned)blocks, threads, 0, stream>>>(a); break;
        LP_CASE(1) LP_CASE(2) LP_CASE(3) LP_CASE(4) LP_CASE(5) LP_CASE(6) LP_CASE(7) LP_CASE(8)
#undef LP_CASE
        default: return cudaErrorInvalidValue;
    }
    ++*launches;
    return cudaGetLastError();
}

}  // namespace sprout
