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

        // ---- per-cell validation (SPROUT_CELL_INVALID) ----
        bool ok = (xi >= 0.0 && xi <= 1.0) && finite_nonneg(k0) && finite_nonneg(kmin) &&
                  finite_nonneg(kmax) && (kmax >= kmin);
#pragma unroll
        for (int i = 0; i < N; ++i)
            ok = ok && (q[i] >= 0.0 && q[i] <= 1.0) && finite_nonneg(e[i]) && finite_nonneg(p[i]);

        double x[N];
        double best = __longlong_as_double(0x7ff0000000000000ll);  // +inf
        int best_id = -1;
        uint8_t status = SPROUT_CELL_OK;
        double b = __longlong_as_double(0x7ff8000000000000ll);      // NaN

        if (!ok) {
            status = SPROUT_CELL_INVALID;
        } else if (a.scheme != 0) {
            // ---- competing schemes: no quality floor; b reports
            // the mix's expected quality q.x, best its expected carbon c.x ----
            const double kp = __dmul_rn(k0, a.pue);
            double c[N];
#pragma unroll
            for (int i = 0; i < N; ++i) c[i] = __dadd_rn(__dmul_rn(kp, e[i]), __dmul_rn(a.k1, p[i]));
            if (a.scheme == 1) {
                // CO2_Opt: the cheapest level, ties to the lowest index (reading L17)
                int m = 0;
                double cm = c[0];
#pragma unroll
                for (int i = 1; i < N; ++i)
                    if (c[i] < cm) { cm = c[i]; m = i; }
#pragma unroll
                for (int i = 0; i < N; ++i) x[i] = i == m ? 1.0 : 0.0;
                best_id = m;
            } else {
                // Sprout_Sta sweep: grid point j of step 1/D (reading L18)
                int k[N];
                grid_unrank<N>(a.grid_den, j, k);
                int nz = 0, last = 0;
#pragma unroll
                for (int i = 0; i < N; ++i) {
                    x[i] = __ddiv_rn((double)k[i], (double)a.grid_den);
                    if (k[i] != 0) { ++nz; last = i; }
                }
                best_id = nz == 1 ? last : SPROUT_VERTEX_GRID;
            }
            double o = 0.0, qx = 0.0;
#pragma unroll
            for (int i = 0; i < N; ++i) {
                o = __dadd_rn(o, __dmul_rn(c[i], x[i]));
                qx = __dadd_rn(qx, __dmul_rn(q[i], x[i]));
            }
            best = o;
            b = qx;
        } else {
            // ---- Eq. 3, readings L3 and L7 ----
            double f = 0.0;
            if (kmax > kmin) {
                f = __ddiv_rn(__dsub_rn(k0, kmin), __dsub_rn(kmax, kmin));
                f = f < 0.0 ? 0.0 : (f > 1.0 ? 1.0 : f);
            }
            b = __dmul_rn(__dsub_rn(1.0, __dmul_rn(f, xi)), q[0]);

            // ---- Eq. 2 + PUE (reading L2) ----
            const double kp = __dmul_rn(k0, a.pue);
            double c[N];
#pragma unroll
            for (int i = 0; i < N; ++i) c[i] = __dadd_rn(__dmul_rn(kp, e[i]), __dmul_rn(a.k1, p[i]));

            // ---- vertex enumeration, first strict minimum (readings L6, L8) ----
            int bi = -1, bj = -1;
            double bxh = 0.0, bxl = 0.0;
#pragma unroll
            for (int i = 0; i < N; ++i) {
                if (q[i] >= b && c[i] < best) {
                    best = c[i]; best_id = i; bi = i; bj = -1;
                }
            }
            int edge = 0;
#pragma unroll
            for (int i = 0; i < N; ++i) {
#pragma unroll
                for (int jj = i + 1; jj < N; ++jj, ++edge) {
                    const bool straddle = (q[i] < b && q[jj] > b) || (q[i] > b && q[jj] < b);
                    if (!straddle) continue;
                    const int h = q[i] > q[jj] ? i : jj;
                    const int l = q[i] > q[jj] ? jj : i;
                    const double ch = h == i ? c[i] : c[jj], cl = h == i ? c[jj] : c[i];
                    const double qh = h == i ? q[i] : q[jj], ql = h == i ? q[jj] : q[i];
                    if (!(cl < ch)) continue;
                    const double xh = __ddiv_rn(__dsub_rn(b, ql), __dsub_rn(qh, ql));
                    const double xl = __dsub_rn(1.0, xh);
                    const double o = __dadd_rn(cl, __dmul_rn(__dsub_rn(ch, cl), xh));
                    if (o < best) {
                        best = o; best_id = N + edge; bi = h; bj = l; bxh = xh; bxl = xl;
                    }
                }
            }
            if (best_id < 0) {
                status = SPROUT_CELL_INFEASIBLE;
            } else {
#pragma unroll
                for (int i = 0; i < N; ++i) x[i] = (i == bi) ? (bj < 0 ? 1.0 : bxh) : (i == bj ? bxl : 0.0);
            }
        }

        // ---- outputs ----
        const double qnan = __longlong_as_double(0x7ff8000000000000ll);
        if (status != SPROUT_CELL_OK) {
#pragma unroll
            for (int i = 0; i < N; ++i) x[i] = qnan;
            best = qnan;
            best_id = 255;
        }
#pragma unroll
        for (int i = 0; i < N; ++i) a.x[cell * N + i] = x[i];
        a.objective[cell] = best;
        a.q_lb[cell] = status == SPROUT_CELL_INVALID ? qnan : b;
        a.vertex[cell] = (uint8_t)best_id;
        a.cell_status[cell] = status;

        // ---- inverse-CDF thresholds (reading L10) ----
        int ml = N - 1;
        if (status != SPROUT_CELL_OK) {
#pragma unroll
            for (int i = 0; i + 1 < N; ++i) a.threshold[cell * (N - 1) + i] = 0xFFFFFFFFu;
            ml = 0;
        } else {
            double cum = 0.0;
            bool found = false;
#pragma unroll
            for (int i = 0; i + 1 < N; ++i) {
                cum = __dadd_rn(cum, x[i]);
                const double cl = ceil(__dmul_rn(cum, 4294967296.0));   // exact scale by 2^32
                uint32_t t;
                if (cl >= 4294967296.0) {
                    t = 0xFFFFFFFFu;                                     // 2^32, saturated
                    if (!found) { ml = i; found = true; }
                } else {
                    t = (uint32_t)(uint64_t)cl;
                }
                a.threshold[cell * (N - 1) + i] = t;
            }
        }
        a.max_level[cell] = (uint8_t)ml;
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
