// lp_cell.cuh -- one cell of step 1 (a1-a4): validation, Eq. 3 floor,
// Eq. 2 cost vector, the LP of Eqs. 4-7 by vertex enumeration (or a
// competing scheme's mix), and the inverse-CDF thresholds -- all in
// registers, every fp64 operation an explicit __d*_rn intrinsic (reading
// L7).  Shared by lp_solve_kernel and the closed-loop kernel.
#pragma once
#include "sprout_device.cuh"

namespace sprout {

template <int N>
struct LpCell {
    double x[N];
    double objective, q_lb;
    uint32_t T[N > 1 ? N - 1 : 1];   // thresholds, 2^32 saturated to 0xFFFFFFFF
    uint8_t vertex, status, max_level;
};

template <int N>
__device__ __forceinline__ void lp_cell(double k0, double kmin, double kmax, double xi, const double (&e)[N],
                                        const double (&p)[N], const double (&q)[N], double k1, double pue,
                                        int scheme, int grid_den, int j, LpCell<N> &o) {
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
    } else if (scheme != 0) {
        // ---- competing schemes: no quality floor; b reports
        // the mix's expected quality q.x, best its expected carbon c.x ----
        const double kp = __dmul_rn(k0, pue);
        double c[N];
#pragma unroll
        for (int i = 0; i < N; ++i) c[i] = __dadd_rn(__dmul_rn(kp, e[i]), __dmul_rn(k1, p[i]));
        if (scheme == 1) {
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
            grid_unrank<N>(grid_den, j, k);
            int nz = 0, last = 0;
#pragma unroll
            for (int i = 0; i < N; ++i) {
                x[i] = __ddiv_rn((double)k[i], (double)grid_den);
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
        const double kp = __dmul_rn(k0, pue);
        double c[N];
#pragma unroll
        for (int i = 0; i < N; ++i) c[i] = __dadd_rn(__dmul_rn(kp, e[i]), __dmul_rn(k1, p[i]));

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
    for (int i = 0; i < N; ++i) o.x[i] = x[i];
    o.objective = best;
    o.q_lb = status == SPROUT_CELL_INVALID ? qnan : b;
    o.vertex = (uint8_t)best_id;
    o.status = status;

    // ---- inverse-CDF thresholds (reading L10) ----
    int ml = N - 1;
    if (status != SPROUT_CELL_OK) {
#pragma unroll
        for (int i = 0; i + 1 < N; ++i) o.T[i] = 0xFFFFFFFFu;
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
            o.T[i] = t;
        }
    }
    o.max_level = (uint8_t)ml;
}

}  // namespace sprout
