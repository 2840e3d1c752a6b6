// schemes.cu -- the Sprout_Sta choice: after a STATIC_GRID sweep
// (steps 1-3 with one cell per grid point), pick per region the static mix
// of least realised carbon whose realised quality meets Eq. 3's floor at the
// region's mean carbon intensity (reading L18).  One warp per region; every
// floating-point operation is an explicit __d*_rn intrinsic (reading L7),
// and the orders are fixed: the k0 mean is a sequential sum in interval
// order, the realised quality a sum in level order, the argmin strict with
// ties to the lowest grid point.
#include "sprout_device.cuh"
#include "sprout_kernels.cuh"

namespace sprout {

__global__ void __launch_bounds__(32) select_static_kernel(const SelectArgs a) {
    const int r = blockIdx.x;
    const int lane = threadIdx.x;
    const double *qr = a.q + (size_t)r * a.n;
    double b = 0.0;
    if (lane == 0) {
        const double *k0 = a.k0 + (int64_t)r * a.T;
        double sum = 0.0;
        for (int64_t t = 0; t < a.T; ++t) sum = __dadd_rn(sum, k0[t]);
        const double kbar = __ddiv_rn(sum, (double)a.T);
        const double kmin = a.kmin[r], kmax = a.kmax[r];
        double f = 0.0;   // Eq. 3, readings L3 and L7, as in lp_solve
        if (kmax > kmin) {
            f = __ddiv_rn(__dsub_rn(kbar, kmin), __dsub_rn(kmax, kmin));
            f = f < 0.0 ? 0.0 : (f > 1.0 ? 1.0 : f);
        }
        b = __dmul_rn(__dsub_rn(1.0, __dmul_rn(f, a.xi)), qr[0]);
    }
    b = __shfl_sync(0xFFFFFFFFu, b, 0);
    int best = -1;
    double best_c = 0.0;
    for (int g = lane; g < a.G; g += 32) {   // ascending g per lane: strict < keeps the lowest
        const double *S = a.group + ((size_t)r * a.G + g) * a.K;
        double Q = 0.0;
        for (int L = 0; L < a.n; ++L) Q = __dadd_rn(Q, __dmul_rn(S[11 + L], qr[L]));
        if (!(Q >= __dmul_rn(b, S[0]))) continue;
        if (best < 0 || S[4] < best_c) { best = g; best_c = S[4]; }
    }
    // warp argmin of (carbon, g); lanes without a feasible point lose
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const int ob = __shfl_xor_sync(0xFFFFFFFFu, best, d);
        const double oc = __shfl_xor_sync(0xFFFFFFFFu, best_c, d);
        const bool take = ob >= 0 && (best < 0 || oc < best_c || (oc == best_c && ob < best));
        if (take) { best = ob; best_c = oc; }
    }
    if (best < 0) best = 0;
    if (lane == 0) a.choice[r] = best;
    if (lane < a.n) {
        int k[SPROUT_MAX_LEVELS];
        grid_unrank_rt(a.n, a.grid_den, best, k);
        int kl = k[0];
        for (int i = 1; i < SPROUT_MAX_LEVELS; ++i) kl = i == lane ? k[i] : kl;
        a.x[(size_t)r * a.n + lane] = __ddiv_rn((double)kl, (double)a.grid_den);
    }
}

cudaError_t launch_select_static(const SelectArgs &a, cudaStream_t stream, int *launches) {
    select_static_kernel<<<(unsigned)a.R, 32, 0, stream>>>(a);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace sprout
