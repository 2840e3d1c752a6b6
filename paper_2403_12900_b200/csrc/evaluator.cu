// evaluator.cu -- the opportunistic evaluator trigger sweep (P:218-235,
// Eq. 8; reading L19): one thread per (region, beta, theta) configuration
// scans the region's carbon-intensity intervals in order.  The decay factor
// d = exp(-beta * interval) comes from the host (one libm call per beta);
// on the device every operation is an explicit __d*_rn multiply or a
// comparison, so the decisions are bit-reproducible against the oracle.
#include "sprout_device.cuh"
#include "sprout_kernels.cuh"

namespace sprout {

__global__ void __launch_bounds__(128) evaluator_kernel(const __grid_constant__ EvalArgs a) {
    const int64_t cfg = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t n_cfg = (int64_t)a.R * a.B * a.H;
    if (cfg >= n_cfg) return;
    const int h = (int)(cfg % a.H), b = (int)((cfg / a.H) % a.B), r = (int)(cfg / ((int64_t)a.H * a.B));
    const double *k2 = a.k2 + (int64_t)r * a.T;
    const double d = a.decay[b];
    const double thr = __dmul_rn(a.theta[h], a.k2_max[r]);
    // the scan is a dependent chain (every decision resets the state), so it
    // is kept short: 32-bit indices, the grace test as an integer compare
    // (a.grace_samples = the least s with s * dt >= grace, host-computed),
    // branch-free state updates, and the loads taken off the chain (8 ahead)
    int i0 = 0, below = 0, n_eval = 0, max_gap = 0;
    double f = 1.0;                      // d^(i - i0)
    double kp1 = __ldg(k2), kp2 = 0.0;   // k'(i-1), k'(i-2) under the current t0 (k'(i0) = k2(i0))
    double carbon = 0.0, sum_k2 = 0.0;
    const int T = (int)a.T;
    constexpr int U = 8;
    double nxt[U];
#pragma unroll
    for (int u = 0; u < U; ++u) nxt[u] = (1 + u < T) ? __ldg(k2 + 1 + u) : 0.0;
    for (int ib = 1; ib < T; ib += U) {
        double cur[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            cur[u] = nxt[u];
            const int j = ib + U + u;
            nxt[u] = j < T ? __ldg(k2 + j) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = ib + u;
            if (i >= T) break;
            const double k = cur[u];
            f = __dmul_rn(f, d);
            const double kp = __dmul_rn(f, k);
            const bool under = kp < thr;
            below = under ? below + 1 : 0;
            const int since = i - i0;
            const bool local_min = since >= 2 && kp1 < kp2 && kp > kp1;   // samples i-2 >= i0
            const bool fire = since >= a.grace_samples && under && (local_min || (a.F > 0 && below >= a.F));
            kp2 = kp1;
            kp1 = fire ? k : kp;            // k'(i) under the new t0 after an evaluation
            if (fire) {
                carbon = __dadd_rn(carbon, __dmul_rn(__dmul_rn(k, a.pue), a.eval_kwh));
                sum_k2 = __dadd_rn(sum_k2, k);
            }
            n_eval += fire ? 1 : 0;
            max_gap = (fire && since > max_gap) ? since : max_gap;
            i0 = fire ? i : i0;
            f = fire ? 1.0 : f;
            below = fire ? 0 : below;
        }
    }
    max_gap = (T - i0) > max_gap ? (T - i0) : max_gap;
    double *o = a.out + cfg * 4;
    o[0] = (double)n_eval;
    o[1] = carbon;
    o[2] = __dmul_rn((double)max_gap, a.dt);
    o[3] = sum_k2;
}

cudaError_t launch_evaluator(const EvalArgs &a, cudaStream_t stream, int *launches) {
    const int64_t n_cfg = (int64_t)a.R * a.B * a.H;
    if (n_cfg == 0) return cudaSuccess;
    evaluator_kernel<<<(unsigned)((n_cfg + 127) / 128), 128, 0, stream>>>(a);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace sprout
