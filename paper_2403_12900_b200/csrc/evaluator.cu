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

namespace sprout {

// NEXT-1's q update per evaluation epoch (reading L24): one CTA per region.
// Thread 0 runs the region's trigger scan (Eq. 8, reading L19: the state and
// rules of evaluator_kernel, t = 0 an evaluation) and marks the evaluations;
// then, per evaluation with requests before it, the CTA counts the latent
// best levels (Philox stream 2 against the region's q row, reading L21) of
// the last `sample` requests before the interval and writes the rates; a
// parallel pass copies every interval's epoch q (the latest evaluation with
// samples at or before it; q_true before any).
constexpr int kEqThreads = 256;

template <int N>
__global__ void __launch_bounds__(kEqThreads) evaluation_q_kernel(const __grid_constant__ EvalQArgs a) {
    const int r = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t T = a.T, s_base = (int64_t)r * T;
    const double *k2 = a.k2 + s_base;
    const double *qt = a.q + (int64_t)r * N;
    uint8_t *fired = a.fired + s_base;
    double *q_out = a.q_out + s_base * N;
    if (tid == 0) {
        const double thr = __dmul_rn(a.theta, a.k2_max[r]);
        int64_t i0 = 0, below = 0;
        double f = 1.0, kp1 = k2[0], kp2 = 0.0;
        fired[0] = 1;
        for (int64_t i = 1; i < T; ++i) {
            const double k = k2[i];
            f = __dmul_rn(f, a.decay);
            const double kp = __dmul_rn(f, k);
            const bool under = kp < thr;
            below = under ? below + 1 : 0;
            const int64_t since = i - i0;
            const bool local_min = since >= 2 && kp1 < kp2 && kp > kp1;
            const bool fire = since >= a.grace_samples && under && (local_min || (a.F > 0 && below >= a.F));
            kp2 = kp1;
            kp1 = fire ? k : kp;
            i0 = fire ? i : i0;
            f = fire ? 1.0 : f;
            below = fire ? 0 : below;
            fired[i] = fire ? 1 : 0;
        }
    }
    __syncthreads();
    // thresholds of the true q (a4 with q as the mix)
    uint32_t Tq[N > 1 ? N - 1 : 1];
    int mlq = N - 1;
    {
        double cum = 0.0;
        bool found = false;
#pragma unroll
        for (int i = 0; i + 1 < N; ++i) {
            cum = __dadd_rn(cum, qt[i]);
            const double cl = ceil(__dmul_rn(cum, 4294967296.0));
            if (cl >= 4294967296.0) { Tq[i] = 0xFFFFFFFFu; if (!found) { mlq = i; found = true; } }
            else Tq[i] = (uint32_t)(uint64_t)cl;
        }
    }
    __shared__ uint32_t cnt_s[kEqThreads / 32][N];
    const int64_t region0 = a.seg_offsets[s_base];
    for (int64_t t = 0; t < T; ++t) {
        if (!fired[t]) continue;   // uniform: every thread reads the same flag
        const int64_t end = a.seg_offsets[s_base + t];
        const int64_t begin = end - a.sample > region0 ? end - a.sample : region0;
        if (end <= begin) continue;
        uint32_t c[N];
#pragma unroll
        for (int L = 0; L < N; ++L) c[L] = 0u;
        for (int64_t rq = begin + tid; rq < end; rq += kEqThreads) {
            const uint64_t g = a.first_request + (uint64_t)rq;
            const Philox4 d = philox4x32_10_rk((uint32_t)(g >> 2), (uint32_t)(g >> 34), 2u, 0u, a.rk0, a.rk1);
            const uint32_t k3 = (uint32_t)(g & 3u);
            const uint32_t w = k3 == 0 ? d.v[0] : k3 == 1 ? d.v[1] : k3 == 2 ? d.v[2] : d.v[3];
            int L = 0;
#pragma unroll
            for (int i = 0; i + 1 < N; ++i) L += (w >= Tq[i]) ? 1 : 0;
            L = L < mlq ? L : mlq;
#pragma unroll
            for (int LL = 0; LL < N; ++LL) c[LL] += LL == L ? 1u : 0u;
        }
#pragma unroll
        for (int L = 0; L < N; ++L) {
            const uint32_t v = __reduce_add_sync(0xFFFFFFFFu, c[L]);
            if (lane == 0) cnt_s[warp][L] = v;
        }
        __syncthreads();
        if (tid < N) {
            uint32_t v = 0u;
            for (int w2 = 0; w2 < kEqThreads / 32; ++w2) v += cnt_s[w2][tid];
            q_out[t * N + tid] = __ddiv_rn((double)v, (double)(end - begin));
        }
        __syncthreads();
    }
    // every interval's epoch q: the latest evaluation with samples at or before it
    for (int64_t t = tid; t < T; t += kEqThreads) {
        int64_t e = t;
        for (; e >= 0; --e) {
            if (!fired[e]) continue;
            const int64_t end = a.seg_offsets[s_base + e];
            if (end > region0) break;   // (an evaluation without requests before it keeps the previous q)
        }
        if (e == t) continue;           // written above
#pragma unroll
        for (int L = 0; L < N; ++L) q_out[t * N + L] = e >= 0 ? q_out[e * N + L] : qt[L];
    }
}

cudaError_t launch_evaluation_q(EvalQArgs &a, cudaStream_t stream, int *launches) {
    if (a.R == 0 || a.T == 0) return cudaSuccess;
    uint32_t k0 = (uint32_t)a.seed, k1 = (uint32_t)(a.seed >> 32);
    for (int r = 0; r < 10; ++r) { a.rk0[r] = k0; a.rk1[r] = k1; k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
#define EQ_CASE(NN) case NN: evaluation_q_kernel<NN><<<(unsigned)a.R, kEqThreads, 0, stream>>>(a); break;
    switch (a.n) {
        EQ_CASE(1) EQ_CASE(2) EQ_CASE(3) EQ_CASE(4) EQ_CASE(5) EQ_CASE(6) EQ_CASE(7) EQ_CASE(8)
        default: return cudaErrorInvalidValue;
    }
#undef EQ_CASE
    ++*launches;
    return cudaGetLastError();
}

}  // namespace sprout
