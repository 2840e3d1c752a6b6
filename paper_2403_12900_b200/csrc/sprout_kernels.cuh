// sprout_kernels.cuh -- kernel argument blocks and launchers (host <-> device).
#pragma once
#include <cstdint>
#include <cstddef>
#include <cuda_runtime.h>
#include "sprout_device.cuh"

namespace sprout {

// bin lookup table: 2^10 buckets (64-bit entries) over the range of the keys; an entry holds
// the bucket's single key and the histogram row offset of the bin at the bucket start
// (see trace_sim.cu build_lut)
#ifndef SPROUT_LUT_BITS
#define SPROUT_LUT_BITS 10
#endif
constexpr int kLutBits = SPROUT_LUT_BITS;
constexpr int kLutBuckets = 1 << kLutBits;
constexpr int kLutMinKeys = 8;      // fewer keys: level-synchronous binary search
constexpr int kLutMaxKeys = 511;    // larger key sets use the binary search
constexpr int kLutMinRequests = 4096;  // shorter segments do not amortise the table build

// Unsigned 32-bit division by a runtime-constant divisor d >= 1 via a
// precomputed multiplier (Granlund-Montgomery, round-up variant):
// q = (t + ((n - t) >> 1)) >> (l - 1), t = umulhi(m, n); exact for all n < 2^32.
struct FastDiv {
    uint32_t d, m, l;
    __host__ __device__ FastDiv() : d(1), m(0), l(0) {}
    __host__ explicit FastDiv(uint32_t div) : d(div) {
        l = 0;
        while (l < 32 && (1ull << l) < div) ++l;
        m = (uint32_t)(((1ull << 32) * ((1ull << l) - div)) / div + 1);
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        if (l == 0) return n;
        const uint32_t t = __umulhi(m, n);
        return (t + ((n - t) >> 1)) >> (l - 1);
    }
};

struct LpArgs {
    int n, X;
    int64_t T, first_segment, n_segments;
    int profile_per_interval;
    const double *k0, *kmin, *kmax, *xi, *e, *p, *q;
    double k1, pue;
    double *x, *objective, *q_lb;
    uint8_t *vertex;
    uint32_t *threshold;
    uint8_t *max_level, *cell_status;
    FastDiv div_x, div_t;      // by X and by T (used when the cell and segment indices fit in 32 bits)
    int small;                 // 1: n_cells and first_segment + n_segments < 2^32
    int scheme;                // SPROUT_SCHEME_* (0 = the Sprout LP)
    int grid_den;              // D of the static grid (scheme 2)
};

struct ClosedArgs {             // closed-loop profiles (closed_loop.cu)
    int n, R, X, NC, W;
    int r0, R_local;           // regions [r0, r0 + R_local) of this call (whole regions)
    int n_groups;              // CTAs per region: chain groups of G xi values (set by the launcher)
    int64_t T, first_segment, n_requests;
    const double *k0, *kmin, *kmax, *xi, *e, *p, *q;   // e, p: priors [R][n]
    const double *q_seg;       // NULL or [R*T][n]: q per interval (evaluation epochs), else q[R][n]
    double k1, pue;
    uint32_t rk0[10], rk1[10];
    CostConst cost;
    uint64_t first_request;
    const int64_t *seg_offsets;
    const uint16_t *tokens;
    int64_t pitch;
    const uint8_t *flags;
    double *x, *objective, *q_lb, *profile;            // profile may be NULL: [cells][2][n]
    uint8_t *vertex, *cell_status, *max_level;
    uint32_t *threshold;
    uint64_t *cnt, *tok;
    double *energy, *time_s, *carbon, *quality;
    uint64_t *seg_count, *seg_pinned, *seg_tok;
    double *seg_base;
    uint32_t *trace_status;
    float *chain_cost;         // scheduling scratch (NULL: chains in index order): [chains] estimates,
    int *chain_order;          // then [chains] chain ids, longest estimate first
};

struct N4Args {                 // NEXT-4 kernels (next4.cu)
    int n, X, NC;
    int64_t T, first_segment, n_segments;
    int profile_per_interval;
    const double *k0, *q;
    double k1, pue;
    const uint32_t *threshold;
    const uint8_t *max_level, *cell_status;
    int64_t n_requests;
    uint64_t first_request;
    const int64_t *seg_offsets;
    const uint16_t *tokens;
    int64_t pitch;
    const uint8_t *flags;
    uint64_t seed;
    uint32_t rk0[10], rk1[10];
    CostConst cost;
    int column;                // request outputs: the xi column
    uint8_t *level_out, *pref_out;
    double *carbon_out, *base_out, *ratio_out;
    uint64_t *stats;           // [cells][3] hits, wins, losses
    // the Oracle scheme (oracle_scheme_kernel)
    const double *xi, *kmin, *kmax;
    int64_t cap;               // max requests per segment (scratch per CTA)
    uint8_t *scratch;          // [grid][32 * cap] bytes
    uint8_t *cell_status_out;
    uint64_t *cnt, *tok;
    double *energy, *time_s, *carbon, *quality;
    uint64_t *seg_count, *seg_pinned, *seg_tok;
    double *seg_base;
    uint32_t *trace_status;
    uint32_t *queue;
};

struct EvalArgs {               // evaluator trigger sweep (evaluator.cu)
    int R, B, H, F;
    int grace_samples;         // least s >= 0 with s * dt >= grace (fp64, as the definition reads)
    int64_t T;
    double dt, grace, eval_kwh, pue;
    const double *k2, *k2_max;
    double decay[SPROUT_MAX_EVAL_PARAMS];   // exp(-beta_b * dt), host-evaluated
    double theta[SPROUT_MAX_EVAL_PARAMS];
    double *out;               // [R][B][H][4]
};

struct EvalQArgs {              // q per evaluation epoch (evaluator.cu)
    int R, n, F, sample;
    int64_t T, grace_samples;
    double decay, theta;       // exp(-beta * dt) (host), theta as a fraction of k2_max
    const double *k2, *k2_max, *q;   // q: true rows [R][n]
    const int64_t *seg_offsets;      // [R*T+1] local
    uint64_t first_request, seed;
    uint32_t rk0[10], rk1[10];
    double *q_out;             // [R*T][n]
    uint8_t *fired;            // [R*T]
};

struct SelectArgs {            // Sprout_Sta choice per region (schemes.cu)
    int n, R, G, K, grid_den;
    int64_t T;
    const double *k0, *kmin, *kmax, *q;
    double xi;
    const double *group;       // [R+1][G][K]
    int32_t *choice;           // [R]
    double *x;                 // [R][n]
};

// Simulation plan shared by the prep and the streaming kernels.
struct SimPlan {
    int n, X, NC;
    int kcap;          // max distinct breakpoints per segment on the fast path; -1 = all slow
    int nb;            // bins per class in the warp histograms: kcap+1 draw bins, a total slot, the pinned bin
    int nw;            // 32-bit histogram words per entry = ceil((n+1)/2)
    int kp;            // key slots per segment in shared memory (power of two >= kcap+1)
    int lut;           // bucket lookup table in use (kcap in [kLutMinKeys, kLutMaxKeys])
    int warps_per_cta;
    size_t warp_smem;  // bytes of shared memory per warp
    int ctas;          // persistent grid size
    int sort_cap;      // power of two >= X*(n-1) (prep sort buffer), 0 if none
};

struct SimArgs {
    // problem / shard
    int n, X, NC;
    int64_t T, first_segment, n_segments;
    int profile_per_interval;
    const double *k0, *q;      // q rows for the quality sums
    double k1, pue;
    // solution
    const uint32_t *threshold;
    const uint8_t *max_level, *cell_status;
    // trace
    int64_t n_requests;
    uint64_t first_request;
    const int64_t *seg_offsets;
    const uint16_t *tokens;
    int64_t pitch;
    const uint8_t *flags;
    uint64_t seed;
    // outputs
    uint64_t *cnt, *tok;
    double *energy, *time_s, *carbon, *quality;
    uint64_t *seg_count, *seg_pinned, *seg_tok;
    double *seg_base;
    uint32_t *trace_status;
    uint8_t *levels_out;
    uint8_t *bins_out;         // verify mode: every request's histogram bin as the streaming kernel found it
    int bins_ready;            // bins_out was written by the streaming kernel (levels_kernel reads it)
    // workspace
    uint32_t *queue;           // work counter
    int32_t *seg_meta;         // [n_segments] K, -1 slow, -2 bad offsets
    uint32_t *seg_keys;        // [n_segments][kcap] sorted distinct breakpoints minus one
    uint16_t *seg_bnd;         // [n_segments][X][n-1] first bin of each level >= 1
    // plan
    int kcap, nb, nw, kp, sort_cap;
    int lut;                   // 1: per-warp bucket table (kLutBuckets entries) for big segments
    size_t warp_smem;
    uint32_t rk0[10], rk1[10]; // Philox round keys of the selection seed
    // trace_wide_kernel: Philox rounds 0-2 of a counter (lo, H, 0, 0) whose high
    // word H is constant over the launch (see trace_sim.cu philox_lo)
    uint32_t ph_a, ph_blo, ph_d, ph_e;
    unsigned long long *wide_scratch;   // [warps][kcap+1][4] 64-bit spill rows
    int wide;                  // 1: the launch runs trace_wide_kernel
    FastDiv div_nt;            // by n - 1 (thresholds per cell)
    FastDiv div_t;             // by T (region of a segment), valid when T < 2^32
    int seg_batch;             // segments per queue ticket
    CostConst cost;
};

struct ReduceArgs {
    int n, X, NC, R, K;
    int64_t T, first_segment, n_segments;
    int64_t r_lo, r_hi;        // regions touched by the shard
    int chunk, n_chunks;       // intervals per stage-1 block
    const uint8_t *cell_status;
    const double *objective;
    const uint64_t *cnt, *tok;
    const double *energy, *time_s, *carbon, *quality;
    const uint64_t *seg_count, *seg_pinned;
    const double *seg_base;
    double *partials;          // [r_hi-r_lo][n_chunks][X][K]
    double *out;               // [R+1][X][K]
};

struct GenArgs {
    uint64_t gen_seed, first_request;
    int64_t n_requests, pitch;
    int n, NC;
    uint32_t pin_thresh;
    const uint16_t *q0_table, *ratio_table;
    uint16_t *tokens;
    uint8_t *flags;
};

struct F64Args {                // per-request fp64 accounting mode (fp64_check.cu)
    int n, X, NC;
    int64_t T, first_segment, n_segments;
    int profile_per_interval;
    const double *k0, *q;
    double k1, pue;
    const uint32_t *threshold;
    const uint8_t *max_level, *cell_status;
    int64_t n_requests;
    uint64_t first_request;
    const int64_t *seg_offsets;
    const uint16_t *tokens;
    int64_t pitch;
    const uint8_t *flags;
    uint32_t rk0[10], rk1[10];
    CostConst cost;
    double *energy, *time_s, *carbon, *quality;
};

cudaError_t launch_fp64_cells(const F64Args &a, cudaStream_t stream, int *launches);
cudaError_t launch_lp_solve(const LpArgs &a, cudaStream_t stream, int *launches);
bool make_sim_plan(int n, int X, int NC, SimPlan *plan, int max_keys = 0);
size_t sim_workspace_bytes(const SimPlan &plan, int64_t n_segments);
cudaError_t launch_simulate(SimArgs &a, const SimPlan &plan, void *ws, cudaStream_t stream, int *launches);
bool trace_x1_supported(int n, int X, int NC);
cudaError_t launch_trace_x1(SimArgs &a, cudaStream_t stream);
size_t reduce_workspace_bytes(int n, int X, int R, int64_t T, int64_t first_segment, int64_t n_segments);
cudaError_t launch_reduce(ReduceArgs &a, void *ws, cudaStream_t stream, int *launches);
cudaError_t launch_generate(const GenArgs &a, cudaStream_t stream, int *launches);
cudaError_t launch_evaluator(const EvalArgs &a, cudaStream_t stream, int *launches);
cudaError_t launch_closed_loop(ClosedArgs &a, cudaStream_t stream, int *launches);
cudaError_t launch_request_outputs(N4Args &a, cudaStream_t stream, int *launches);
cudaError_t launch_evaluation_q(EvalQArgs &a, cudaStream_t stream, int *launches);
cudaError_t launch_pref_stats(N4Args &a, cudaStream_t stream, int *launches);
cudaError_t launch_oracle_scheme(N4Args &a, cudaStream_t stream, int *launches);
size_t oracle_scheme_workspace_bytes(int64_t cap);
cudaError_t launch_select_static(const SelectArgs &a, cudaStream_t stream, int *launches);
cudaError_t launch_check_cells(const uint8_t *status, int64_t n_cells, uint32_t *out, cudaStream_t stream, int *launches);

}  // namespace sprout
