/*
 * sprout.h -- C ABI of the B200-native Sprout hot path (arXiv 2403.12900).
 *
 * The path, per (region r x carbon-intensity interval t x quality
 * coefficient xi_j) cell:
 *   1. sprout_solve_directives: quality floor q_lb (Eq. 3), the
 *      expected-carbon cost vector c (Eq. 2, with PUE) and
 *      the directive LP  min c.x  s.t. q.x >= q_lb, 0 <= x <= 1, sum x = 1
 *      (Eqs. 4-7), solved exactly by vertex enumeration in fp64;
 *      plus the inverse-CDF thresholds of the solved mix x.
 *   2. sprout_simulate_trace: for every request of the cell's interval, a
 *      counter-based Philox4x32-10 draw selects a directive level from x
 *      (selector (1); opted-out users always L0); its energy,
 *      time and carbon follow Eq. 1 with E, T linear in the
 *      generated tokens; per-cell totals are reduced.
 *   3. sprout_reduce_totals: per (region, xi) and per xi group totals; the
 *      caller then all-reduces them across GPUs (NCCL, torch.distributed).
 * P:<line> cites /root/reference/PAPER.md.  Readings of silent or ambiguous
 * passages (tie-break, rounding order, RNG layout, ...) are DESIGN.md L1-L20.
 *
 * Conventions
 *   - Every array pointer inside the structs is a DEVICE pointer (cudaMalloc
 *     / torch CUDA tensor) owned by the caller, except where a function says
 *     HOST.  The library allocates nothing persistent; its only state is a
 *     thread-local launch counter (sprout_last_launch_count), so calls are
 *     thread-safe and asynchronous on `stream`.
 *   - Host-checkable arguments are validated synchronously before anything
 *     is enqueued; a non-OK status means nothing was launched.
 *   - Data in device arrays is validated on the device, per cell
 *     (cell_status) or per trace (trace_status), without a host sync.
 *   - Cells are indexed cell = (s - first_segment) * n_xi + j with segment
 *     s = r * n_intervals + t (xi innermost).
 */
#ifndef SPROUT_H
#define SPROUT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

struct CUstream_st;                       /* the CUDA runtime's cudaStream_t */
typedef struct CUstream_st *sprout_stream;

typedef enum {
    SPROUT_OK = 0,
    SPROUT_ERR_INVALID_ARGUMENT = 1,  /* bad scalar, NULL required pointer, misalignment, range */
    SPROUT_ERR_INFEASIBLE = 2,        /* sprout_check_cells: some cell infeasible (status 2) */
    SPROUT_ERR_OVERFLOW = 3,          /* sizes whose counts could exceed 2^53 / index ranges */
    SPROUT_ERR_CUDA = 4,              /* a CUDA runtime call or launch failed (incl. no device) */
    SPROUT_ERR_INVALID_CELL = 5       /* sprout_check_cells: some cell had invalid inputs (status 1) */
} sprout_status;

#define SPROUT_MAX_LEVELS 8
#define SPROUT_MAX_CLASSES 4
#define SPROUT_MAX_XI 4096

/* cell_status codes (device, one byte per cell) */
#define SPROUT_CELL_OK 0
#define SPROUT_CELL_INVALID 1     /* xi not in [0,1]; q_i not in [0,1]; NaN/inf; negative k0/e/p; kmax < kmin */
#define SPROUT_CELL_INFEASIBLE 2  /* no feasible vertex (impossible when q_lb <= q0) */

/* trace_status bits (device word, OR-ed) */
#define SPROUT_TRACE_BAD_CLASS   0x1u   /* a request's class (flags bits 1-2) >= n_classes: request skipped */
#define SPROUT_TRACE_BAD_OFFSETS 0x2u   /* seg_offsets not non-decreasing within [0, n_requests]: segment skipped */
#define SPROUT_TRACE_SLOW_PATH   0x100u /* informational: a segment needed the generic (slow) kernel path */
#define SPROUT_TRACE_TOO_LONG    0x4u   /* Oracle scheme: a segment longer than max_segment_requests: skipped */

/* ---------------------------------------------------------------------- */
/* The directive LP over a (region x interval x xi) grid, Eqs. 2-7.        */
typedef struct {
    int32_t n_levels;          /* n: directive levels L0..L(n-1), L0 = no directive; 1..8 */
    int32_t n_regions;         /* R >= 1 */
    int64_t n_intervals;       /* T >= 1 carbon-intensity intervals per region (zero-order hold) */
    int32_t n_xi;              /* X: 1..SPROUT_MAX_XI quality coefficients */
    int32_t profile_per_interval; /* 0: e,p,q are [R][n]; 1: they are [R*T][n] */
    const double *k0;          /* [R*T] carbon intensity, gCO2/kWh */
    const double *k0_min;      /* [R] historical minimum (Table II) */
    const double *k0_max;      /* [R] historical maximum */
    const double *xi;          /* [X] paper xi in [0,1]: allowed quality deviation */
    const double *e;           /* [R|R*T][n] mean energy per request at each level, kWh */
    const double *p;           /* [R|R*T][n] mean processing time per request, s */
    const double *q;           /* [R|R*T][n] preference rate of each level, in [0,1] */
    double k1;                 /* embodied carbon rate CO2_embed / T_life, gCO2/s; >= 0 */
    double pue;                /* power usage effectiveness, >= 1 (reading L2) */
    int64_t first_segment;     /* this call covers segments [first_segment, first_segment + n_segments) */
    int64_t n_segments;        /* of the R*T grid (a rank's shard) */
} sprout_lp_problem;

/* Outputs of sprout_solve_directives, one entry per local cell. */
typedef struct {
    double *x;                 /* [cells][n] the solved mix: probability of each level */
    double *objective;         /* [cells] expected gCO2 per request f(x) (Eq. 2) */
    double *q_lb;              /* [cells] the quality floor b of Eq. 3 */
    uint8_t *vertex;           /* [cells] optimal vertex: i = pure level i; n + k = k-th pair (i<j)
                                  in lexicographic order; 255 = none (invalid/infeasible) */
    uint32_t *threshold;       /* [cells][n-1] inverse-CDF thresholds T_i = min(ceil(cum_i 2^32), 2^32),
                                  2^32 stored saturated as 0xFFFFFFFF; may be NULL iff n == 1 */
    uint8_t *max_level;        /* [cells] first i with T_i = 2^32, else n-1 */
    uint8_t *cell_status;      /* [cells] SPROUT_CELL_* */
} sprout_lp_solution;

/* A rank's slice of the request trace. */
typedef struct {
    int64_t n_requests;        /* local requests held in the buffers */
    uint64_t first_request;    /* global index of local request 0 (Philox counter base); multiple of 8 */
    const int64_t *seg_offsets;/* [n_segments+1] local request offsets of the segments (CSR) */
    const uint16_t *tokens;    /* [n][plane_pitch] generated tokens of each request at each level */
    int64_t plane_pitch;       /* elements; multiple of 8, >= n_requests; tokens 16-byte aligned */
    const uint8_t *flags;      /* [plane_pitch] or NULL: bit0 = opted-out user (always L0),
                                  bits1-2 = model class (cost-model row); 16-byte aligned */
} sprout_trace;

/* Per-request energy/time model and the selection seed (HOST struct, by pointer).
 * E = ef[c][L] + et[c][L]*tok, T = pf[c][L] + pt[c][L]*tok (reading L11). */
typedef struct {
    uint64_t seed;             /* Philox key (lo32, hi32) of the selection draws (reading L10) */
    int32_t n_classes;         /* 1..4 */
    int32_t reserved;
    double ef[SPROUT_MAX_CLASSES][SPROUT_MAX_LEVELS];  /* kWh */
    double et[SPROUT_MAX_CLASSES][SPROUT_MAX_LEVELS];  /* kWh per generated token */
    double pf[SPROUT_MAX_CLASSES][SPROUT_MAX_LEVELS];  /* s */
    double pt[SPROUT_MAX_CLASSES][SPROUT_MAX_LEVELS];  /* s per generated token */
} sprout_cost_model;

/* Outputs of sprout_simulate_trace (all written in full; no pre-zeroing needed). */
typedef struct {
    uint64_t *cnt;             /* [cells][n_classes][n] requests assigned each level */
    uint64_t *tok;             /* [cells][n_classes][n] generated tokens at the assigned level */
    double *energy_kwh;        /* [cells] sum of E over the cell's requests */
    double *time_s;            /* [cells] sum of T */
    double *carbon_g;          /* [cells] sum of Eq. 1 carbon (k0*PUE*E + k1*T) */
    double *quality;           /* [cells] sum of q[level] (reading L15) */
    uint64_t *seg_count;       /* [n_segments][n_classes] requests per segment */
    uint64_t *seg_pinned;      /* [n_segments][n_classes] opted-out requests */
    uint64_t *seg_tok;         /* [n_segments][n_classes][n] sum of tokens at every level (all requests) */
    double *seg_base;          /* [n_segments][4] Base counterfactual (all at L0):
                                  energy, time, carbon, quality */
    uint32_t *trace_status;    /* [1] SPROUT_TRACE_* bits */
} sprout_cell_totals;

/* Harness-only synthetic trace generator (not part of the method). */
typedef struct {
    uint64_t gen_seed;         /* Philox key of the generator (stream 1) */
    uint64_t first_request;    /* global index of local request 0 */
    int64_t n_requests;
    int32_t n_levels;          /* 1..8 */
    int32_t n_classes;         /* 1..4 */
    uint32_t pin_thresh;       /* pinned iff (w3 & 0xFFFFFF) < pin_thresh */
    uint32_t reserved;
    const uint16_t *q0_table;  /* [n_classes][4096] L0 generated-token quantiles */
    const uint16_t *ratio_table; /* [8][256] per-level length ratios, fixed point 2^-16 */
} sprout_trace_generator;

/* ---------------------------------------------------------------------- */

/* Step 1 (a1-a4).  One thread per cell: Eq. 3 floor, Eq. 2 cost vector,
 * vertex enumeration in a fixed order keeping the first strict minimum
 * (pure levels ascending, then pairs lexicographically; reading L6), IEEE
 * fp64 without contraction (reading L7), thresholds.  Writes every field of
 * `solution` for the n_segments*n_xi local cells.  Errors: INVALID_ARGUMENT
 * (n outside [1,8], R/T/X < 1 or X > SPROUT_MAX_XI, shard outside R*T, PUE < 1
 * or NaN, k1 < 0 or NaN, NULL pointers); CUDA on launch failure. */
sprout_status sprout_solve_directives(const sprout_lp_problem *problem,
                                      const sprout_lp_solution *solution,
                                      sprout_stream stream);

/* Bytes of device workspace sprout_simulate_trace needs (0 on invalid args). */
size_t sprout_workspace_bytes(const sprout_lp_problem *problem, const sprout_trace *trace);

/* Step 2 (a5-a8).  Streams the trace once.  Selection draw of global
 * request g: Philox4x32-10, key = (seed lo32, seed hi32), counter =
 * (g>>2 lo32, g>>2 hi32, 0, 0), word g&3 (reading L10); one draw per request
 * shared by all xi cells of its segment.  level = pinned ? 0 :
 * min(#{i <= n-2 : w >= T_i}, max_level).  Cells with cell_status != 0 are
 * skipped (totals 0).  `levels_out` (verify mode, slow) is NULL or
 * [n_xi][plane_pitch]: level of every request for every cell of its
 * segment (0xFF for skipped cells).  Errors: INVALID_ARGUMENT (as above, plus
 * NULL tokens/seg_offsets/outputs, misaligned tokens/flags, pitch, first_request
 * not a multiple of 8, n_classes outside [1,4], workspace too small); OVERFLOW
 * (n_requests >= 2^40); CUDA. */
sprout_status sprout_simulate_trace(const sprout_lp_problem *problem,
                                    const sprout_lp_solution *solution,
                                    const sprout_trace *trace,
                                    const sprout_cost_model *cost,
                                    const sprout_cell_totals *totals,
                                    uint8_t *levels_out,
                                    void *workspace, size_t workspace_bytes,
                                    sprout_stream stream);

/* sprout_simulate_trace with the caller's bound on the distinct non-zero
 * thresholds (breakpoints) of any one segment's valid cells: it sizes the
 * per-warp histograms (more warps per SM when the bound is small).  0 = the
 * bound of LP mixes (<= 2 non-zero levels), min(n_xi*(n-1), n_xi+1).  A
 * segment with more breakpoints than the bound takes the generic path
 * (correct, slower; SPROUT_TRACE_SLOW_PATH).  A STATIC_GRID sweep of step
 * 1/D has at most 2(D-1): the cumulative sums are multiples j/D (reading
 * L18), each rounded up to one of two adjacent integers.  Errors: as
 * sprout_simulate_trace, plus INVALID_ARGUMENT for a negative bound. */
sprout_status sprout_simulate_trace_bounded(const sprout_lp_problem *problem,
                                            const sprout_lp_solution *solution,
                                            const sprout_trace *trace,
                                            const sprout_cost_model *cost,
                                            const sprout_cell_totals *totals,
                                            uint8_t *levels_out, int32_t max_breakpoints,
                                            void *workspace, size_t workspace_bytes,
                                            sprout_stream stream);

/* Number of statistics K per group row: 11 + 2n.  Row layout: 0 requests,
 * 1 opted-out, 2 energy kWh, 3 time s, 4 carbon g, 5 quality, 6-9 Base
 * energy/time/carbon/quality, 10 expected carbon (requests x objective),
 * 11.. requests per level (n), 11+n.. tokens per level (n). */
int32_t sprout_group_stat_count(int32_t n_levels);

/* Bytes of device workspace sprout_reduce_totals needs. */
size_t sprout_reduce_workspace_bytes(const sprout_lp_problem *problem);

/* Step 3 (a9, local part).  group_totals (device, fp64) = [R][X][K] followed
 * by [X][K]; rows of regions outside the shard are 0.  Integer statistics
 * are exact in fp64 (< 2^53).  The caller all-reduces group_totals (SUM)
 * across ranks.  Deterministic (fixed summation order). */
sprout_status sprout_reduce_totals(const sprout_lp_problem *problem,
                                   const sprout_lp_solution *solution,
                                   const sprout_cell_totals *totals,
                                   int32_t n_classes,
                                   double *group_totals,
                                   void *workspace, size_t workspace_bytes,
                                   sprout_stream stream);

/* Blocking helper: worst cell_status over the local cells -> OK,
 * INVALID_CELL or INFEASIBLE.  Synchronises `stream`. */
sprout_status sprout_check_cells(const sprout_lp_problem *problem,
                                 const sprout_lp_solution *solution,
                                 sprout_stream stream);

/* End-to-end call with HOST buffers: copies the problem arrays and the trace
 * from host memory (pinned for full speed) into `device_workspace`, runs
 * steps 1-3 and copies the [R+1][X][K] group totals back into
 * `host_group_totals`; synchronises `stream` before returning.  Every array
 * pointer inside `problem` and `trace` is a HOST pointer here. */
size_t sprout_sweep_workspace_bytes(const sprout_lp_problem *problem, const sprout_trace *trace,
                                    int32_t n_classes);
sprout_status sprout_sweep_host(const sprout_lp_problem *problem, const sprout_trace *trace,
                                const sprout_cost_model *cost, double *host_group_totals,
                                uint32_t *host_trace_status,
                                void *device_workspace, size_t device_workspace_bytes,
                                sprout_stream stream);

/* Harness only: synthetic Llama2-shaped trace (not part of the method).
 * Writes tokens [n][plane_pitch] and (if flags != NULL) flags [plane_pitch]
 * for local requests [0, n_requests). */
sprout_status sprout_generate_trace(const sprout_trace_generator *gen,
                                    uint16_t *tokens, int64_t plane_pitch, uint8_t *flags,
                                    sprout_stream stream);

/* ---------------------------------------------------------------------- */
/* Competing schemes of the paper's evaluation (SURVEY 8(f)
 * NEXT-3).  Base (every request at L0) needs no solve: every
 * simulate call reports it as the per-segment counterfactual (seg_base).
 * The other schemes replace step 1 and reuse steps 2-3 unchanged.          */
#define SPROUT_SCHEME_SPROUT 0       /* the directive LP of Eqs. 4-7 per (segment, xi) cell */
#define SPROUT_SCHEME_CO2_OPT 1      /* always the lowest-carbon level */
#define SPROUT_SCHEME_STATIC_GRID 2  /* the static configurations swept by Sprout_Sta */
#define SPROUT_VERTEX_GRID 254       /* vertex code of a grid point with >= 2 non-zero levels */

/* Step 1 for a scheme.  SPROUT: identical to sprout_solve_directives.
 * CO2_OPT: per cell x = e_m, m = argmin_i c_i of the Eq. 2 cost vector
 *   (ties to the lowest index, reading L17); xi is ignored (may be NULL).
 * STATIC_GRID: cell j of every segment is point j of the simplex grid of
 *   step 1/grid_den (x_i = k_i / grid_den, k_i >= 0 integers summing to
 *   grid_den, ordered by k_0 descending, then k_1 descending, ...; point 0
 *   is pure L0; reading L18); requires n_xi == sprout_static_grid_size(n,
 *   grid_den); xi is ignored (may be NULL).
 * For CO2_OPT and STATIC_GRID there is no quality floor: q_lb holds the
 * mix's expected quality q.x and objective its expected carbon c.x (both
 * summed in level order); vertex = the level of a pure mix, else
 * SPROUT_VERTEX_GRID.  Thresholds and max_level as for SPROUT, so
 * sprout_simulate_trace and sprout_reduce_totals apply unchanged.
 * Errors: as sprout_solve_directives, plus INVALID_ARGUMENT for an unknown
 * scheme, grid_den < 1 or a grid size other than n_xi. */
sprout_status sprout_solve_scheme(const sprout_lp_problem *problem, int32_t scheme, int32_t grid_den,
                                  const sprout_lp_solution *solution, sprout_stream stream);

/* Points of the static grid, C(grid_den + n - 1, n - 1); -1 if n is outside
 * [1,8] or grid_den < 1, or the count exceeds SPROUT_MAX_XI. */
int64_t sprout_static_grid_size(int32_t n_levels, int32_t grid_den);

/* Sprout_Sta choice ("the best static configuration is determined
 * by sweeping the possible static configurations"; reading L18), from the
 * group totals (device, [R+1][G][K], all segments of every region, i.e.
 * after the cross-rank all-reduce) of a STATIC_GRID sweep.  Per region r:
 * floor b_r = Eq. 3 at the region's mean carbon intensity (sum of k0 over
 * its T intervals in index order, / T) with the given xi and q0 = q[r][0];
 * point g is feasible iff  sum_L requests_L(g) * q_L >= b_r * requests(g)
 * (realised quality, level order); choice[r] = the feasible g of least
 * realised carbon (stat 4), ties to the lowest g (point 0, pure L0, is
 * always feasible).  Outputs (device): choice [R] int32, x [R][n] fp64.
 * Requires profile_per_interval == 0 and n_xi == G.  Errors:
 * INVALID_ARGUMENT (as above, xi outside [0,1], NULL pointers); CUDA. */
sprout_status sprout_select_static(const sprout_lp_problem *problem, int32_t grid_den, double xi,
                                   const double *group_totals, int32_t *choice, double *x,
                                   sprout_stream stream);

/* ---------------------------------------------------------------------- */
/* Opportunistic evaluator trigger sweep (Eq. 8; SURVEY 8(f)
 * NEXT-2).  The evaluation server's carbon intensity k2 is the region's CI
 * ("it resides in the same region as the inference server").  For
 * every (region r, urgency beta_b, threshold theta_h) configuration, one
 * sequential scan over the region's T intervals (reading L19):
 *   state: i0 = index of the last evaluation (the trace start counts as one),
 *   factor f = d_b^(i - i0) by repeated multiplication, d_b = exp(-beta_b *
 *   interval_hours) evaluated once on the host (Eq. 8's e^{-beta (t - t0)});
 *   k'(i) = f * k2(i).  Evaluate at i iff (i - i0) * interval_hours >=
 *   grace_hours (condition ii) AND k'(i) < theta_h * k2_max[r] (iii) AND
 *   either k' has a trailing local minimum at i-1 (k'(i-1) < k'(i-2) and
 *   k'(i) > k'(i-1), both samples after i0; condition i) or the last
 *   `fallback` samples after i0 were all below the threshold (Fig. 4(b):
 *   "the increasing evaluation urgency ensures that offline evaluation
 *   always occurs"; 0 disables).  An evaluation at i costs
 *   k2(i) * pue * eval_kwh gCO2 and restarts the state at i0 = i.
 * Output (device, fp64) [R][n_beta][n_theta][4]: evaluations, their carbon
 * (g), the longest time without an evaluation (hours, counting the trace
 * start and end), and the sum of k2 at the evaluations.                    */
#define SPROUT_MAX_EVAL_PARAMS 64
typedef struct {
    int32_t n_regions;         /* R >= 1 */
    int32_t n_beta;            /* 1..SPROUT_MAX_EVAL_PARAMS */
    int64_t n_intervals;       /* T >= 1 */
    double interval_hours;     /* > 0: length of one CI interval */
    const double *k2;          /* [R*T] device: carbon intensity, gCO2/kWh */
    const double *k2_max;      /* [R] device: historical maximum ("50% of the historical maximum") */
    const double *beta;        /* [n_beta] HOST: urgency, 1/hour (>= 0; P:233 uses 0.028) */
    int32_t n_theta;           /* 1..SPROUT_MAX_EVAL_PARAMS */
    int32_t fallback;          /* >= 0 samples (0 = local minimum only) */
    const double *theta;       /* [n_theta] HOST: threshold as a fraction of k2_max (>= 0) */
    double grace_hours;        /* >= 0 */
    double eval_kwh;           /* energy of one evaluation, kWh (>= 0) */
    double pue;                /* >= 1 */
} sprout_evaluator_problem;

/* Errors: INVALID_ARGUMENT (sizes, NULL pointers, NaN/negative parameters);
 * CUDA.  One thread per configuration; deterministic. */
sprout_status sprout_evaluator_sweep(const sprout_evaluator_problem *problem, double *out,
                                     sprout_stream stream);

/* ---------------------------------------------------------------------- */
/* Per-request fp64 accounting (a cross-check of sprout_simulate_trace's
 * closed form).  For every cell: each request's level by
 * the a6 rule straight from the cell's thresholds at its Philox word
 * (reading L10; opted-out requests L0; invalid classes skipped), its
 * Eq. 1 energy E = ef + et*tok, time T = pf + pt*tok (
 * reading L11), carbon k0*PUE*E + k1*T (reading L2) and quality q[level]
 * (reading L15), summed in fp64 per thread in request order and then by a
 * fixed warp-shuffle / block tree -- deterministic.  energy_kwh, time_s,
 * carbon_g, quality: device, [cells] fp64, caller-owned, written for every
 * cell (0 for invalid cells and segments with invalid offsets).  Equal to
 * sprout_simulate_trace's totals within fp64 summation error (the tests use
 * 1e-12 relative).  One CTA per segment; every cell re-reads the segment:
 * a verification mode, not the timed path.  Errors: INVALID_ARGUMENT (as
 * sprout_simulate_trace); CUDA. */
sprout_status sprout_cell_totals_fp64(const sprout_lp_problem *problem, const sprout_lp_solution *solution,
                                      const sprout_trace *trace, const sprout_cost_model *cost, double *energy_kwh,
                                      double *time_s, double *carbon_g, double *quality, sprout_stream stream);

/* ---------------------------------------------------------------------- */
/* Closed-loop profiles (reading L20).  P:183: e and p
 * are "the average energy consumption and processing time for recent
 * requests at each level".  Steps 1-2 as one causal scan per (region, xi)
 * chain: at interval t the profile of level L is the mean Eq. 1 energy and
 * time of the last `window` requests this chain ran at level L (any class;
 * opted-out requests count at L0), or the problem's e/p[r][L] (priors) while
 * none has; with E = ef + et*tok it is computed from the window's per-class
 * request counts n_c and token sums k_c (exact integers) as
 *   e_L = (sum_c (n_c ef[c][L] + k_c et[c][L])) / sum_c n_c   (class order),
 * p_L likewise.  The interval's LP (as sprout_solve_directives) uses it; the
 * interval's requests are then selected and accounted exactly as in
 * sprout_simulate_trace, and pushed in request order into their level's
 * window.  Writes every field of `solution` and every field of `totals`
 * (cells: cnt, tok, energy_kwh, time_s, carbon_g, quality; segments:
 * seg_count, seg_pinned, seg_tok, seg_base -- the same values
 * sprout_simulate_trace gives for the solved thresholds; and trace_status),
 * so sprout_reduce_totals can follow directly.  Invalid offsets (s0 > s1,
 * or past n_requests) flag SPROUT_TRACE_BAD_OFFSETS and the interval is
 * skipped: its cells and segment fields are zero and no request enters a
 * window.  `profile_out` is NULL or (device) [cells][2][n]: the e and p each
 * interval's LP used.  Two passes: one CTA per (region, xi) chain solves the
 * chain's LPs in interval order and, per interval, scans its requests
 * backwards from the interval end only until every level the mix can reach
 * has its last `window` requests (the windows need no more); then the
 * streaming kernel of sprout_simulate_trace accounts every request with the
 * solved thresholds.  `workspace` (device, 256-byte aligned, caller-owned,
 * >= sprout_workspace_bytes) is that pass's; before it, its first 8 bytes
 * per chain hold the chain schedule (an estimate of each chain's time from
 * the LP on the priors, and the launch order that packs the chains into the
 * GPU's resident slots -- scheduling only: no output depends on it).  Requires whole regions
 * (first_segment and n_segments multiples of n_intervals: a rank may take a
 * range of regions; outputs are indexed by local cell), profile_per_interval
 * 0, and 1 <= window <= 4096 with n*window*4 bytes <= 96 KiB.  Errors:
 * INVALID_ARGUMENT (as sprout_simulate_trace, plus the above); CUDA. */
sprout_status sprout_simulate_closed_loop(const sprout_lp_problem *problem, int32_t window,
                                          const sprout_trace *trace, const sprout_cost_model *cost,
                                          const sprout_lp_solution *solution,
                                          const sprout_cell_totals *totals, double *profile_out,
                                          void *workspace, size_t workspace_bytes, sprout_stream stream);

/* ---------------------------------------------------------------------- */
/* NEXT-4: per-request outputs, the latent best level and the
 * head-to-head preference against Base, and the Oracle scheme.
 *
 * Reading L21 (latent best level): the evaluator "identifies the directive
 * level that yields the best response for each request" and q holds
 * the preference rates of those levels.  Synthetic ground truth:
 * request g's latent best level l*(g) is the inverse-CDF level of its
 * segment's q row (the rules a4/a6 with q in place of the mix) at the word
 * of Philox4x32-10 stream 2: key (seed lo, seed hi), counter (g>>2 lo32,
 * g>>2 hi32, 2, 0), word g & 3 (the selection draw is stream 0).
 * Reading L22 (head-to-head vs Base): a request served at L = 0 ties
 * (identical response); otherwise the scheme wins iff l* = L and Base wins
 * iff l* = 0, a third best level ties.  w = (wins + ties/2) / requests and
 * the normalized preference score is w / (1 - w)
 * (sprout_normalized_preference; w = 0.48 -> 0.923). */

/* Per-request outputs of cell column xi_index (one xi value) of a solved
 * (solution) sweep -- the per-request carbon normalised to Base behind the
 * CDF of Fig. eval2.  For every local request r of a valid segment:
 * level_out[r] its level (a6; 0xFF for an invalid class or cell),
 * carbon_out[r] its Eq. 1 carbon at its level and its segment's CI,
 * base_out[r] its carbon at L0 (Base), ratio_out[r] = carbon / base
 * (NaN when invalid), and pref_out[r] (may be NULL) its l*.  Same operation
 * order as the accounting of sprout_simulate_trace per request (no FMA).
 * All arrays device, [n_requests].  Errors: INVALID_ARGUMENT (as
 * sprout_simulate_trace; xi_index outside [0, n_xi); NULL or misaligned
 * outputs); CUDA. */
sprout_status sprout_request_outputs(const sprout_lp_problem *problem, const sprout_lp_solution *solution,
                                     const sprout_trace *trace, const sprout_cost_model *cost, int32_t xi_index,
                                     uint8_t *level_out, double *carbon_out, double *base_out, double *ratio_out,
                                     uint8_t *pref_out, sprout_stream stream);

/* Head-to-head statistics per cell of a solved sweep: stats[cell][0..2] =
 * hits (requests at their latent best level: the realised Eq. 3 left-hand
 * side), wins and losses against Base (reading L22); u64, device,
 * [n_segments * n_xi][3].  Requests with an invalid class, invalid cells and
 * invalid segments count nothing.  n_xi * 12 bytes <= 200 KiB.  Errors as
 * sprout_request_outputs. */
sprout_status sprout_preference_stats(const sprout_lp_problem *problem, const sprout_lp_solution *solution,
                                      const sprout_trace *trace, const sprout_cost_model *cost, uint64_t *stats,
                                      sprout_stream stream);

/* The Oracle scheme ("the inference carbon emission on every
 * generation directive level is known ahead of time for all user prompts,
 * and [it] knows the exact generation quality feedback for future prompts";
 * reading L23).  Per cell (segment, xi): with every request's Eq. 1 carbon at
 * every level and its latent best level l*, each request's level minimises
 * the cell's carbon subject to the realised quality #{L(g) = l*(g)} >=
 * ceil(fl(b * m)), b the cell's Eq. 3 floor and m its valid requests;
 * opted-out requests stay at L0.  The optimum serves every request
 * at its cheapest level (lowest index among ties) and moves the requests
 * with l* != cheapest of smallest extra carbon (ties: lower request index)
 * to l* until the floor is met.  Writes every field of `totals` (cells and
 * segments, as sprout_simulate_trace; E/T/C/Q in its closed form from the
 * integer statistics), stats [cells][3] = (hits, wins, losses) as
 * sprout_preference_stats, and cell_status [cells] (0 ok; 1 invalid cell
 * input; 2 the floor cannot be met even with every candidate moved -- all
 * moved).  Segments longer than max_segment_requests are skipped with
 * SPROUT_TRACE_TOO_LONG (their outputs zero); workspace >=
 * sprout_oracle_scheme_workspace_bytes (256-byte aligned; 32 bytes per
 * request of the longest segment per SM).  Errors: INVALID_ARGUMENT; CUDA. */
size_t sprout_oracle_scheme_workspace_bytes(const sprout_lp_problem *problem, int64_t max_segment_requests);
sprout_status sprout_simulate_oracle_scheme(const sprout_lp_problem *problem, const sprout_trace *trace,
                                            const sprout_cost_model *cost, int64_t max_segment_requests,
                                            const sprout_cell_totals *totals, uint64_t *stats, uint8_t *cell_status,
                                            void *workspace, size_t workspace_bytes, sprout_stream stream);

/* P:377's normalized preference score w / (1 - w) of a head-to-head win
 * fraction w in [0, 1] (+inf at w = 1; NaN for w < 0 or NaN).  Host. */
double sprout_normalized_preference(double w);

/* NEXT-1's q update per evaluation epoch (reading L24).  An evaluation
 * offers "a timely update to the q^T vector": it samples 500 requests
 * and records the best level of each.  For ONE evaluator
 * configuration (ev: n_beta = n_theta = 1; k2 = the CI per region and
 * interval, as in sprout_evaluator_sweep) the evaluations fire where the
 * trigger scan of Eq. 8 fires (reading L19; t = 0 counts).  An evaluation
 * at interval t samples the last `sample` requests of the region before
 * interval t (all if fewer; none: q unchanged) and sets q_i = #{l* = i} /
 * #sampled, l* the latent best level (reading L21) against the region's row
 * of problem->q (the truth); that q holds from t until the next evaluation.
 * problem must be the whole sweep (first_segment 0, n_segments = R*T,
 * profile_per_interval 0).  Outputs (device): q_out [R*T][n] fp64 -- the q
 * of every interval's epoch, e.g. for sprout_simulate_closed_loop_q --, and
 * fired_out [R*T] u8 (1 at an evaluation).  One CTA per region.  Errors:
 * INVALID_ARGUMENT; CUDA. */
sprout_status sprout_evaluation_q(const sprout_evaluator_problem *ev, const sprout_lp_problem *problem,
                                  const sprout_trace *trace, const sprout_cost_model *cost, int32_t sample,
                                  double *q_out, uint8_t *fired_out, sprout_stream stream);

/* sprout_simulate_closed_loop with the LP's q taken per interval from
 * q_interval [R*T][n] (device; global segment index; NULL: problem->q per
 * region) -- the closed loop with the q of each evaluation epoch (NEXT-1,
 * reading L24).  Quality sums use the same rows. */
sprout_status sprout_simulate_closed_loop_q(const sprout_lp_problem *problem, int32_t window, const double *q_interval,
                                            const sprout_trace *trace, const sprout_cost_model *cost,
                                            const sprout_lp_solution *solution, const sprout_cell_totals *totals,
                                            double *profile_out, void *workspace, size_t workspace_bytes,
                                            sprout_stream stream);

/* Number of kernel launches (not memsets) the last successful call of each
 * entry point on this thread enqueued -- for launch accounting in benches. */
int32_t sprout_last_launch_count(void);

const char *sprout_status_string(sprout_status status);

#ifdef __cplusplus
}
#endif
#endif /* SPROUT_H */
