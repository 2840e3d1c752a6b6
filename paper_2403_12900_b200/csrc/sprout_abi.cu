// sprout_abi.cu -- the extern "C" boundary declared in include/sprout.h:
// synchronous host-side validation, then asynchronous kernel launches on the
// caller's stream.  No allocation, no global state (the launch counter is a
// thread-local diagnostic).
#include <cmath>
#include <cstring>
#include <cuda_runtime.h>
#include "sprout.h"
#include "sprout_kernels.cuh"

using namespace sprout;

static thread_local int g_last_launches = 0;

static bool aligned(const void *p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

static sprout_status validate_problem(const sprout_lp_problem *P) {
    if (!P) return SPROUT_ERR_INVALID_ARGUMENT;
    if (P->n_levels < 1 || P->n_levels > SPROUT_MAX_LEVELS) return SPROUT_ERR_INVALID_ARGUMENT;
    if (P->n_regions < 1 || P->n_intervals < 1 || P->n_xi < 1 || P->n_xi > SPROUT_MAX_XI)
        return SPROUT_ERR_INVALID_ARGUMENT;
    if (P->profile_per_interval != 0 && P->profile_per_interval != 1) return SPROUT_ERR_INVALID_ARGUMENT;
    if (!(P->pue >= 1.0) || !std::isfinite(P->pue)) return SPROUT_ERR_INVALID_ARGUMENT;
    if (!(P->k1 >= 0.0) || !std::isfinite(P->k1)) return SPROUT_ERR_INVALID_ARGUMENT;
    if ((double)P->n_regions * (double)P->n_intervals > 9.0e15) return SPROUT_ERR_OVERFLOW;
    const int64_t S = (int64_t)P->n_regions * P->n_intervals;
    if (P->first_segment < 0 || P->n_segments < 0 || P->first_segment + P->n_segments > S)
        return SPROUT_ERR_INVALID_ARGUMENT;
    if ((double)P->n_segments * P->n_xi > 4.0e12) return SPROUT_ERR_OVERFLOW;
    if (!P->k0 || !P->k0_min || !P->k0_max || !P->xi || !P->e || !P->p || !P->q) return SPROUT_ERR_INVALID_ARGUMENT;
    return SPROUT_OK;
}

static sprout_status validate_solution(const sprout_lp_problem *P, const sprout_lp_solution *X) {
    if (!X) return SPROUT_ERR_INVALID_ARGUMENT;
    if (P->n_segments == 0) return SPROUT_OK;
    if (!X->x || !X->objective || !X->q_lb || !X->vertex || !X->max_level || !X->cell_status)
        return SPROUT_ERR_INVALID_ARGUMENT;
    if (P->n_levels > 1 && !X->threshold) return SPROUT_ERR_INVALID_ARGUMENT;
    if (!aligned(X->x, 8) || !aligned(X->objective, 8) || !aligned(X->q_lb, 8) ||
        (X->threshold && !aligned(X->threshold, 4)))
        return SPROUT_ERR_INVALID_ARGUMENT;
    return SPROUT_OK;
}

static sprout_status validate_trace(const sprout_lp_problem *P, const sprout_trace *T) {
    if (!T) return SPROUT_ERR_INVALID_ARGUMENT;
    if (T->n_requests < 0) return SPROUT_ERR_INVALID_ARGUMENT;
    if (T->n_requests >= ((int64_t)1 << 40)) return SPROUT_ERR_OVERFLOW;
    if (!T->seg_offsets) return SPROUT_ERR_INVALID_ARGUMENT;
    if (T->first_request % 8 != 0) return SPROUT_ERR_INVALID_ARGUMENT;
    if (T->plane_pitch < T->n_requests || T->plane_pitch % 8 != 0) return SPROUT_ERR_INVALID_ARGUMENT;
    if (T->plane_pitch > 0 && (!T->tokens || !aligned(T->tokens, 16))) return SPROUT_ERR_INVALID_ARGUMENT;
    if (T->flags && !aligned(T->flags, 16)) return SPROUT_ERR_INVALID_ARGUMENT;
    if (!aligned(T->seg_offsets, 8)) return SPROUT_ERR_INVALID_ARGUMENT;
    (void)P;
    return SPROUT_OK;
}

static sprout_status validate_totals(const sprout_lp_problem *P, const sprout_cell_totals *C) {
    if (!C) return SPROUT_ERR_INVALID_ARGUMENT;
    if (!C->trace_status) return SPROUT_ERR_INVALID_ARGUMENT;
    if (P->n_segments == 0) return SPROUT_OK;
    if (!C->cnt || !C->tok || !C->energy_kwh || !C->time_s || !C->carbon_g || !C->quality || !C->seg_count ||
        !C->seg_pinned || !C->seg_tok || !C->seg_base)
        return SPROUT_ERR_INVALID_ARGUMENT;
    if (!aligned(C->cnt, 8) || !aligned(C->tok, 8) || !aligned(C->energy_kwh, 8) || !aligned(C->seg_count, 8))
        return SPROUT_ERR_INVALID_ARGUMENT;
    return SPROUT_OK;
}

static sprout_status validate_cost(const sprout_cost_model *M) {
    if (!M) return SPROUT_ERR_INVALID_ARGUMENT;
    if (M->n_classes < 1 || M->n_classes > SPROUT_MAX_CLASSES) return SPROUT_ERR_INVALID_ARGUMENT;
    return SPROUT_OK;
}

static sprout_status cuda_status(cudaError_t e) { return e == cudaSuccess ? SPROUT_OK : SPROUT_ERR_CUDA; }

static LpArgs lp_args(const sprout_lp_problem *P, const sprout_lp_solution *X) {
    LpArgs a{};
    a.n = P->n_levels; a.X = P->n_xi; a.T = P->n_intervals;
    a.first_segment = P->first_segment; a.n_segments = P->n_segments;
    a.profile_per_interval = P->profile_per_interval;
    a.k0 = P->k0; a.kmin = P->k0_min; a.kmax = P->k0_max; a.xi = P->xi;
    a.e = P->e; a.p = P->p; a.q = P->q; a.k1 = P->k1; a.pue = P->pue;
    a.x = X->x; a.objective = X->objective; a.q_lb = X->q_lb; a.vertex = X->vertex;
    a.threshold = X->threshold; a.max_level = X->max_level; a.cell_status = X->cell_status;
    return a;
}

extern "C" {

sprout_status sprout_solve_directives(const sprout_lp_problem *problem, const sprout_lp_solution *solution,
                                      sprout_stream stream) {
    sprout_status st = validate_problem(problem);
    if (st != SPROUT_OK) return st;
    st = validate_solution(problem, solution);
    if (st != SPROUT_OK) return st;
    int launches = 0;
    const LpArgs a = lp_args(problem, solution);
    st = cuda_status(launch_lp_solve(a, reinterpret_cast<cudaStream_t>(stream), &launches));
    if (st == SPROUT_OK) g_last_launches = launches;
    return st;
}

int64_t sprout_static_grid_size(int32_t n_levels, int32_t grid_den) {
    if (n_levels < 1 || n_levels > SPROUT_MAX_LEVELS || grid_den < 1) return -1;
    int64_t c = 1;   // C(grid_den + n - 1, n - 1), stopping once past SPROUT_MAX_XI
    for (int i = 1; i < n_levels; ++i) {
        c = c * (grid_den + i) / i;
        if (c > SPROUT_MAX_XI) return -1;
    }
    return c;
}

sprout_status sprout_solve_scheme(const sprout_lp_problem *problem, int32_t scheme, int32_t grid_den,
                                  const sprout_lp_solution *solution, sprout_stream stream) {
    if (scheme == SPROUT_SCHEME_SPROUT) return sprout_solve_directives(problem, solution, stream);
    if (!problem || (scheme != SPROUT_SCHEME_CO2_OPT && scheme != SPROUT_SCHEME_STATIC_GRID))
        return SPROUT_ERR_INVALID_ARGUMENT;
    if (scheme == SPROUT_SCHEME_STATIC_GRID &&
        (grid_den < 1 || sprout_static_grid_size(problem->n_levels, grid_den) != (int64_t)problem->n_xi))
        return SPROUT_ERR_INVALID_ARGUMENT;
    sprout_lp_problem P = *problem;
    static const double zero = 0.0;
    if (!P.xi) P.xi = &zero;   // not read by these schemes; keeps the shared validation
    sprout_status st = validate_problem(&P);
    if (st != SPROUT_OK) return st;
    st = validate_solution(&P, solution);
    if (st != SPROUT_OK) return st;
    int launches = 0;
    LpArgs a = lp_args(&P, solution);
    a.scheme = scheme;
    a.grid_den = scheme == SPROUT_SCHEME_STATIC_GRID ? grid_den : 0;
    st = cuda_status(launch_lp_solve(a, reinterpret_cast<cudaStream_t>(stream), &launches));
    if (st == SPROUT_OK) g_last_launches = launches;
    return st;
}

sprout_status sprout_select_static(const sprout_lp_problem *problem, int32_t grid_den, double xi,
                                   const double *group_totals, int32_t *choice, double *x, sprout_stream stream) {
    if (!problem || !group_totals || !choice || !x) return SPROUT_ERR_INVALID_ARGUMENT;
    if (!(xi >= 0.0 && xi <= 1.0)) return SPROUT_ERR_INVALID_ARGUMENT;
    if (problem->profile_per_interval != 0) return SPROUT_ERR_INVALID_ARGUMENT;
    if (grid_den < 1 || sprout_static_grid_size(problem->n_levels, grid_den) != (int64_t)problem->n_xi)
        return SPROUT_ERR_INVALID_ARGUMENT;
    sprout_lp_problem P = *problem;
    static const double zero = 0.0;
    if (!P.xi) P.xi = &zero;
    sprout_status st = validate_problem(&P);
    if (st != SPROUT_OK) return st;
    if (!aligned(group_totals, 8) || !aligned(x, 8) || !aligned(choice, 4)) return SPROUT_ERR_INVALID_ARGUMENT;
    SelectArgs a{};
    a.n = P.n_levels; a.R = P.n_regions; a.G = P.n_xi; a.K = 11 + 2 * P.n_levels; a.grid_den = grid_den;
    a.T = P.n_intervals;
    a.k0 = P.k0; a.kmin = P.k0_min; a.kmax = P.k0_max; a.q = P.q; a.xi = xi;
    a.group = group_totals; a.choice = choice; a.x = x;
    int launches = 0;
    st = cuda_status(launch_select_static(a, reinterpret_cast<cudaStream_t>(stream), &launches));
    if (st == SPROUT_OK) g_last_launches = launches;
    return st;
}

// the grace test in samples: the least s with (double)s * dt >= grace (the same decision for every s)
static int64_t grace_samples(double grace_hours, double interval_hours) {
    double s0 = std::ceil(grace_hours / interval_hours);
    if (s0 > 2147483647.0) s0 = 2147483647.0;
    int64_t s = (int64_t)s0;
    while (s > 0 && (double)(s - 1) * interval_hours >= grace_hours) --s;
    while (s < 2147483647 && !((double)s * interval_hours >= grace_hours)) ++s;
    return s;
}

sprout_status sprout_evaluator_sweep(const sprout_evaluator_problem *P, double *out, sprout_stream stream) {
    if (!P || !out) return SPROUT_ERR_INVALID_ARGUMENT;
    if (P->n_regions < 1 || P->n_intervals < 1 || P->n_beta < 1 || P->n_beta > SPROUT_MAX_EVAL_PARAMS ||
        P->n_theta < 1 || P->n_theta > SPROUT_MAX_EVAL_PARAMS || P->fallback < 0)
        return SPROUT_ERR_INVALID_ARGUMENT;
    if (!(P->interval_hours > 0.0) || !std::isfinite(P->interval_hours) || !(P->grace_hours >= 0.0) ||
        !std::isfinite(P->grace_hours) || !(P->eval_kwh >= 0.0) || !std::isfinite(P->eval_kwh) ||
        !(P->pue >= 1.0) || !std::isfinite(P->pue))
        return SPROUT_ERR_INVALID_ARGUMENT;
    if (!P->k2 || !P->k2_max || !P->beta || !P->theta || !aligned(out, 8)) return SPROUT_ERR_INVALID_ARGUMENT;
    if (P->n_intervals >= ((int64_t)1 << 31)) return SPROUT_ERR_OVERFLOW;
    EvalArgs a{};
    a.grace_samples = (int)grace_samples(P->grace_hours, P->interval_hours);
    a.R = P->n_regions; a.B = P->n_beta; a.H = P->n_theta; a.F = P->fallback; a.T = P->n_intervals;
    a.dt = P->interval_hours; a.grace = P->grace_hours; a.eval_kwh = P->eval_kwh; a.pue = P->pue;
    a.k2 = P->k2; a.k2_max = P->k2_max; a.out = out;
    for (int b = 0; b < a.B; ++b) {
        const double beta = P->beta[b];
        if (!(beta >= 0.0) || !std::isfinite(beta)) return SPROUT_ERR_INVALID_ARGUMENT;
        a.decay[b] = std::exp(-(beta * a.dt));   // Eq. 8's factor over one interval (reading L19)
    }
    for (int h = 0; h < a.H; ++h) {
        if (!(P->theta[h] >= 0.0) || !std::isfinite(P->theta[h])) return SPROUT_ERR_INVALID_ARGUMENT;
        a.theta[h] = P->theta[h];
    }
    int launches = 0;
    sprout_status st = cuda_status(launch_evaluator(a, reinterpret_cast<cudaStream_t>(stream), &launches));
    if (st == SPROUT_OK) g_last_launches = launches;
    return st;
}

static sprout_status simulate_impl(const sprout_lp_problem *problem, const sprout_lp_solution *solution,
                                   const sprout_trace *trace, const sprout_cost_model *cost,
                                   const sprout_cell_totals *totals, uint8_t *levels_out, int32_t max_breakpoints,
                                   void *workspace, size_t workspace_bytes, sprout_stream stream,
                                   const double *q_rows);

sprout_status sprout_simulate_closed_loop(const sprout_lp_problem *problem, int32_t window,
                                          const sprout_trace *trace, const sprout_cost_model *cost,
                                          const sprout_lp_solution *solution, const sprout_cell_totals *totals,
                                          double *profile_out, void *workspace, size_t workspace_bytes,
                                          sprout_stream stream) {
    return sprout_simulate_closed_loop_q(problem, window, nullptr, trace, cost, solution, totals, profile_out,
                                         workspace, workspace_bytes, stream);
}

sprout_status sprout_simulate_closed_loop_q(const sprout_lp_problem *problem, int32_t window, const double *q_interval,
                                            const sprout_trace *trace, const sprout_cost_model *cost,
                                            const sprout_lp_solution *solution, const sprout_cell_totals *totals,
                                            double *profile_out, void *workspace, size_t workspace_bytes,
                                            sprout_stream stream) {
    if (q_interval && !aligned(q_interval, 8)) return SPROUT_ERR_INVALID_ARGUMENT;
    sprout_status st = validate_problem(problem);
    if (st == SPROUT_OK) st = validate_solution(problem, solution);
    if (st == SPROUT_OK) st = validate_trace(problem, trace);
    if (st == SPROUT_OK) st = validate_cost(cost);
    if (st != SPROUT_OK) return st;
    if (st == SPROUT_OK) st = validate_totals(problem, totals);
    if (st != SPROUT_OK) return st;
    // whole regions only: a chain is one region's intervals in order
    if (problem->first_segment % problem->n_intervals != 0 || problem->n_segments % problem->n_intervals != 0 ||
        problem->profile_per_interval != 0)
        return SPROUT_ERR_INVALID_ARGUMENT;
    const int64_t S = problem->n_segments;
    if (window < 1 || window > 4096 || (int64_t)problem->n_levels * window * 4 > 96 * 1024)
        return SPROUT_ERR_INVALID_ARGUMENT;
    {   // the totals pass's workspace (sprout_workspace_bytes)
        SimPlan plan;
        if (!make_sim_plan(problem->n_levels, problem->n_xi, cost->n_classes, &plan) || !workspace ||
            workspace_bytes < sim_workspace_bytes(plan, problem->n_segments) || !aligned(workspace, 256))
            return SPROUT_ERR_INVALID_ARGUMENT;
    }
    if (profile_out && !aligned(profile_out, 8)) return SPROUT_ERR_INVALID_ARGUMENT;
    ClosedArgs a{};
    a.n = problem->n_levels; a.R = problem->n_regions; a.X = problem->n_xi; a.NC = cost->n_classes; a.W = window;
    a.T = problem->n_intervals;
    a.first_segment = problem->first_segment;
    a.n_requests = trace->n_requests;
    a.r0 = (int)(problem->first_segment / problem->n_intervals);
    a.R_local = (int)(problem->n_segments / problem->n_intervals);
    a.k0 = problem->k0; a.kmin = problem->k0_min; a.kmax = problem->k0_max; a.xi = problem->xi;
    a.e = problem->e; a.p = problem->p; a.q = problem->q; a.k1 = problem->k1; a.pue = problem->pue;
    a.q_seg = q_interval;
    {
        uint32_t k0 = (uint32_t)cost->seed, k1 = (uint32_t)(cost->seed >> 32);
        for (int r = 0; r < 10; ++r) { a.rk0[r] = k0; a.rk1[r] = k1; k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    }
    std::memcpy(a.cost.ef, cost->ef, sizeof(cost->ef));
    std::memcpy(a.cost.et, cost->et, sizeof(cost->et));
    std::memcpy(a.cost.pf, cost->pf, sizeof(cost->pf));
    std::memcpy(a.cost.pt, cost->pt, sizeof(cost->pt));
    a.first_request = trace->first_request; a.seg_offsets = trace->seg_offsets; a.tokens = trace->tokens;
    a.pitch = trace->plane_pitch; a.flags = trace->flags;
    a.x = solution->x; a.objective = solution->objective; a.q_lb = solution->q_lb; a.profile = profile_out;
    a.vertex = solution->vertex; a.cell_status = solution->cell_status; a.max_level = solution->max_level;
    a.threshold = solution->threshold;
    a.cnt = totals->cnt; a.tok = totals->tok; a.energy = totals->energy_kwh; a.time_s = totals->time_s;
    a.carbon = totals->carbon_g; a.quality = totals->quality; a.trace_status = totals->trace_status;
    a.seg_count = totals->seg_count; a.seg_pinned = totals->seg_pinned; a.seg_tok = totals->seg_tok;
    a.seg_base = totals->seg_base;
    {   // the chain schedule's scratch: the head of the totals pass's workspace, free until that pass
        const size_t chains = (size_t)a.R_local * a.X;
        if (chains * 8 <= workspace_bytes) {
            a.chain_cost = static_cast<float *>(workspace);
            a.chain_order = reinterpret_cast<int *>(static_cast<float *>(workspace) + chains);
        }
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    int launches = 0;
    st = cuda_status(launch_closed_loop(a, s, &launches));   // every interval's LP, the windows
    if (st != SPROUT_OK) return st;
    // the totals of the solved thresholds: the open-loop streaming pass (cells,
    // segments, trace_status), quality rows per interval when q varies
    st = simulate_impl(problem, solution, trace, cost, totals, nullptr, 0, workspace, workspace_bytes, stream,
                       q_interval);
    if (st == SPROUT_OK) g_last_launches += launches;
    return st;
}

size_t sprout_workspace_bytes(const sprout_lp_problem *problem, const sprout_trace *trace) {
    if (validate_problem(problem) != SPROUT_OK) return 0;
    (void)trace;
    SimPlan plan;
    if (!make_sim_plan(problem->n_levels, problem->n_xi, SPROUT_MAX_CLASSES, &plan)) return 0;
    // the plan's workspace does not depend on the class count
    return sim_workspace_bytes(plan, problem->n_segments);
}

sprout_status sprout_simulate_trace(const sprout_lp_problem *problem, const sprout_lp_solution *solution,
                                    const sprout_trace *trace, const sprout_cost_model *cost,
                                    const sprout_cell_totals *totals, uint8_t *levels_out, void *workspace,
                                    size_t workspace_bytes, sprout_stream stream) {
    return sprout_simulate_trace_bounded(problem, solution, trace, cost, totals, levels_out, 0, workspace,
                                         workspace_bytes, stream);
}

// the streaming simulate (steps a5-a8) of a solution; q_rows (NULL: the
// problem's q) overrides the quality rows with one per interval
static sprout_status simulate_impl(const sprout_lp_problem *problem, const sprout_lp_solution *solution,
                                   const sprout_trace *trace, const sprout_cost_model *cost,
                                   const sprout_cell_totals *totals, uint8_t *levels_out, int32_t max_breakpoints,
                                   void *workspace, size_t workspace_bytes, sprout_stream stream,
                                   const double *q_rows) {
    if (max_breakpoints < 0) return SPROUT_ERR_INVALID_ARGUMENT;
    sprout_status st = validate_problem(problem);
    if (st == SPROUT_OK) st = validate_solution(problem, solution);
    if (st == SPROUT_OK) st = validate_trace(problem, trace);
    if (st == SPROUT_OK) st = validate_cost(cost);
    if (st == SPROUT_OK) st = validate_totals(problem, totals);
    if (st != SPROUT_OK) return st;
    SimPlan plan;
    if (!make_sim_plan(problem->n_levels, problem->n_xi, cost->n_classes, &plan, max_breakpoints))
        return SPROUT_ERR_INVALID_ARGUMENT;
    if (!workspace || workspace_bytes < sim_workspace_bytes(plan, problem->n_segments) || !aligned(workspace, 256))
        return SPROUT_ERR_INVALID_ARGUMENT;

    SimArgs a{};
    a.n = problem->n_levels; a.X = problem->n_xi; a.NC = cost->n_classes;
    a.T = problem->n_intervals; a.first_segment = problem->first_segment; a.n_segments = problem->n_segments;
    a.profile_per_interval = problem->profile_per_interval;
    a.k0 = problem->k0; a.q = problem->q; a.k1 = problem->k1; a.pue = problem->pue;
    if (q_rows) { a.q = q_rows; a.profile_per_interval = 1; }
    a.threshold = solution->threshold; a.max_level = solution->max_level; a.cell_status = solution->cell_status;
    a.n_requests = trace->n_requests; a.first_request = trace->first_request; a.seg_offsets = trace->seg_offsets;
    a.tokens = trace->tokens; a.pitch = trace->plane_pitch; a.flags = trace->flags; a.seed = cost->seed;
    a.cnt = totals->cnt; a.tok = totals->tok; a.energy = totals->energy_kwh; a.time_s = totals->time_s;
    a.carbon = totals->carbon_g; a.quality = totals->quality; a.seg_count = totals->seg_count;
    a.seg_pinned = totals->seg_pinned; a.seg_tok = totals->seg_tok; a.seg_base = totals->seg_base;
    a.trace_status = totals->trace_status; a.levels_out = levels_out;
    static_assert(sizeof(a.cost.ef) == sizeof(cost->ef), "cost layout");
    std::memcpy(a.cost.ef, cost->ef, sizeof(cost->ef));
    std::memcpy(a.cost.et, cost->et, sizeof(cost->et));
    std::memcpy(a.cost.pf, cost->pf, sizeof(cost->pf));
    std::memcpy(a.cost.pt, cost->pt, sizeof(cost->pt));
    int launches = 0;
    st = cuda_status(launch_simulate(a, plan, workspace, reinterpret_cast<cudaStream_t>(stream), &launches));
    if (st == SPROUT_OK) g_last_launches = launches;
    return st;
}

sprout_status sprout_simulate_trace_bounded(const sprout_lp_problem *problem, const sprout_lp_solution *solution,
                                            const sprout_trace *trace, const sprout_cost_model *cost,
                                            const sprout_cell_totals *totals, uint8_t *levels_out,
                                            int32_t max_breakpoints, void *workspace, size_t workspace_bytes,
                                            sprout_stream stream) {
    return simulate_impl(problem, solution, trace, cost, totals, levels_out, max_breakpoints, workspace,
                         workspace_bytes, stream, nullptr);
}

sprout_status sprout_cell_totals_fp64(const sprout_lp_problem *problem, const sprout_lp_solution *solution,
                                      const sprout_trace *trace, const sprout_cost_model *cost, double *energy_kwh,
                                      double *time_s, double *carbon_g, double *quality, sprout_stream stream) {
    sprout_status st = validate_problem(problem);
    if (st == SPROUT_OK) st = validate_solution(problem, solution);
    if (st == SPROUT_OK) st = validate_trace(problem, trace);
    if (st == SPROUT_OK) st = validate_cost(cost);
    if (st != SPROUT_OK) return st;
    if (!energy_kwh || !time_s || !carbon_g || !quality || !aligned(energy_kwh, 8) || !aligned(time_s, 8) ||
        !aligned(carbon_g, 8) || !aligned(quality, 8))
        return SPROUT_ERR_INVALID_ARGUMENT;
    F64Args a{};
    a.n = problem->n_levels; a.X = problem->n_xi; a.NC = cost->n_classes;
    a.T = problem->n_intervals; a.first_segment = problem->first_segment; a.n_segments = problem->n_segments;
    a.profile_per_interval = problem->profile_per_interval;
    a.k0 = problem->k0; a.q = problem->q; a.k1 = problem->k1; a.pue = problem->pue;
    a.threshold = solution->threshold; a.max_level = solution->max_level; a.cell_status = solution->cell_status;
    a.n_requests = trace->n_requests; a.first_request = trace->first_request; a.seg_offsets = trace->seg_offsets;
    a.tokens = trace->tokens; a.pitch = trace->plane_pitch; a.flags = trace->flags;
    {
        uint32_t k0 = (uint32_t)cost->seed, k1 = (uint32_t)(cost->seed >> 32);
        for (int r = 0; r < 10; ++r) { a.rk0[r] = k0; a.rk1[r] = k1; k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    }
    std::memcpy(a.cost.ef, cost->ef, sizeof(cost->ef));
    std::memcpy(a.cost.et, cost->et, sizeof(cost->et));
    std::memcpy(a.cost.pf, cost->pf, sizeof(cost->pf));
    std::memcpy(a.cost.pt, cost->pt, sizeof(cost->pt));
    a.energy = energy_kwh; a.time_s = time_s; a.carbon = carbon_g; a.quality = quality;
    int launches = 0;
    st = cuda_status(launch_fp64_cells(a, reinterpret_cast<cudaStream_t>(stream), &launches));
    if (st == SPROUT_OK) g_last_launches = launches;
    return st;
}

static sprout_status n4_args(const sprout_lp_problem *problem, const sprout_lp_solution *solution,
                             const sprout_trace *trace, const sprout_cost_model *cost, N4Args &a) {
    sprout_status st = validate_problem(problem);
    if (st == SPROUT_OK) st = validate_solution(problem, solution);
    if (st == SPROUT_OK) st = validate_trace(problem, trace);
    if (st == SPROUT_OK) st = validate_cost(cost);
    if (st != SPROUT_OK) return st;
    a = N4Args{};
    a.n = problem->n_levels; a.X = problem->n_xi; a.NC = cost->n_classes;
    a.T = problem->n_intervals; a.first_segment = problem->first_segment; a.n_segments = problem->n_segments;
    a.profile_per_interval = problem->profile_per_interval;
    a.k0 = problem->k0; a.q = problem->q; a.k1 = problem->k1; a.pue = problem->pue;
    a.threshold = solution->threshold; a.max_level = solution->max_level; a.cell_status = solution->cell_status;
    a.n_requests = trace->n_requests; a.first_request = trace->first_request; a.seg_offsets = trace->seg_offsets;
    a.tokens = trace->tokens; a.pitch = trace->plane_pitch; a.flags = trace->flags; a.seed = cost->seed;
    std::memcpy(a.cost.ef, cost->ef, sizeof(cost->ef));
    std::memcpy(a.cost.et, cost->et, sizeof(cost->et));
    std::memcpy(a.cost.pf, cost->pf, sizeof(cost->pf));
    std::memcpy(a.cost.pt, cost->pt, sizeof(cost->pt));
    return SPROUT_OK;
}

sprout_status sprout_request_outputs(const sprout_lp_problem *problem, const sprout_lp_solution *solution,
                                     const sprout_trace *trace, const sprout_cost_model *cost, int32_t xi_index,
                                     uint8_t *level_out, double *carbon_out, double *base_out, double *ratio_out,
                                     uint8_t *pref_out, sprout_stream stream) {
    N4Args a;
    sprout_status st = n4_args(problem, solution, trace, cost, a);
    if (st != SPROUT_OK) return st;
    if (xi_index < 0 || xi_index >= problem->n_xi) return SPROUT_ERR_INVALID_ARGUMENT;
    if (trace->n_requests > 0 && (!level_out || !carbon_out || !base_out || !ratio_out || !aligned(carbon_out, 8) ||
                                  !aligned(base_out, 8) || !aligned(ratio_out, 8)))
        return SPROUT_ERR_INVALID_ARGUMENT;
    a.column = xi_index;
    a.level_out = level_out; a.carbon_out = carbon_out; a.base_out = base_out; a.ratio_out = ratio_out;
    a.pref_out = pref_out;
    int launches = 0;
    st = cuda_status(launch_request_outputs(a, reinterpret_cast<cudaStream_t>(stream), &launches));
    if (st == SPROUT_OK) g_last_launches = launches;
    return st;
}

sprout_status sprout_preference_stats(const sprout_lp_problem *problem, const sprout_lp_solution *solution,
                                      const sprout_trace *trace, const sprout_cost_model *cost, uint64_t *stats,
                                      sprout_stream stream) {
    N4Args a;
    sprout_status st = n4_args(problem, solution, trace, cost, a);
    if (st != SPROUT_OK) return st;
    if (problem->n_segments > 0 && (!stats || !aligned(stats, 8))) return SPROUT_ERR_INVALID_ARGUMENT;
    if ((size_t)problem->n_xi * 12 > 200 * 1024) return SPROUT_ERR_INVALID_ARGUMENT;
    a.stats = stats;
    int launches = 0;
    st = cuda_status(launch_pref_stats(a, reinterpret_cast<cudaStream_t>(stream), &launches));
    if (st == SPROUT_OK) g_last_launches = launches;
    return st;
}

size_t sprout_oracle_scheme_workspace_bytes(const sprout_lp_problem *problem, int64_t max_segment_requests) {
    if (validate_problem(problem) != SPROUT_OK || max_segment_requests < 0 ||
        max_segment_requests > ((int64_t)1 << 32))
        return 0;
    return oracle_scheme_workspace_bytes(max_segment_requests);
}

sprout_status sprout_simulate_oracle_scheme(const sprout_lp_problem *problem, const sprout_trace *trace,
                                            const sprout_cost_model *cost, int64_t max_segment_requests,
                                            const sprout_cell_totals *totals, uint64_t *stats, uint8_t *cell_status,
                                            void *workspace, size_t workspace_bytes, sprout_stream stream) {
    sprout_status st = validate_problem(problem);
    if (st == SPROUT_OK) st = validate_trace(problem, trace);
    if (st == SPROUT_OK) st = validate_cost(cost);
    if (st == SPROUT_OK) st = validate_totals(problem, totals);
    if (st != SPROUT_OK) return st;
    if (max_segment_requests < 0 || max_segment_requests > ((int64_t)1 << 32)) return SPROUT_ERR_INVALID_ARGUMENT;
    if (problem->n_segments > 0 && (!stats || !cell_status || !aligned(stats, 8))) return SPROUT_ERR_INVALID_ARGUMENT;
    if (!workspace || !aligned(workspace, 256) ||
        workspace_bytes < oracle_scheme_workspace_bytes(max_segment_requests))
        return SPROUT_ERR_INVALID_ARGUMENT;
    N4Args a{};
    a.n = problem->n_levels; a.X = problem->n_xi; a.NC = cost->n_classes;
    a.T = problem->n_intervals; a.first_segment = problem->first_segment; a.n_segments = problem->n_segments;
    a.profile_per_interval = problem->profile_per_interval;
    a.k0 = problem->k0; a.q = problem->q; a.k1 = problem->k1; a.pue = problem->pue;
    a.xi = problem->xi; a.kmin = problem->k0_min; a.kmax = problem->k0_max;
    a.n_requests = trace->n_requests; a.first_request = trace->first_request; a.seg_offsets = trace->seg_offsets;
    a.tokens = trace->tokens; a.pitch = trace->plane_pitch; a.flags = trace->flags; a.seed = cost->seed;
    std::memcpy(a.cost.ef, cost->ef, sizeof(cost->ef));
    std::memcpy(a.cost.et, cost->et, sizeof(cost->et));
    std::memcpy(a.cost.pf, cost->pf, sizeof(cost->pf));
    std::memcpy(a.cost.pt, cost->pt, sizeof(cost->pt));
    a.cap = max_segment_requests;
    a.queue = static_cast<uint32_t *>(workspace);
    a.scratch = static_cast<uint8_t *>(workspace) + 256;
    a.stats = stats; a.cell_status_out = cell_status;
    a.cnt = totals->cnt; a.tok = totals->tok; a.energy = totals->energy_kwh; a.time_s = totals->time_s;
    a.carbon = totals->carbon_g; a.quality = totals->quality; a.seg_count = totals->seg_count;
    a.seg_pinned = totals->seg_pinned; a.seg_tok = totals->seg_tok; a.seg_base = totals->seg_base;
    a.trace_status = totals->trace_status;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (cudaMemsetAsync(totals->trace_status, 0, 4, s) != cudaSuccess) return SPROUT_ERR_CUDA;
    int launches = 0;
    st = cuda_status(launch_oracle_scheme(a, s, &launches));
    if (st == SPROUT_OK) g_last_launches = launches;
    return st;
}

sprout_status sprout_evaluation_q(const sprout_evaluator_problem *ev, const sprout_lp_problem *problem,
                                  const sprout_trace *trace, const sprout_cost_model *cost, int32_t sample,
                                  double *q_out, uint8_t *fired_out, sprout_stream stream) {
    sprout_status st = validate_problem(problem);
    if (st == SPROUT_OK) st = validate_trace(problem, trace);
    if (st == SPROUT_OK) st = validate_cost(cost);
    if (st != SPROUT_OK) return st;
    if (!ev || ev->n_beta != 1 || ev->n_theta != 1 || !ev->beta || !ev->theta || !ev->k2 || !ev->k2_max ||
        ev->fallback < 0 || ev->n_regions != problem->n_regions || ev->n_intervals != problem->n_intervals)
        return SPROUT_ERR_INVALID_ARGUMENT;
    if (!(ev->interval_hours > 0.0) || !std::isfinite(ev->interval_hours) || !(ev->grace_hours >= 0.0) ||
        !std::isfinite(ev->grace_hours) || !(ev->beta[0] >= 0.0) || !std::isfinite(ev->beta[0]) ||
        !(ev->theta[0] >= 0.0) || !std::isfinite(ev->theta[0]))
        return SPROUT_ERR_INVALID_ARGUMENT;
    // the whole sweep (every region's intervals in order), q per region (the truth behind l*)
    if (problem->first_segment != 0 || problem->n_segments != (int64_t)problem->n_regions * problem->n_intervals ||
        problem->profile_per_interval != 0 || sample < 1 || !q_out || !fired_out || !aligned(q_out, 8))
        return SPROUT_ERR_INVALID_ARGUMENT;
    EvalQArgs a{};
    a.R = problem->n_regions; a.n = problem->n_levels; a.F = ev->fallback; a.sample = sample;
    a.T = problem->n_intervals;
    a.grace_samples = grace_samples(ev->grace_hours, ev->interval_hours);
    a.decay = std::exp(-(ev->beta[0] * ev->interval_hours));   // Eq. 8's factor over one interval (reading L19)
    a.theta = ev->theta[0];
    a.k2 = ev->k2; a.k2_max = ev->k2_max; a.q = problem->q;
    a.seg_offsets = trace->seg_offsets; a.first_request = trace->first_request; a.seed = cost->seed;
    a.q_out = q_out; a.fired = fired_out;
    int launches = 0;
    st = cuda_status(launch_evaluation_q(a, reinterpret_cast<cudaStream_t>(stream), &launches));
    if (st == SPROUT_OK) g_last_launches = launches;
    return st;
}

double sprout_normalized_preference(double w) {
    if (!(w >= 0.0)) return std::nan("");
    return w >= 1.0 ? HUGE_VAL : w / (1.0 - w);
}

int32_t sprout_group_stat_count(int32_t n_levels) { return 11 + 2 * n_levels; }

size_t sprout_reduce_workspace_bytes(const sprout_lp_problem *problem) {
    if (validate_problem(problem) != SPROUT_OK) return 0;
    return reduce_workspace_bytes(problem->n_levels, problem->n_xi, problem->n_regions, problem->n_intervals,
                                  problem->first_segment, problem->n_segments);
}

sprout_status sprout_reduce_totals(const sprout_lp_problem *problem, const sprout_lp_solution *solution,
                                   const sprout_cell_totals *totals, int32_t n_classes, double *group_totals,
                                   void *workspace, size_t workspace_bytes, sprout_stream stream) {
    sprout_status st = validate_problem(problem);
    if (st == SPROUT_OK) st = validate_solution(problem, solution);
    if (st == SPROUT_OK) st = validate_totals(problem, totals);
    if (st != SPROUT_OK) return st;
    if (n_classes < 1 || n_classes > SPROUT_MAX_CLASSES || !group_totals || !aligned(group_totals, 8))
        return SPROUT_ERR_INVALID_ARGUMENT;
    if (!workspace || workspace_bytes < sprout_reduce_workspace_bytes(problem)) return SPROUT_ERR_INVALID_ARGUMENT;
    ReduceArgs a{};
    a.n = problem->n_levels; a.X = problem->n_xi; a.NC = n_classes; a.R = problem->n_regions;
    a.T = problem->n_intervals; a.first_segment = problem->first_segment; a.n_segments = problem->n_segments;
    a.cell_status = solution->cell_status; a.objective = solution->objective;
    a.cnt = totals->cnt; a.tok = totals->tok; a.energy = totals->energy_kwh; a.time_s = totals->time_s;
    a.carbon = totals->carbon_g; a.quality = totals->quality; a.seg_count = totals->seg_count;
    a.seg_pinned = totals->seg_pinned; a.seg_base = totals->seg_base; a.out = group_totals;
    int launches = 0;
    st = cuda_status(launch_reduce(a, workspace, reinterpret_cast<cudaStream_t>(stream), &launches));
    if (st == SPROUT_OK) g_last_launches = launches;
    return st;
}

sprout_status sprout_check_cells(const sprout_lp_problem *problem, const sprout_lp_solution *solution,
                                 sprout_stream stream) {
    sprout_status st = validate_problem(problem);
    if (st == SPROUT_OK) st = validate_solution(problem, solution);
    if (st != SPROUT_OK) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    uint32_t *d = nullptr, h = 0;
    if (cudaMallocAsync(&d, sizeof(uint32_t), s) != cudaSuccess) return SPROUT_ERR_CUDA;
    int launches = 0;
    cudaError_t e = launch_check_cells(solution->cell_status, problem->n_segments * (int64_t)problem->n_xi, d, s,
                                       &launches);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(d, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return SPROUT_ERR_CUDA;
    g_last_launches = launches;
    if (h & 1u) return SPROUT_ERR_INVALID_CELL;
    if (h & 2u) return SPROUT_ERR_INFEASIBLE;
    return SPROUT_OK;
}

// ---------------------------------------------------------------------------
// end-to-end with host buffers

namespace {
struct SweepLayout {
    size_t k0, kmin, kmax, xi, e, p, q;               // problem arrays
    size_t x, obj, qlb, vertex, thr, maxl, status;    // solution
    size_t segoff, tokens, flags;                     // trace
    size_t cnt, tok, energy, time, carbon, quality, seg_count, seg_pinned, seg_tok, seg_base, trace_status;
    size_t group, sim_ws, red_ws;
    size_t sim_ws_bytes, red_ws_bytes, total;
};

size_t up(size_t v) { return (v + 255) & ~(size_t)255; }

bool sweep_layout(const sprout_lp_problem *P, const sprout_trace *T, int NC, SweepLayout *L) {
    SimPlan plan;
    if (!make_sim_plan(P->n_levels, P->n_xi, NC, &plan)) return false;
    const int n = P->n_levels, X = P->n_xi;
    const int64_t S = (int64_t)P->n_regions * P->n_intervals;
    const int64_t rows = P->profile_per_interval ? S : P->n_regions;
    const int64_t cells = P->n_segments * X;
    size_t o = 0;
    auto take = [&](size_t bytes) { const size_t at = o; o += up(bytes); return at; };
    L->k0 = take(S * 8); L->kmin = take(P->n_regions * 8); L->kmax = take(P->n_regions * 8);
    L->xi = take((size_t)X * 8); L->e = take(rows * n * 8); L->p = take(rows * n * 8); L->q = take(rows * n * 8);
    L->x = take(cells * n * 8); L->obj = take(cells * 8); L->qlb = take(cells * 8); L->vertex = take(cells);
    L->thr = take(cells * (n > 1 ? n - 1 : 1) * 4); L->maxl = take(cells); L->status = take(cells);
    L->segoff = take((P->n_segments + 1) * 8);
    L->tokens = take((size_t)n * T->plane_pitch * 2);
    L->flags = take(T->flags ? (size_t)T->plane_pitch : 0);
    L->cnt = take(cells * NC * n * 8); L->tok = take(cells * NC * n * 8);
    L->energy = take(cells * 8); L->time = take(cells * 8); L->carbon = take(cells * 8); L->quality = take(cells * 8);
    L->seg_count = take(P->n_segments * NC * 8); L->seg_pinned = take(P->n_segments * NC * 8);
    L->seg_tok = take(P->n_segments * NC * n * 8); L->seg_base = take(P->n_segments * 4 * 8);
    L->trace_status = take(4);
    L->group = take((size_t)(P->n_regions + 1) * X * (11 + 2 * n) * 8);
    L->sim_ws_bytes = sim_workspace_bytes(plan, P->n_segments);
    L->sim_ws = take(L->sim_ws_bytes);
    L->red_ws_bytes = reduce_workspace_bytes(n, X, P->n_regions, P->n_intervals, P->first_segment, P->n_segments);
    L->red_ws = take(L->red_ws_bytes);
    L->total = o;
    return true;
}
}  // namespace

size_t sprout_sweep_workspace_bytes(const sprout_lp_problem *problem, const sprout_trace *trace, int32_t n_classes) {
    if (validate_problem(problem) != SPROUT_OK || validate_trace(problem, trace) != SPROUT_OK) return 0;
    if (n_classes < 1 || n_classes > SPROUT_MAX_CLASSES) return 0;
    SweepLayout L;
    if (!sweep_layout(problem, trace, n_classes, &L)) return 0;
    return L.total;
}

sprout_status sprout_sweep_host(const sprout_lp_problem *problem, const sprout_trace *trace,
                                const sprout_cost_model *cost, double *host_group_totals,
                                uint32_t *host_trace_status, void *device_workspace,
                                size_t device_workspace_bytes, sprout_stream stream) {
    sprout_status st = validate_problem(problem);
    if (st == SPROUT_OK) st = validate_trace(problem, trace);
    if (st == SPROUT_OK) st = validate_cost(cost);
    if (st != SPROUT_OK) return st;
    if (!host_group_totals || !device_workspace || !aligned(device_workspace, 256)) return SPROUT_ERR_INVALID_ARGUMENT;
    SweepLayout L;
    if (!sweep_layout(problem, trace, cost->n_classes, &L) || device_workspace_bytes < L.total)
        return SPROUT_ERR_INVALID_ARGUMENT;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    uint8_t *w = static_cast<uint8_t *>(device_workspace);
    const int n = problem->n_levels, X = problem->n_xi, NC = cost->n_classes;
    const int64_t S = (int64_t)problem->n_regions * problem->n_intervals;
    const int64_t rows = problem->profile_per_interval ? S : problem->n_regions;
    auto h2d = [&](size_t off, const void *src, size_t bytes) {
        return bytes ? cudaMemcpyAsync(w + off, src, bytes, cudaMemcpyHostToDevice, s) : cudaSuccess;
    };
    cudaError_t e = cudaSuccess;
    if (e == cudaSuccess) e = h2d(L.k0, problem->k0, S * 8);
    if (e == cudaSuccess) e = h2d(L.kmin, problem->k0_min, problem->n_regions * 8);
    if (e == cudaSuccess) e = h2d(L.kmax, problem->k0_max, problem->n_regions * 8);
    if (e == cudaSuccess) e = h2d(L.xi, problem->xi, (size_t)X * 8);
    if (e == cudaSuccess) e = h2d(L.e, problem->e, rows * n * 8);
    if (e == cudaSuccess) e = h2d(L.p, problem->p, rows * n * 8);
    if (e == cudaSuccess) e = h2d(L.q, problem->q, rows * n * 8);
    if (e == cudaSuccess) e = h2d(L.segoff, trace->seg_offsets, (problem->n_segments + 1) * 8);
    if (e == cudaSuccess) e = h2d(L.tokens, trace->tokens, (size_t)n * trace->plane_pitch * 2);
    if (e == cudaSuccess && trace->flags) e = h2d(L.flags, trace->flags, (size_t)trace->plane_pitch);
    if (e != cudaSuccess) return SPROUT_ERR_CUDA;

    sprout_lp_problem dp = *problem;
    dp.k0 = reinterpret_cast<double *>(w + L.k0); dp.k0_min = reinterpret_cast<double *>(w + L.kmin);
    dp.k0_max = reinterpret_cast<double *>(w + L.kmax); dp.xi = reinterpret_cast<double *>(w + L.xi);
    dp.e = reinterpret_cast<double *>(w + L.e); dp.p = reinterpret_cast<double *>(w + L.p);
    dp.q = reinterpret_cast<double *>(w + L.q);
    sprout_lp_solution sol{reinterpret_cast<double *>(w + L.x), reinterpret_cast<double *>(w + L.obj),
                           reinterpret_cast<double *>(w + L.qlb), w + L.vertex,
                           n > 1 ? reinterpret_cast<uint32_t *>(w + L.thr) : nullptr, w + L.maxl, w + L.status};
    sprout_trace tr = *trace;
    tr.seg_offsets = reinterpret_cast<int64_t *>(w + L.segoff);
    tr.tokens = reinterpret_cast<uint16_t *>(w + L.tokens);
    tr.flags = trace->flags ? w + L.flags : nullptr;
    sprout_cell_totals tot{reinterpret_cast<uint64_t *>(w + L.cnt), reinterpret_cast<uint64_t *>(w + L.tok),
                           reinterpret_cast<double *>(w + L.energy), reinterpret_cast<double *>(w + L.time),
                           reinterpret_cast<double *>(w + L.carbon), reinterpret_cast<double *>(w + L.quality),
                           reinterpret_cast<uint64_t *>(w + L.seg_count), reinterpret_cast<uint64_t *>(w + L.seg_pinned),
                           reinterpret_cast<uint64_t *>(w + L.seg_tok), reinterpret_cast<double *>(w + L.seg_base),
                           reinterpret_cast<uint32_t *>(w + L.trace_status)};
    int launches = 0;
    st = sprout_solve_directives(&dp, &sol, stream);
    launches += g_last_launches;
    if (st == SPROUT_OK) {
        st = sprout_simulate_trace(&dp, &sol, &tr, cost, &tot, nullptr, w + L.sim_ws, L.sim_ws_bytes, stream);
        launches += g_last_launches;
    }
    double *group = reinterpret_cast<double *>(w + L.group);
    if (st == SPROUT_OK) {
        st = sprout_reduce_totals(&dp, &sol, &tot, NC, group, w + L.red_ws, L.red_ws_bytes, stream);
        launches += g_last_launches;
    }
    if (st != SPROUT_OK) return st;
    e = cudaMemcpyAsync(host_group_totals, group, (size_t)(problem->n_regions + 1) * X * (11 + 2 * n) * 8,
                        cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && host_trace_status)
        e = cudaMemcpyAsync(host_trace_status, w + L.trace_status, 4, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return SPROUT_ERR_CUDA;
    g_last_launches = launches;
    return SPROUT_OK;
}

sprout_status sprout_generate_trace(const sprout_trace_generator *gen, uint16_t *tokens, int64_t plane_pitch,
                                    uint8_t *flags, sprout_stream stream) {
    if (!gen || gen->n_levels < 1 || gen->n_levels > SPROUT_MAX_LEVELS || gen->n_classes < 1 ||
        gen->n_classes > SPROUT_MAX_CLASSES || gen->n_requests < 0 || plane_pitch < gen->n_requests ||
        plane_pitch % 8 != 0 || !gen->q0_table || !gen->ratio_table)
        return SPROUT_ERR_INVALID_ARGUMENT;
    if (plane_pitch > 0 && (!tokens || !aligned(tokens, 16))) return SPROUT_ERR_INVALID_ARGUMENT;
    if (flags && !aligned(flags, 16)) return SPROUT_ERR_INVALID_ARGUMENT;
    GenArgs a{};
    a.gen_seed = gen->gen_seed; a.first_request = gen->first_request; a.n_requests = gen->n_requests;
    a.pitch = plane_pitch; a.n = gen->n_levels; a.NC = gen->n_classes; a.pin_thresh = gen->pin_thresh;
    a.q0_table = gen->q0_table; a.ratio_table = gen->ratio_table; a.tokens = tokens; a.flags = flags;
    int launches = 0;
    sprout_status st = cuda_status(launch_generate(a, reinterpret_cast<cudaStream_t>(stream), &launches));
    if (st == SPROUT_OK) g_last_launches = launches;
    return st;
}

int32_t sprout_last_launch_count(void) { return g_last_launches; }

const char *sprout_status_string(sprout_status status) {
    switch (status) {
        case SPROUT_OK: return "ok";
        case SPROUT_ERR_INVALID_ARGUMENT: return "invalid argument";
        case SPROUT_ERR_INFEASIBLE: return "infeasible cell";
        case SPROUT_ERR_OVERFLOW: return "size overflow";
        case SPROUT_ERR_CUDA: return "CUDA error";
        case SPROUT_ERR_INVALID_CELL: return "invalid cell input";
    }
    return "unknown status";
}

}  // extern "C"
