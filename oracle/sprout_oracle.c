/*
 * sprout_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the Sprout hot path
 * (arXiv 2403.12900): quality floor (Eq. 3), expected-carbon cost vector
 * (Eq. 2 + PUE), the directive LP (Eqs. 4-7) solved by enumerating the
 * vertices of its feasible polytope, inverse-CDF directive selection from the
 * solved mix, and per-request carbon accounting (Eq. 1) summed sequentially.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or constant generator with the CUDA path in paper_2403_12900_b200/.
 *
 * Citations: P:<line> = /root/reference/PAPER.md line, S:<line> = SPEC.md
 * line (SPEC binds only its own CPU program; used for worked examples).
 * Every reading of a silent/ambiguous passage is listed in DESIGN.md
 * ("Readings"), named L1..L16 as in SURVEY.md section 8(c).
 *
 * Build: gcc -O2 -std=c11 -fPIC -shared -ffp-contract=off -fno-fast-math -pthread
 * (-ffp-contract=off: no FMA contraction, reading L7.)
 *
 * Parity status: every function below is pinned by tests in tests/ against
 * something other than itself (Random123 known-answer vectors, the paper's
 * and SPEC's worked examples, exact-rational vertex brute force, SciPy HiGHS
 * dual simplex, a simplex grid, closed forms and invariants).  None is
 * "parity unpinned".
 */
#include <math.h>
#include <float.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define ORC_MAX_LEVELS 8
#define ORC_MAX_CLASSES 4

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11 "Parallel random numbers:
 * as easy as 1, 2, 3"; the Random123 reference constants).  The paper only
 * says x_i is "the probability of applying the i-th directive level"
 * (P:181); the counter-based mechanism is reading L10.                       */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {                 /* key schedule: bump before rounds 2..10 */
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t prod0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t prod1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(prod0 >> 32), lo0 = (uint32_t)prod0;
        uint32_t hi1 = (uint32_t)(prod1 >> 32), lo1 = (uint32_t)prod1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* The selection draw of global request g (reading L10):
 * key = (seed lo32, seed hi32); counter = (g>>2 lo32, g>>2 hi32, 0, 0)
 * (stream 0 = selection); request g takes output word g & 3.                */
uint32_t orc_draw_word(uint64_t seed, uint64_t g)
{
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    uint64_t blk = g >> 2;
    uint32_t ctr[4] = { (uint32_t)blk, (uint32_t)(blk >> 32), 0u, 0u };
    uint32_t out[4];
    orc_philox4x32_10(ctr, key, out);
    return out[g & 3u];
}

/* ------------------------------------------------------------------------ */
/* Eq. 3: q_lb = (1 - (k0 - k0min)/(k0max - k0min) * xi) * q0.
 * Reading L3: the fraction is clamped to [0,1] and defined as 0 when
 * k0max <= k0min.  Evaluation order (reading L7): f = (k0-kmin)/(kmax-kmin);
 * clamp; t = f*xi; u = 1 - t; b = u*q0.                                      */
double orc_quality_lower_bound(double k0, double kmin, double kmax, double xi, double q0)
{
    double f;
    if (kmax > kmin) {
        f = (k0 - kmin) / (kmax - kmin);
        if (f < 0.0) f = 0.0;
        if (f > 1.0) f = 1.0;
    } else {
        f = 0.0;
    }
    double t = f * xi;
    double u = 1.0 - t;
    return u * q0;
}

/* Eq. 2 with the PUE multiplier of P:153 on the operational term
 * (reading L2): c_i = (k0*PUE)*e_i + k1*p_i, the expected gCO2 of one request
 * at level i (Eq. 1, with E = e_i, T = p_i).                        */
void orc_cost_vector(int n, double k0, double pue, double k1,
                     const double *e, const double *p, double *c)
{
    double kp = k0 * pue;
    for (int i = 0; i < n; ++i) {
        double op = kp * e[i];
        double em = k1 * p[i];
        c[i] = op + em;
    }
}

/* Eq. 1 for one request: C = CI*PUE*E + (CO2_embed/T_life)*T.
 * kp = k0*PUE is computed by the caller once per interval.                  */
double orc_request_carbon(double kp, double k1, double energy_kwh, double time_s)
{
    double op = kp * energy_kwh;
    double em = k1 * time_s;
    return op + em;
}

/* ------------------------------------------------------------------------ */
/* The LP of Eqs. 4-7:  min c.x  s.t.  q.x >= b, 0 <= x_i <= 1,
 * sum x = 1.  The feasible set is the unit simplex cut by one half-space, so
 * its vertices are (i) the pure levels e_i with q_i >= b and (ii) for every
 * pair i<j whose q strictly straddles b, the point on edge (e_i, e_j) where
 * q.x = b.  An LP attains its minimum at a vertex, so enumerating them in a
 * fixed order and keeping the first strict minimum IS the LP solution with
 * a fixed tie-break (readings L6, L8).  Edge arithmetic, reading L7:
 *   h = higher-q end, l = lower-q end; kept only if c_l < c_h (otherwise the
 *   pure vertex h, enumerated earlier, is at least as cheap);
 *   x_h = (b - q_l)/(q_h - q_l);  x_l = 1 - x_h;  obj = c_l + (c_h - c_l)*x_h.
 * Vertex ids: pure i -> i; edge (i,j) -> n + (lexicographic index of (i,j)).
 * Returns 0 (ok) or 2 (infeasible: no vertex; impossible when b <= q0).     */
int orc_solve_lp(int n, const double *c, const double *q, double b,
                 double *x, double *obj, int *vertex)
{
    double best = INFINITY;
    int best_id = -1, best_i = -1, best_j = -1;
    double best_xi = 0.0, best_xj = 0.0;

    for (int i = 0; i < n; ++i) {                  /* pure vertices, ascending */
        if (q[i] >= b) {
            if (c[i] < best) {
                best = c[i]; best_id = i; best_i = i; best_j = -1;
            }
        }
    }
    int edge_id = 0;
    for (int i = 0; i < n; ++i) {                  /* edges, lexicographic */
        for (int j = i + 1; j < n; ++j, ++edge_id) {
            int straddle = (q[i] < b && q[j] > b) || (q[i] > b && q[j] < b);
            if (!straddle) continue;
            int h = (q[i] > q[j]) ? i : j;
            int l = (h == i) ? j : i;
            if (!(c[l] < c[h])) continue;
            double xh = (b - q[l]) / (q[h] - q[l]);
            double xl = 1.0 - xh;
            double o = c[l] + (c[h] - c[l]) * xh;
            if (o < best) {
                best = o; best_id = n + edge_id;
                best_i = h; best_j = l; best_xi = xh; best_xj = xl;
            }
        }
    }
    if (best_id < 0) {
        for (int i = 0; i < n; ++i) x[i] = NAN;
        *obj = NAN;
        *vertex = 255;
        return 2;
    }
    for (int i = 0; i < n; ++i) x[i] = 0.0;
    if (best_j < 0) {
        x[best_i] = 1.0;
    } else {
        x[best_i] = best_xi;
        x[best_j] = best_xj;
    }
    *obj = best;
    *vertex = best_id;
    return 0;
}

/* Inverse-CDF thresholds of the solved mix ("probability of selecting
 * each directive level"; reading L10): cum_i = sum_{k<=i} x_k added
 * sequentially in fp64, T_i = min(ceil(cum_i * 2^32), 2^32) for i <= n-2,
 * max_level = first i with T_i = 2^32, else n-1.  T is returned unsaturated
 * as uint64 (value up to 2^32).                                             */
void orc_thresholds(int n, const double *x, uint64_t *T, int *max_level)
{
    double cum = 0.0;
    int ml = n - 1, found = 0;
    for (int i = 0; i + 1 < n; ++i) {
        cum = cum + x[i];
        double scaled = ldexp(cum, 32);           /* exact: power-of-two scale */
        double cl = ceil(scaled);
        uint64_t t = (cl >= 4294967296.0) ? (uint64_t)4294967296ull : (uint64_t)cl;
        T[i] = t;
        if (t == 4294967296ull && !found) { ml = i; found = 1; }
    }
    *max_level = ml;
}

/* Directive selector (P:162 selector (1)), the plain
 * inverse-CDF definition: with u = w * 2^-32, the level is the smallest
 * i <= n-2 with u < cum_i, else n-1.  A pinned (opted-out) user always gets
 * L0.                                                    */
int orc_select_level(int n, const double *x, uint32_t w, int pinned)
{
    if (pinned) return 0;
    double u = ldexp((double)w, -32);
    double cum = 0.0;
    for (int i = 0; i + 1 < n; ++i) {
        cum = cum + x[i];
        if (u < cum) return i;
    }
    return n - 1;
}

/* ------------------------------------------------------------------------ */
/* Competing schemes of the evaluation.
 * Base (all requests at L0) is the per-segment counterfactual that
 * every run already reports.  The other two set the mix x per cell:        */
#define ORC_SCHEME_SPROUT 0
#define ORC_SCHEME_CO2_OPT 1
#define ORC_SCHEME_STATIC_GRID 2

/* CO2_Opt: "always use the generation directive level that
 * yields the lowest carbon footprint", i.e. x = e_m with m = argmin_i c_i of
 * the Eq. 2 cost vector; ties to the lowest index (reading L17).           */
int orc_co2opt_level(int n, const double *c)
{
    int m = 0;
    for (int i = 1; i < n; ++i)
        if (c[i] < c[m]) m = i;
    return m;
}

/* Sprout_Sta: "a single, month-long optimal generation directive
 * configuration ... determined by sweeping the possible static
 * configurations".  The swept configurations are the points of the simplex
 * grid of step 1/D (reading L18): every (k_0..k_{n-1}) of non-negative
 * integers with sum D, x_i = k_i / D, listed by k_0 descending, then k_1
 * descending, ..., k_{n-1} = the remainder (point 0 = pure L0).  Written as
 * the plain enumeration: walk the list in that order until point j.         */
static int grid_walk(int i, int n, int rem, int64_t *j, int *k)
{
    if (i == n - 1) {
        k[i] = rem;
        if (*j == 0) return 1;
        --*j;
        return 0;
    }
    for (int v = rem; v >= 0; --v) {
        k[i] = v;
        if (grid_walk(i + 1, n, rem - v, j, k)) return 1;
    }
    return 0;
}

/* Number of grid points C(D + n - 1, n - 1), counted by walking the list. */
int64_t orc_grid_size(int n, int D)
{
    int64_t cnt = 0;
    int k[ORC_MAX_LEVELS];
    for (;;) {
        int64_t j = cnt;
        if (!grid_walk(0, n, D, &j, k)) return cnt;
        ++cnt;
    }
}

/* Point j of the grid: x_i = k_i / D (IEEE division).  Returns 0, or 1 if j
 * is past the end.                                                          */
int orc_grid_point(int n, int D, int64_t j, double *x)
{
    int k[ORC_MAX_LEVELS];
    int64_t jj = j;
    if (j < 0 || !grid_walk(0, n, D, &jj, k)) return 1;
    for (int i = 0; i < n; ++i) x[i] = (double)k[i] / (double)D;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Per-cell input validation (SURVEY 8(b) cell_status code 1).               */
static int finite_nonneg(double v) { return v >= 0.0 && v <= DBL_MAX; }

static int cell_inputs_valid(int n, double k0, double kmin, double kmax, double xi,
                             const double *e, const double *p, const double *q)
{
    if (!(xi >= 0.0 && xi <= 1.0)) return 0;
    if (!finite_nonneg(k0) || !finite_nonneg(kmin) || !finite_nonneg(kmax)) return 0;
    if (!(kmax >= kmin)) return 0;
    for (int i = 0; i < n; ++i) {
        if (!(q[i] >= 0.0 && q[i] <= 1.0)) return 0;
        if (!finite_nonneg(e[i]) || !finite_nonneg(p[i])) return 0;
    }
    return 1;
}

typedef struct {
    int n, R, X, ppi, n_classes;
    int64_t T;
    const double *k0, *kmin, *kmax, *xi, *e, *p, *q;
    double k1, pue;
    int scheme, grid_den;   /* ORC_SCHEME_*; grid_den = D of the static grid */
} orc_problem;

static const double *prof(const orc_problem *P, const double *base, int64_t seg)
{
    int64_t row = P->ppi ? seg : seg / P->T;
    return base + row * P->n;
}

/* One LP cell (segment seg = r*T + t, quality coefficient index j).
 * Returns the cell status: 0 ok, 1 invalid input, 2 infeasible.             */
static int solve_cell(const orc_problem *P, int64_t seg, int j,
                      double *x, double *obj, double *qlb, int *vertex,
                      uint64_t *T, int *max_level)
{
    int n = P->n;
    int64_t r = seg / P->T;
    double k0 = P->k0[seg], kmin = P->kmin[r], kmax = P->kmax[r];
    double xi = P->scheme == ORC_SCHEME_SPROUT ? P->xi[j] : 0.0;   /* other schemes have no xi */
    const double *e = prof(P, P->e, seg), *p = prof(P, P->p, seg), *q = prof(P, P->q, seg);
    if (!cell_inputs_valid(n, k0, kmin, kmax, xi, e, p, q)) {
        for (int i = 0; i < n; ++i) x[i] = NAN;
        *obj = NAN; *qlb = NAN; *vertex = 255;
        for (int i = 0; i + 1 < n; ++i) T[i] = 4294967296ull;
        *max_level = 0;
        return 1;
    }
    double c[ORC_MAX_LEVELS];
    orc_cost_vector(n, k0, P->pue, P->k1, e, p, c);
    if (P->scheme != ORC_SCHEME_SPROUT) {
        /* CO2_Opt: the cheapest pure level; Sprout_Sta: grid point j.  No
         * quality floor: q_lb reports the mix's expected quality q.x and the
         * objective its expected carbon c.x, both summed in level order.     */
        if (P->scheme == ORC_SCHEME_CO2_OPT) {
            int m = orc_co2opt_level(n, c);
            for (int i = 0; i < n; ++i) x[i] = (i == m) ? 1.0 : 0.0;
            *vertex = m;
        } else {
            orc_grid_point(n, P->grid_den, j, x);
            int nz = 0, last = 0;
            for (int i = 0; i < n; ++i) if (x[i] != 0.0) { ++nz; last = i; }
            *vertex = nz == 1 ? last : 254;
        }
        double o = 0.0, qx = 0.0;
        for (int i = 0; i < n; ++i) { o = o + c[i] * x[i]; qx = qx + q[i] * x[i]; }
        *obj = o;
        *qlb = qx;
        orc_thresholds(n, x, T, max_level);
        return 0;
    }
    double b = orc_quality_lower_bound(k0, kmin, kmax, xi, q[0]);
    *qlb = b;
    int st = orc_solve_lp(n, c, q, b, x, obj, vertex);
    if (st != 0) {
        for (int i = 0; i + 1 < n; ++i) T[i] = 4294967296ull;
        *max_level = 0;
        return st;
    }
    orc_thresholds(n, x, T, max_level);
    return 0;
}

/* All cells of segments [first_segment, first_segment + n_segments), cell
 * index (s - first_segment)*X + j (reading: xi innermost, SURVEY 8 notation).
 * Returns 0, or 1 on invalid scalar arguments.                              */
static int scheme_args_ok(int n, int X, int scheme, int grid_den)
{
    if (scheme == ORC_SCHEME_SPROUT || scheme == ORC_SCHEME_CO2_OPT) return 1;
    if (scheme != ORC_SCHEME_STATIC_GRID || grid_den < 1) return 0;
    return orc_grid_size(n, grid_den) == X;   /* one cell per grid point */
}

int orc_solve_cells_scheme(int n, int R, int64_t T, int X,
                    const double *k0, const double *kmin, const double *kmax, const double *xi,
                    const double *e, const double *p, const double *q, int profile_per_interval,
                    double k1, double pue, int64_t first_segment, int64_t n_segments,
                    double *x, double *objective, double *q_lb, uint8_t *vertex,
                    uint64_t *threshold, uint8_t *max_level, uint8_t *cell_status,
                    int scheme, int grid_den)
{
    if (n < 1 || n > ORC_MAX_LEVELS || R < 1 || T < 1 || X < 1) return 1;
    if (!(pue >= 1.0 && pue <= DBL_MAX) || !(k1 >= 0.0 && k1 <= DBL_MAX)) return 1;
    if (first_segment < 0 || n_segments < 0 || first_segment + n_segments > (int64_t)R * T) return 1;
    if (!scheme_args_ok(n, X, scheme, grid_den)) return 1;
    orc_problem P = { n, R, X, profile_per_interval, 1, T, k0, kmin, kmax, xi, e, p, q, k1, pue,
                      scheme, grid_den };
    for (int64_t s = 0; s < n_segments; ++s) {
        for (int j = 0; j < X; ++j) {
            int64_t cell = s * X + j;
            int vid, ml;
            uint64_t Tl[ORC_MAX_LEVELS];
            int st = solve_cell(&P, first_segment + s, j, x + cell * n, objective + cell,
                                q_lb + cell, &vid, Tl, &ml);
            vertex[cell] = (uint8_t)vid;
            max_level[cell] = (uint8_t)ml;
            cell_status[cell] = (uint8_t)st;
            for (int i = 0; i + 1 < n; ++i) threshold[cell * (n - 1) + i] = Tl[i];
        }
    }
    return 0;
}

int orc_solve_cells(int n, int R, int64_t T, int X,
                    const double *k0, const double *kmin, const double *kmax, const double *xi,
                    const double *e, const double *p, const double *q, int profile_per_interval,
                    double k1, double pue, int64_t first_segment, int64_t n_segments,
                    double *x, double *objective, double *q_lb, uint8_t *vertex,
                    uint64_t *threshold, uint8_t *max_level, uint8_t *cell_status)
{
    return orc_solve_cells_scheme(n, R, T, X, k0, kmin, kmax, xi, e, p, q, profile_per_interval, k1, pue,
                                  first_segment, n_segments, x, objective, q_lb, vertex, threshold,
                                  max_level, cell_status, ORC_SCHEME_SPROUT, 0);
}

/* ------------------------------------------------------------------------ */
/* Trace replay of selected segments.  For every request of a segment, in
 * index order: draw w (L10), read pinned/class flags (reading L11),
 * and for every cell of the segment select the level, evaluate the
 * request's energy E = ef + et*tok and time T = pf + pt*tok (P:87-98 linear
 * in generated tokens; reading L11), its carbon C = (k0*PUE)*E + k1*T
 * (Eq. 1, reading L2), and add to the cell's running fp64 sums in
 * request order (reading L16).  Also: integer counts and token sums per
 * (cell, class, level), the per-segment Base counterfactual (all requests at
 * L0), and the realised quality sum q[level] (reading L15).   */
typedef struct {
    const orc_problem *P;
    uint64_t seed;
    const double *ef, *et, *pf, *pt;   /* [4][8] */
    const int64_t *seg_id, *req_begin, *seg_m;
    const uint64_t *g0;
    const uint16_t *tokens; int64_t pitch;
    const uint8_t *flags;
    uint64_t *cnt, *tok;
    double *energy, *time_s, *carbon, *quality;
    uint64_t *seg_count, *seg_pinned, *seg_tok;
    double *seg_base;
    uint8_t *levels_out;
    int64_t lo, hi;
    int64_t bad_requests;
} sim_job;

static void simulate_segment(sim_job *J, int64_t k)
{
    const orc_problem *P = J->P;
    const int n = P->n, X = P->X, NC = P->n_classes;
    const int64_t seg = J->seg_id[k];
    const int64_t m = J->seg_m[k], rb = J->req_begin[k];
    const uint64_t g0 = J->g0[k];
    const double kp = P->k0[seg] * P->pue;
    const double *q = prof(P, P->q, seg);

    double *xs = (double *)malloc(sizeof(double) * (size_t)X * n);
    int *ok = (int *)malloc(sizeof(int) * (size_t)X);
    for (int j = 0; j < X; ++j) {
        double obj, qlb; int vid, ml; uint64_t Tl[ORC_MAX_LEVELS];
        ok[j] = solve_cell(P, seg, j, xs + (size_t)j * n, &obj, &qlb, &vid, Tl, &ml) == 0;
    }
    uint64_t *cnt = J->cnt + (size_t)k * X * NC * n;
    uint64_t *tok = J->tok + (size_t)k * X * NC * n;
    double *E = J->energy + (size_t)k * X, *Tm = J->time_s + (size_t)k * X;
    double *Cb = J->carbon + (size_t)k * X, *Q = J->quality + (size_t)k * X;
    uint64_t *sc = J->seg_count + (size_t)k * NC, *sp = J->seg_pinned + (size_t)k * NC;
    uint64_t *st = J->seg_tok + (size_t)k * NC * n;
    double *base = J->seg_base + (size_t)k * 4;
    memset(cnt, 0, sizeof(uint64_t) * (size_t)X * NC * n);
    memset(tok, 0, sizeof(uint64_t) * (size_t)X * NC * n);
    for (int j = 0; j < X; ++j) { E[j] = 0.0; Tm[j] = 0.0; Cb[j] = 0.0; Q[j] = 0.0; }
    memset(sc, 0, sizeof(uint64_t) * NC);
    memset(sp, 0, sizeof(uint64_t) * NC);
    memset(st, 0, sizeof(uint64_t) * NC * n);
    base[0] = base[1] = base[2] = base[3] = 0.0;

    for (int64_t r = 0; r < m; ++r) {
        const int64_t ri = rb + r;
        const uint64_t g = g0 + (uint64_t)r;
        const uint32_t w = orc_draw_word(J->seed, g);
        int pinned = 0, cls = 0;
        if (J->flags) {
            uint8_t f = J->flags[ri];
            pinned = f & 1;
            cls = (f >> 1) & 3;
        }
        if (cls >= NC) {                                /* invalid class: skipped */
            J->bad_requests++;
            if (J->levels_out)
                for (int j = 0; j < X; ++j) J->levels_out[(size_t)j * J->pitch + ri] = 0xFF;
            continue;
        }
        uint32_t t[ORC_MAX_LEVELS];
        for (int i = 0; i < n; ++i) t[i] = J->tokens[(size_t)i * J->pitch + ri];

        /* Base: every request at L0 */
        {
            double e0 = J->ef[cls * 8 + 0] + J->et[cls * 8 + 0] * (double)t[0];
            double p0 = J->pf[cls * 8 + 0] + J->pt[cls * 8 + 0] * (double)t[0];
            base[0] += e0;
            base[1] += p0;
            base[2] += orc_request_carbon(kp, P->k1, e0, p0);
            base[3] += q[0];
        }
        sc[cls] += 1;
        sp[cls] += (uint64_t)pinned;
        for (int i = 0; i < n; ++i) st[cls * n + i] += t[i];

        for (int j = 0; j < X; ++j) {
            if (!ok[j]) {
                if (J->levels_out) J->levels_out[(size_t)j * J->pitch + ri] = 0xFF;
                continue;
            }
            int L = orc_select_level(n, xs + (size_t)j * n, w, pinned);
            double el = J->ef[cls * 8 + L] + J->et[cls * 8 + L] * (double)t[L];
            double pl = J->pf[cls * 8 + L] + J->pt[cls * 8 + L] * (double)t[L];
            E[j] += el;
            Tm[j] += pl;
            Cb[j] += orc_request_carbon(kp, P->k1, el, pl);
            Q[j] += q[L];
            cnt[((size_t)j * NC + cls) * n + L] += 1;
            tok[((size_t)j * NC + cls) * n + L] += t[L];
            if (J->levels_out) J->levels_out[(size_t)j * J->pitch + ri] = (uint8_t)L;
        }
    }
    free(xs);
    free(ok);
}

static void *sim_worker(void *arg)
{
    sim_job *J = (sim_job *)arg;
    for (int64_t k = J->lo; k < J->hi; ++k) simulate_segment(J, k);
    return NULL;
}

/* Returns 0 ok, 1 invalid argument.  *bad_requests = requests skipped because
 * their class index (flags bits 1-2) is >= n_classes.                       */
int orc_simulate_scheme(int n, int R, int64_t T, int X,
                 const double *k0, const double *kmin, const double *kmax, const double *xi,
                 const double *e, const double *p, const double *q, int profile_per_interval,
                 double k1, double pue,
                 uint64_t seed, int n_classes, const double *ef, const double *et,
                 const double *pf, const double *pt,
                 int64_t n_sel, const int64_t *seg_id, const int64_t *req_begin,
                 const int64_t *seg_m, const uint64_t *g0,
                 const uint16_t *tokens, int64_t pitch, const uint8_t *flags,
                 uint64_t *cnt, uint64_t *tok, double *energy, double *time_s,
                 double *carbon, double *quality,
                 uint64_t *seg_count, uint64_t *seg_pinned, uint64_t *seg_tok, double *seg_base,
                 uint8_t *levels_out, int n_threads, int64_t *bad_requests, int scheme, int grid_den)
{
    if (n < 1 || n > ORC_MAX_LEVELS || R < 1 || T < 1 || X < 1) return 1;
    if (n_classes < 1 || n_classes > ORC_MAX_CLASSES) return 1;
    if (!scheme_args_ok(n, X, scheme, grid_den)) return 1;
    if (!(pue >= 1.0 && pue <= DBL_MAX) || !(k1 >= 0.0 && k1 <= DBL_MAX)) return 1;
    for (int64_t k = 0; k < n_sel; ++k)
        if (seg_id[k] < 0 || seg_id[k] >= (int64_t)R * T || seg_m[k] < 0) return 1;
    orc_problem P = { n, R, X, profile_per_interval, n_classes, T, k0, kmin, kmax, xi, e, p, q, k1, pue,
                      scheme, grid_den };
    if (n_threads < 1) n_threads = 1;
    if (n_threads > 256) n_threads = 256;
    if (n_sel < n_threads) n_threads = n_sel > 0 ? (int)n_sel : 1;

    sim_job jobs[256];
    pthread_t th[256];
    for (int t = 0; t < n_threads; ++t) {
        sim_job J = { &P, seed, ef, et, pf, pt, seg_id, req_begin, seg_m, g0, tokens, pitch, flags,
                      cnt, tok, energy, time_s, carbon, quality, seg_count, seg_pinned, seg_tok,
                      seg_base, levels_out, n_sel * t / n_threads, n_sel * (t + 1) / n_threads, 0 };
        jobs[t] = J;
    }
    if (n_threads == 1) {
        sim_worker(&jobs[0]);
    } else {
        for (int t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, sim_worker, &jobs[t]);
        for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
    }
    int64_t bad = 0;
    for (int t = 0; t < n_threads; ++t) bad += jobs[t].bad_requests;
    if (bad_requests) *bad_requests = bad;
    return 0;
}

int orc_simulate(int n, int R, int64_t T, int X,
                 const double *k0, const double *kmin, const double *kmax, const double *xi,
                 const double *e, const double *p, const double *q, int profile_per_interval,
                 double k1, double pue,
                 uint64_t seed, int n_classes, const double *ef, const double *et,
                 const double *pf, const double *pt,
                 int64_t n_sel, const int64_t *seg_id, const int64_t *req_begin,
                 const int64_t *seg_m, const uint64_t *g0,
                 const uint16_t *tokens, int64_t pitch, const uint8_t *flags,
                 uint64_t *cnt, uint64_t *tok, double *energy, double *time_s,
                 double *carbon, double *quality,
                 uint64_t *seg_count, uint64_t *seg_pinned, uint64_t *seg_tok, double *seg_base,
                 uint8_t *levels_out, int n_threads, int64_t *bad_requests)
{
    return orc_simulate_scheme(n, R, T, X, k0, kmin, kmax, xi, e, p, q, profile_per_interval, k1, pue, seed,
                               n_classes, ef, et, pf, pt, n_sel, seg_id, req_begin, seg_m, g0, tokens, pitch,
                               flags, cnt, tok, energy, time_s, carbon, quality, seg_count, seg_pinned, seg_tok,
                               seg_base, levels_out, n_threads, bad_requests, ORC_SCHEME_SPROUT, 0);
}

/* ------------------------------------------------------------------------ */
/* Group totals (conservation S:485): per (region, xi) and per
 * xi, summed sequentially over cells in (region, interval) order.  Stats
 * k = 0..K-1 with K = 11 + 2n:
 *   0 requests, 1 pinned, 2 energy kWh, 3 time s, 4 carbon g, 5 quality
 *   (sum q[level]), 6..9 Base energy/time/carbon/quality (all-L0),
 *   10 expected carbon (m * LP objective, Eq. 2), 11..11+n-1 requests per
 *   level, 11+n..11+2n-1 generated tokens per level.
 * Inputs are this oracle's own per-cell / per-segment results for ALL
 * segments [first_segment, first_segment + n_segments).  Output layout:
 * group[R][X][K] followed by global[X][K]; rows of regions outside the
 * segment range are zero.                                                   */
int orc_reduce(int n, int R, int64_t T, int X, int n_classes,
               int64_t first_segment, int64_t n_segments,
               const uint8_t *cell_status, const double *objective,
               const uint64_t *cnt, const uint64_t *tok, const double *energy,
               const double *time_s, const double *carbon, const double *quality,
               const uint64_t *seg_count, const uint64_t *seg_pinned, const double *seg_base,
               double *out)
{
    const int K = 11 + 2 * n;
    const int NC = n_classes;
    memset(out, 0, sizeof(double) * (size_t)(R + 1) * X * K);
    for (int64_t s = 0; s < n_segments; ++s) {
        int64_t r = (first_segment + s) / T;
        double m = 0.0, pin = 0.0;
        for (int c = 0; c < NC; ++c) { m += (double)seg_count[s * NC + c]; pin += (double)seg_pinned[s * NC + c]; }
        for (int j = 0; j < X; ++j) {
            int64_t cell = s * X + j;
            double *G = out + ((size_t)r * X + j) * K;
            G[0] += m;
            G[1] += pin;
            G[6] += seg_base[s * 4 + 0];
            G[7] += seg_base[s * 4 + 1];
            G[8] += seg_base[s * 4 + 2];
            G[9] += seg_base[s * 4 + 3];
            if (cell_status[cell] != 0) continue;
            G[2] += energy[cell];
            G[3] += time_s[cell];
            G[4] += carbon[cell];
            G[5] += quality[cell];
            G[10] += m * objective[cell];
            for (int L = 0; L < n; ++L) {
                double cL = 0.0, tL = 0.0;
                for (int c = 0; c < NC; ++c) {
                    cL += (double)cnt[(cell * NC + c) * n + L];
                    tL += (double)tok[(cell * NC + c) * n + L];
                }
                G[11 + L] += cL;
                G[11 + n + L] += tL;
            }
        }
    }
    double *glob = out + (size_t)R * X * K;
    for (int r = 0; r < R; ++r)
        for (int j = 0; j < X; ++j)
            for (int k = 0; k < K; ++k)
                glob[(size_t)j * K + k] += out[((size_t)r * X + j) * K + k];
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Sprout_Sta selection (reading L18).  For every region r, from
 * the group totals of a sweep over the G grid points (orc_reduce layout,
 * [R+1][G][K]): the region's floor is Eq. 3 at its mean carbon intensity,
 * b_r = orc_quality_lower_bound(mean_t k0[r][t], kmin_r, kmax_r, xi, q0_r)
 * (mean = sequential sum / T); grid point g meets it iff its realised
 * quality sum_L (requests at level L) * q_L >= b_r * (requests); the choice
 * is the feasible point of least realised carbon (stat 4), ties to the
 * lowest g.  Point 0 (pure L0) is always feasible.  q is per region [R][n].
 * Outputs choice[R] and x[R][n].  Returns 0, or 1 on invalid arguments.     */
int orc_select_static(int n, int R, int64_t T, const double *k0, const double *kmin,
                      const double *kmax, const double *q, double xi, int grid_den,
                      int64_t G, const double *group, int32_t *choice, double *x)
{
    if (n < 1 || n > ORC_MAX_LEVELS || R < 1 || T < 1 || grid_den < 1) return 1;
    if (orc_grid_size(n, grid_den) != G) return 1;
    const int K = 11 + 2 * n;
    for (int r = 0; r < R; ++r) {
        double sum = 0.0;
        for (int64_t t = 0; t < T; ++t) sum = sum + k0[(int64_t)r * T + t];
        double kbar = sum / (double)T;
        const double *qr = q + (size_t)r * n;
        double b = orc_quality_lower_bound(kbar, kmin[r], kmax[r], xi, qr[0]);
        int64_t best = -1;
        double best_c = 0.0;
        for (int64_t g = 0; g < G; ++g) {
            const double *S = group + ((size_t)r * G + g) * K;
            double Q = 0.0;
            for (int L = 0; L < n; ++L) Q = Q + S[11 + L] * qr[L];
            if (!(Q >= b * S[0])) continue;
            if (best < 0 || S[4] < best_c) { best = g; best_c = S[4]; }
        }
        if (best < 0) best = 0;
        choice[r] = (int32_t)best;
        orc_grid_point(n, grid_den, best, x + (size_t)r * n);
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Opportunistic evaluator trigger sweep (Eq. 8; reading L19).
 * For each (region r, beta b, theta h), scan t = 1..T-1 in order with the
 * state of the last evaluation t0 (the trace start counts as one):
 *   Eq. 8, urgency-adjusted intensity k'(t) = e^{-beta (t - t0)} k2(t), the
 *   factor kept as d^(t - t0) by repeated multiplication, d = exp(-beta*dt);
 *   evaluate at t iff (ii) the grace period has elapsed, (t - t0)*dt >= grace;
 *   (iii) k'(t) < theta * k2max_r ("below a predefined threshold, such as
 *   50% of the historical maximum"); and (i) t-1 was a local minimum of k'
 *   (k'(t-1) < k'(t-2), k'(t) > k'(t-1), with t-2 >= t0), or the last F
 *   samples after t0 were all below the threshold (fallback; Fig. 4(b)).
 * An evaluation costs k2(t) * pue * eval_kwh gCO2 (16 GPUs x 250 W x 0.5 s x
 * 500 samples in SURVEY's accounting is the caller's eval_kwh).
 * out[r][b][h] = {evaluations, carbon g, longest gap h (trace start and end
 * included), sum of k2 at the evaluations}.                                 */
int orc_evaluator_sweep(int R, int64_t T, double dt, const double *k2, const double *k2max,
                        int B, const double *beta, int H, const double *theta,
                        double grace, int F, double eval_kwh, double pue, double *out)
{
    if (R < 1 || T < 1 || B < 1 || H < 1 || F < 0 || !(dt > 0.0)) return 1;
    for (int r = 0; r < R; ++r)
        for (int b = 0; b < B; ++b)
            for (int h = 0; h < H; ++h) {
                const double *k = k2 + (int64_t)r * T;
                double d = exp(-(beta[b] * dt));
                double thr = theta[h] * k2max[r];
                int64_t t0 = 0;
                double f = 1.0;
                /* k'(s) for the samples s since t0, recomputed from the definition */
                double prev1 = k[0], prev2 = 0.0;
                int64_t below = 0, gap = 0;
                double n_eval = 0.0, carbon = 0.0, sum_k2 = 0.0;
                for (int64_t t = 1; t < T; ++t) {
                    f = f * d;
                    double kp = f * k[t];
                    int under = kp < thr;
                    if (under) below = below + 1; else below = 0;
                    int64_t since = t - t0;
                    int grace_ok = (double)since * dt >= grace;
                    int local_min = since >= 2 && prev1 < prev2 && kp > prev1;
                    int fallback = F > 0 && below >= F;
                    prev2 = prev1;
                    prev1 = kp;
                    if (grace_ok && under && (local_min || fallback)) {
                        n_eval = n_eval + 1.0;
                        carbon = carbon + (k[t] * pue) * eval_kwh;
                        sum_k2 = sum_k2 + k[t];
                        if (since > gap) gap = since;
                        t0 = t;
                        f = 1.0;
                        prev1 = k[t];
                        below = 0;
                    }
                }
                if (T - t0 > gap) gap = T - t0;
                double *o = out + (((size_t)r * B + b) * H + h) * 4;
                o[0] = n_eval;
                o[1] = carbon;
                o[2] = (double)gap * dt;
                o[3] = sum_k2;
            }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Closed-loop profiles (reading L20).  P:183: the
 * optimiser's e and p are "the average energy consumption and processing
 * time for recent requests at each level".  Per (region r, xi_j) chain, in
 * interval order: the profile of level L is the mean of Eq. 1's E and T
 * over the last W requests executed at level L (by this chain, any class;
 * pinned requests count at L0), or the caller's prior e/p[r][L] while none
 * has run.  With E = ef[c][L] + et[c][L]*tok the mean is, from the window's
 * per-class request counts n_c and token sums k_c (exact integers):
 *   e_L = (sum_c (n_c*ef[c][L] + k_c*et[c][L])) / (sum_c n_c),
 * summed in class order (p_L likewise with pf, pt).  The LP of the interval
 * (solve_cell with these e, p and the region's q -- or interval s's row of
 * q_seg when given: the q of its evaluation epoch, reading L24) gives x and
 * thresholds;
 * then the interval's requests are replayed as in orc_simulate and pushed,
 * in request order, into their level's window.  Outputs per cell
 * (r*T + t)*X + j: the solution and the cell totals.  Requests: global
 * seg_offsets [R*T+1]; request g's tokens at tokens[L][g], flags[g].        */
int orc_closed_loop(int n, int R, int64_t T, int X,
                    const double *k0, const double *kmin, const double *kmax, const double *xi,
                    const double *e_prior, const double *p_prior, const double *q, double k1, double pue,
                    uint64_t seed, int n_classes, const double *ef, const double *et,
                    const double *pf, const double *pt, int W, const double *q_seg,
                    const int64_t *seg_offsets, const uint16_t *tokens, int64_t pitch, const uint8_t *flags,
                    double *x_out, uint64_t *thr_out, uint8_t *status_out, double *obj_out, double *prof_out,
                    uint64_t *cnt, uint64_t *tok, double *energy, double *time_s, double *carbon, double *quality)
{
    if (n < 1 || n > ORC_MAX_LEVELS || R < 1 || T < 1 || X < 1 || W < 1) return 1;
    if (n_classes < 1 || n_classes > ORC_MAX_CLASSES) return 1;
    const int NC = n_classes;
    int *ring_c = (int *)malloc(sizeof(int) * (size_t)n * W);
    uint32_t *ring_t = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)n * W);
    for (int r = 0; r < R; ++r) {
        for (int j = 0; j < X; ++j) {
            int head[ORC_MAX_LEVELS], size[ORC_MAX_LEVELS];
            uint64_t wn[ORC_MAX_LEVELS][ORC_MAX_CLASSES], wk[ORC_MAX_LEVELS][ORC_MAX_CLASSES];
            memset(wn, 0, sizeof(wn)); memset(wk, 0, sizeof(wk));
            for (int L = 0; L < n; ++L) { head[L] = 0; size[L] = 0; }
            for (int64_t t = 0; t < T; ++t) {
                const int64_t s = (int64_t)r * T + t;
                const int64_t cell = s * X + j;
                double e[ORC_MAX_LEVELS], p[ORC_MAX_LEVELS];
                for (int L = 0; L < n; ++L) {
                    uint64_t m = 0;
                    for (int c = 0; c < NC; ++c) m += wn[L][c];
                    if (m == 0) {
                        e[L] = e_prior[(size_t)r * n + L];
                        p[L] = p_prior[(size_t)r * n + L];
                    } else {
                        double se = 0.0, sp = 0.0;
                        for (int c = 0; c < NC; ++c) {
                            se = se + ((double)wn[L][c] * ef[c * 8 + L] + (double)wk[L][c] * et[c * 8 + L]);
                            sp = sp + ((double)wn[L][c] * pf[c * 8 + L] + (double)wk[L][c] * pt[c * 8 + L]);
                        }
                        e[L] = se / (double)m;
                        p[L] = sp / (double)m;
                    }
                }
                for (int L = 0; L < n; ++L) {          /* profiles used: [cell][2][n] */
                    prof_out[(cell * 2 + 0) * n + L] = e[L];
                    prof_out[(cell * 2 + 1) * n + L] = p[L];
                }
                /* the interval's LP with the closed-loop profile */
                const double *qs = q_seg ? &q_seg[(size_t)s * n] : &q[(size_t)r * n];   /* L24: q per epoch */
                orc_problem P = { n, R, 1, 0, NC, 1, &k0[s], &kmin[r], &kmax[r], &xi[j], e, p,
                                  qs, k1, pue, ORC_SCHEME_SPROUT, 0 };
                double xs[ORC_MAX_LEVELS], obj, qlb; int vid, ml; uint64_t Tl[ORC_MAX_LEVELS];
                int st = solve_cell(&P, 0, 0, xs, &obj, &qlb, &vid, Tl, &ml);
                obj_out[cell] = obj;
                for (int i = 0; i < n; ++i) x_out[cell * n + i] = xs[i];
                for (int i = 0; i + 1 < n; ++i) thr_out[cell * (n - 1) + i] = Tl[i];
                status_out[cell] = (uint8_t)st;
                uint64_t *cn = cnt + (size_t)cell * NC * n, *tk = tok + (size_t)cell * NC * n;
                memset(cn, 0, sizeof(uint64_t) * NC * n);
                memset(tk, 0, sizeof(uint64_t) * NC * n);
                double E = 0.0, Tm = 0.0, Cb = 0.0, Q = 0.0;
                const double kp = k0[s] * pue;
                if (st == 0) {
                    for (int64_t g = seg_offsets[s]; g < seg_offsets[s + 1]; ++g) {
                        const uint32_t w = orc_draw_word(seed, (uint64_t)g);
                        int pinned = 0, cls = 0;
                        if (flags) { pinned = flags[g] & 1; cls = (flags[g] >> 1) & 3; }
                        if (cls >= NC) continue;
                        const int L = orc_select_level(n, xs, w, pinned);
                        const uint32_t tl = tokens[(size_t)L * pitch + g];
                        const double el = ef[cls * 8 + L] + et[cls * 8 + L] * (double)tl;
                        const double pl = pf[cls * 8 + L] + pt[cls * 8 + L] * (double)tl;
                        E += el; Tm += pl; Cb += orc_request_carbon(kp, k1, el, pl); Q += qs[L];
                        cn[cls * n + L] += 1; tk[cls * n + L] += tl;
                        /* push into level L's window (FIFO of the last W) */
                        int slot = head[L];
                        if (size[L] == W) {
                            wn[L][ring_c[L * W + slot]] -= 1;
                            wk[L][ring_c[L * W + slot]] -= ring_t[L * W + slot];
                        } else {
                            size[L] += 1;
                        }
                        ring_c[L * W + slot] = cls;
                        ring_t[L * W + slot] = tl;
                        wn[L][cls] += 1;
                        wk[L][cls] += tl;
                        head[L] = (slot + 1) % W;
                    }
                }
                energy[cell] = E; time_s[cell] = Tm; carbon[cell] = Cb; quality[cell] = Q;
            }
        }
    }
    free(ring_c); free(ring_t);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* NEXT-4: the latent preferred level, head-to-head preference
 * against Base, per-request outputs, and the Oracle scheme.                 */

/* Reading L21.  The evaluator "generates responses for each [sampled prompt]
 * at all generation directive levels, and identifies the directive level that
 * yields the best response for each request"; q holds the preference
 * rates of those levels.  Synthetic ground truth: request g's latent
 * best level l*(g) is the inverse-CDF level of q -- the a4/a6 rules with q in
 * place of the mix x -- at the word of Philox stream 2: key (seed lo, seed
 * hi), counter (g>>2 lo32, g>>2 hi32, 2, 0), word g & 3.                     */
uint32_t orc_pref_word(uint64_t seed, uint64_t g)
{
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    uint64_t blk = g >> 2;
    uint32_t ctr[4] = { (uint32_t)blk, (uint32_t)(blk >> 32), 2u, 0u };
    uint32_t out[4];
    orc_philox4x32_10(ctr, key, out);
    return out[g & 3u];
}

int orc_pref_level(int n, const double *q, uint64_t seed, uint64_t g)
{
    return orc_select_level(n, q, orc_pref_word(seed, g), 0);
}

/* "if the auto-evaluator shows a preference for Sprout's responses 48%
 * of the time versus 52% for Base, Sprout's normalized generation preference
 * score would be 92.3%": score = w / (1 - w).  No finite score at w = 1.     */
double orc_normalized_preference(double w)
{
    return w >= 1.0 ? INFINITY : w / (1.0 - w);
}

/* Reading L22: the head-to-head of a scheme's response (level L) against
 * Base's (L0) for a request whose latent best level is l*: L = 0 gives
 * the identical response, a tie; otherwise the scheme wins iff l* = L, Base
 * wins iff l* = 0, and a third best level is a tie.  Ties count half:
 * w = (wins + ties/2) / m.                                                   */
void orc_head_to_head(int L, int lstar, int *win, int *loss)
{
    *win = (L != 0 && lstar == L);
    *loss = (L != 0 && lstar == 0);
}

/* Per-cell preference statistics of a scheme's run (levels by each cell's
 * mix, a6): stats[cell][0..2] = hits (L = l*, the realised Eq. 3 left-hand
 * side), wins, losses against Base.  Requests with an invalid class and
 * invalid cells are skipped.  Arguments as orc_simulate_scheme (all R*T
 * segments); requests indexed by seg_offsets, global index g0[s] + (i -
 * seg_offsets[s]) (g0 NULL: the index itself).                              */
int orc_preference(int n, int R, int64_t T, int X,
                   const double *k0, const double *kmin, const double *kmax, const double *xi,
                   const double *e, const double *p, const double *q, int profile_per_interval,
                   double k1, double pue, uint64_t seed, int n_classes,
                   const int64_t *seg_offsets, const uint64_t *g0, const uint8_t *flags, int scheme,
                   int grid_den, uint64_t *stats)
{
    if (n < 1 || n > ORC_MAX_LEVELS || R < 1 || T < 1 || X < 1) return 1;
    if (n_classes < 1 || n_classes > ORC_MAX_CLASSES) return 1;
    if (!scheme_args_ok(n, X, scheme, grid_den)) return 1;
    orc_problem P = { n, R, X, profile_per_interval, n_classes, T, k0, kmin, kmax, xi, e, p, q, k1, pue,
                      scheme, grid_den };
    double xs[ORC_MAX_LEVELS];
    for (int64_t s = 0; s < (int64_t)R * T; ++s) {
        const double *qs = prof(&P, q, s);
        for (int j = 0; j < X; ++j) {
            double obj, qlb; int vid, ml; uint64_t Tl[ORC_MAX_LEVELS];
            uint64_t *st = stats + ((size_t)s * X + j) * 3;
            st[0] = st[1] = st[2] = 0;
            if (solve_cell(&P, s, j, xs, &obj, &qlb, &vid, Tl, &ml) != 0) continue;
            for (int64_t i = seg_offsets[s]; i < seg_offsets[s + 1]; ++i) {
                const uint64_t g = g0 ? g0[s] + (uint64_t)(i - seg_offsets[s]) : (uint64_t)i;   /* global index */
                int pinned = 0, cls = 0;
                if (flags) { pinned = flags[i] & 1; cls = (flags[i] >> 1) & 3; }
                if (cls >= n_classes) continue;
                const int L = orc_select_level(n, xs, orc_draw_word(seed, g), pinned);
                const int ls = orc_pref_level(n, qs, seed, g);
                int win, loss;
                orc_head_to_head(L, ls, &win, &loss);
                st[0] += (uint64_t)(L == ls);
                st[1] += (uint64_t)win;
                st[2] += (uint64_t)loss;
            }
        }
    }
    return 0;
}

/* Per-request outputs of cell column j (one xi value) of a scheme's run:
 * for every request g of segments [0, R*T): its level, its carbon (Eq. 1,
 * P:50-54, at its segment's CI), the carbon it would have under Base (all
 * at L0), their ratio -- the per-request carbon normalised to Base of
 * Fig. eval2 -- and its latent best level.  Invalid class or cell:
 * level 0xFF, carbon and ratio NaN.                                         */
int orc_request_outputs(int n, int R, int64_t T, int X,
                        const double *k0, const double *kmin, const double *kmax, const double *xi,
                        const double *e, const double *p, const double *q, int profile_per_interval,
                        double k1, double pue, uint64_t seed, int n_classes,
                        const double *ef, const double *et, const double *pf, const double *pt,
                        const int64_t *seg_offsets, const uint64_t *g0, const uint16_t *tokens, int64_t pitch,
                        const uint8_t *flags, int scheme, int grid_den, int j,
                        uint8_t *level, double *carbon, double *base, double *ratio, uint8_t *pref)
{
    if (n < 1 || n > ORC_MAX_LEVELS || R < 1 || T < 1 || X < 1 || j < 0 || j >= X) return 1;
    if (n_classes < 1 || n_classes > ORC_MAX_CLASSES) return 1;
    if (!scheme_args_ok(n, X, scheme, grid_den)) return 1;
    orc_problem P = { n, R, X, profile_per_interval, n_classes, T, k0, kmin, kmax, xi, e, p, q, k1, pue,
                      scheme, grid_den };
    double xs[ORC_MAX_LEVELS];
    for (int64_t s = 0; s < (int64_t)R * T; ++s) {
        double obj, qlb; int vid, ml; uint64_t Tl[ORC_MAX_LEVELS];
        const int ok = solve_cell(&P, s, j, xs, &obj, &qlb, &vid, Tl, &ml) == 0;
        const double kp = P.k0[s] * pue;
        const double *qs = prof(&P, q, s);
        for (int64_t i = seg_offsets[s]; i < seg_offsets[s + 1]; ++i) {
            const uint64_t g = g0 ? g0[s] + (uint64_t)(i - seg_offsets[s]) : (uint64_t)i;   /* global index */
            int pinned = 0, cls = 0;
            if (flags) { pinned = flags[i] & 1; cls = (flags[i] >> 1) & 3; }
            pref[i] = (uint8_t)orc_pref_level(n, qs, seed, g);
            if (!ok || cls >= n_classes) {
                level[i] = 0xFF; carbon[i] = NAN; base[i] = NAN; ratio[i] = NAN;
                continue;
            }
            const int L = orc_select_level(n, xs, orc_draw_word(seed, g), pinned);
            const double tl = (double)tokens[(size_t)L * pitch + i], t0 = (double)tokens[i];
            const double el = ef[cls * 8 + L] + et[cls * 8 + L] * tl, pl = pf[cls * 8 + L] + pt[cls * 8 + L] * tl;
            const double e0 = ef[cls * 8] + et[cls * 8] * t0, p0 = pf[cls * 8] + pt[cls * 8] * t0;
            level[i] = (uint8_t)L;
            carbon[i] = orc_request_carbon(kp, k1, el, pl);
            base[i] = orc_request_carbon(kp, k1, e0, p0);
            ratio[i] = carbon[i] / base[i];
        }
    }
    return 0;
}

/* Reading L23 -- the Oracle scheme (it "assumes the inference carbon
 * emission on every generation directive level is known ahead of time for
 * all user prompts, and knows the exact generation quality feedback for
 * future prompts").  Per cell (segment, xi): with every request's carbon at
 * every level (Eq. 1) and its latent best level l*, choose each request's
 * level to minimise the cell's carbon subject to the realised quality
 * #{g : L(g) = l*(g)} >= k = ceil(fl(b * m)), b the cell's Eq. 3 floor
 * and m its valid requests; opted-out requests stay at L0
 * (P:240).  Any level other than a request's cheapest level m(g) (lowest
 * index among equal carbon) or its l* is dominated, so the optimum serves
 * every request at m(g) and moves the (k - free hits) requests with
 * l* != m(g) of smallest extra carbon Delta = C_l* - C_m(g) (equal Delta:
 * lower request index first) to l*: a unit-gain selection, exact by the
 * exchange argument.  Too few candidates: all move, status 2.  Invalid cell
 * inputs: status 1, totals 0.  Outputs per cell: cnt/tok [NC][n], fp64 sums
 * of E, T, carbon and q[level] over the requests in index order, stats
 * (hits, wins, losses as orc_preference) and status.                        */
typedef struct { double d; int64_t g; } orc_cand;
static int cand_cmp(const void *a, const void *b)
{
    const orc_cand *x = (const orc_cand *)a, *y = (const orc_cand *)b;
    if (x->d < y->d) return -1;
    if (x->d > y->d) return 1;
    return (x->g > y->g) - (x->g < y->g);
}

int orc_oracle_scheme(int n, int R, int64_t T, int X,
                      const double *k0, const double *kmin, const double *kmax, const double *xi,
                      const double *q, int profile_per_interval, double k1, double pue,
                      uint64_t seed, int n_classes, const double *ef, const double *et,
                      const double *pf, const double *pt,
                      const int64_t *seg_offsets, const uint64_t *gbase, const uint16_t *tokens, int64_t pitch,
                      const uint8_t *flags, uint64_t *cnt, uint64_t *tok, double *energy, double *time_s, double *carbon,
                      double *quality, uint64_t *stats, uint8_t *status)
{
    if (n < 1 || n > ORC_MAX_LEVELS || R < 1 || T < 1 || X < 1) return 1;
    if (n_classes < 1 || n_classes > ORC_MAX_CLASSES) return 1;
    const int NC = n_classes;
    for (int64_t s = 0; s < (int64_t)R * T; ++s) {
        const int64_t r = s / T, g0 = seg_offsets[s], m_all = seg_offsets[s + 1] - g0;
        const double *qs = q + (profile_per_interval ? s : r) * n;
        const double kp = k0[s] * pue;
        /* per request: class, pinned, cheapest level, l*, the base choice */
        int *cls = (int *)malloc(sizeof(int) * (size_t)(m_all > 0 ? m_all : 1));
        int *lm = (int *)malloc(sizeof(int) * (size_t)(m_all > 0 ? m_all : 1));
        int *ls = (int *)malloc(sizeof(int) * (size_t)(m_all > 0 ? m_all : 1));
        int *ch = (int *)malloc(sizeof(int) * (size_t)(m_all > 0 ? m_all : 1));
        orc_cand *cand = (orc_cand *)malloc(sizeof(orc_cand) * (size_t)(m_all > 0 ? m_all : 1));
        int64_t m = 0, free_hits = 0, nc = 0;
        for (int64_t i = 0; i < m_all; ++i) {
            const int64_t g = g0 + i;                                            /* local index */
            const uint64_t gg = gbase ? gbase[s] + (uint64_t)i : (uint64_t)g;   /* global index */
            int pinned = 0, c = 0;
            if (flags) { pinned = flags[g] & 1; c = (flags[g] >> 1) & 3; }
            cls[i] = c;
            if (c >= NC) continue;
            ++m;
            double C[ORC_MAX_LEVELS];
            for (int L = 0; L < n; ++L) {
                const double t = (double)tokens[(size_t)L * pitch + g];
                C[L] = orc_request_carbon(kp, k1, ef[c * 8 + L] + et[c * 8 + L] * t, pf[c * 8 + L] + pt[c * 8 + L] * t);
            }
            int best = 0;
            for (int L = 1; L < n; ++L) if (C[L] < C[best]) best = L;
            lm[i] = best;
            ls[i] = orc_pref_level(n, qs, seed, gg);
            ch[i] = pinned ? 0 : best;
            free_hits += (ch[i] == ls[i]);
            if (!pinned && ls[i] != best) {
                cand[nc].d = C[ls[i]] - C[best];
                cand[nc].g = i;
                ++nc;
            }
        }
        qsort(cand, (size_t)nc, sizeof(orc_cand), cand_cmp);
        uint8_t *moved = (uint8_t *)malloc((size_t)(m_all > 0 ? m_all : 1));
        for (int j = 0; j < X; ++j) {
            const int64_t cell = s * X + j;
            uint64_t *cn = cnt + (size_t)cell * NC * n, *tk = tok + (size_t)cell * NC * n;
            uint64_t *st = stats + (size_t)cell * 3;
            memset(cn, 0, sizeof(uint64_t) * NC * n);
            memset(tk, 0, sizeof(uint64_t) * NC * n);
            st[0] = st[1] = st[2] = 0;
            energy[cell] = 0.0; time_s[cell] = 0.0; carbon[cell] = 0.0; quality[cell] = 0.0;
            double dummy_e[ORC_MAX_LEVELS], dummy_p[ORC_MAX_LEVELS];
            for (int L = 0; L < n; ++L) { dummy_e[L] = 0.0; dummy_p[L] = 0.0; }
            if (!cell_inputs_valid(n, k0[s], kmin[r], kmax[r], xi[j], dummy_e, dummy_p, qs)) {
                status[cell] = 1;
                continue;
            }
            const double b = orc_quality_lower_bound(k0[s], kmin[r], kmax[r], xi[j], qs[0]);
            const double bm = ceil(b * (double)m);
            int64_t need = (int64_t)bm - free_hits;
            if (need < 0) need = 0;
            status[cell] = need > nc ? 2 : 0;
            if (need > nc) need = nc;
            memset(moved, 0, (size_t)(m_all > 0 ? m_all : 1));
            for (int64_t k = 0; k < need; ++k) moved[cand[k].g] = 1;
            double E = 0.0, Tm = 0.0, Cb = 0.0, Q = 0.0;
            for (int64_t i = 0; i < m_all; ++i) {
                const int c = cls[i];
                if (c >= NC) continue;
                const int64_t g = g0 + i;
                const int L = moved[i] ? ls[i] : ch[i];
                const uint32_t t = tokens[(size_t)L * pitch + g];
                const double el = ef[c * 8 + L] + et[c * 8 + L] * (double)t;
                const double pl = pf[c * 8 + L] + pt[c * 8 + L] * (double)t;
                E += el; Tm += pl; Cb += orc_request_carbon(kp, k1, el, pl); Q += qs[L];
                cn[c * n + L] += 1; tk[c * n + L] += t;
                int win, loss;
                orc_head_to_head(L, ls[i], &win, &loss);
                st[0] += (uint64_t)(L == ls[i]); st[1] += (uint64_t)win; st[2] += (uint64_t)loss;
            }
            energy[cell] = E; time_s[cell] = Tm; carbon[cell] = Cb; quality[cell] = Q;
        }
        free(moved); free(cls); free(lm); free(ls); free(ch); free(cand);
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* NEXT-1's q update per evaluation epoch (reading L24).  An
 * evaluation offers "a timely update to the q^T vector": the
 * evaluator samples 500 requests, generates every level's response
 * and records the best level of each; q is their preference rates
 * (P:190).  For region r and ONE evaluator configuration (beta, theta, grace,
 * fallback), the evaluations fire at the intervals of the trigger scan of
 * orc_evaluator_sweep (Eq. 8, reading L19; the trace start counts as one).
 * An evaluation at interval t samples the last `sample` requests of the
 * region before interval t starts (all of them if fewer; none: q unchanged)
 * and sets q_i = #{l* = i} / #sampled (the latent best level of reading L21,
 * drawn against the region's true q row q_true); that q holds from interval t
 * until the next evaluation.  Before any evaluation with samples, q is
 * q_true.  Outputs: q_out [R*T][n], fired [R*T] (1 where an evaluation
 * fired, t = 0 included).  seg_offsets [R*T+1] global request indices.     */
int orc_evaluation_q(int R, int64_t T, double dt, const double *k2, const double *k2max, double beta,
                     double theta, double grace, int F, int n, const double *q_true, uint64_t seed,
                     const int64_t *seg_offsets, int sample, double *q_out, uint8_t *fired)
{
    if (R < 1 || T < 1 || F < 0 || !(dt > 0.0) || n < 1 || n > ORC_MAX_LEVELS || sample < 1) return 1;
    for (int r = 0; r < R; ++r) {
        const double *k = k2 + (int64_t)r * T;
        const double *qt = q_true + (size_t)r * n;
        const double d = exp(-(beta * dt));
        const double thr = theta * k2max[r];
        double qc[ORC_MAX_LEVELS];
        for (int i = 0; i < n; ++i) qc[i] = qt[i];
        /* the trigger scan (orc_evaluator_sweep's state and rules) */
        int64_t t0 = 0, below = 0;
        double f = 1.0, prev1 = k[0], prev2 = 0.0;
        for (int64_t t = 0; t < T; ++t) {
            int fire = t == 0;
            if (t > 0) {
                f = f * d;
                double kp = f * k[t];
                int under = kp < thr;
                if (under) below = below + 1; else below = 0;
                int64_t since = t - t0;
                int grace_ok = (double)since * dt >= grace;
                int local_min = since >= 2 && prev1 < prev2 && kp > prev1;
                int fallback = F > 0 && below >= F;
                prev2 = prev1;
                prev1 = kp;
                if (grace_ok && under && (local_min || fallback)) {
                    fire = 1;
                    t0 = t;
                    f = 1.0;
                    prev1 = k[t];
                    below = 0;
                }
            }
            const int64_t s = (int64_t)r * T + t;
            fired[s] = (uint8_t)fire;
            if (fire) {
                const int64_t region0 = seg_offsets[(int64_t)r * T], end = seg_offsets[s];
                const int64_t begin = end - sample > region0 ? end - sample : region0;
                if (end > begin) {
                    int64_t cnt[ORC_MAX_LEVELS] = { 0 };
                    for (int64_t g = begin; g < end; ++g) cnt[orc_pref_level(n, qt, seed, (uint64_t)g)] += 1;
                    for (int i = 0; i < n; ++i) qc[i] = (double)cnt[i] / (double)(end - begin);
                }
            }
            for (int i = 0; i < n; ++i) q_out[(size_t)s * n + i] = qc[i];
        }
    }
    return 0;
}
