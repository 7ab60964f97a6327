/* oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Built with: gcc -O2 -ffp-contract=off -fno-fast-math -fPIC -shared -lm
 * so that every expression is evaluated exactly as written (no FMA
 * contraction, no reassociation).  fma() is used only where DESIGN.md §3
 * writes "fma".
 *
 * Section map (DESIGN.md §3 = the written definitions):
 *   §3.1 correctly rounded sums ........ or_fsum / or_dot / or_sumabs
 *   §3.2 7-point operator ................ or_spmv
 *   §3.3 momentum row .................... or_assemble_mom     (Eq. 2)
 *   §3.4 pressure-correction row ......... or_assemble_pp      (Eq. 1)
 *   §3.5 scalar row ...................... or_assemble_scalar
 *   §3.6 BiCGSTAB ........................ or_bicgstab
 *   §3.7 correction ...................... or_correct
 *   §3.8 SIMPLE outer iteration .......... or_simple_iter
 */
#include "oracle.h"

#include <math.h>
#include <omp.h>
#include <quadmath.h>
#include <stdlib.h>
#include <string.h>

/* Threading (bench.py cpu_baseline, SURVEY §8(d) "OpenMP over all cores").
 * Row loops are split over threads with no change to any row's expression;
 * a correctly rounded sum is split into per-thread exact partial expansions
 * that are merged exactly before the single rounding, so every result is
 * bit-identical to the serial evaluation for any thread count ("parity
 * mode", tested).  or_set_mode(threads, naive = 1) replaces the exact sums by
 * plain per-thread sequential sums for the "plain CPU" timing only (not
 * correctly rounded; never used by a parity test). */
#define OR_PAR_MIN 32768
static int g_naive = 0;

void or_set_mode(int threads, int naive)
{
    if (threads > 0) omp_set_num_threads(threads);
    g_naive = naive != 0;
}

int or_max_threads(void) { return omp_get_max_threads(); }

/* ------------------------------------------------------------------ §3.1 */
/* Exact summation with Shewchuk's non-overlapping partials (the algorithm of
 * Python's math.fsum): the returned value is the exact sum rounded once to
 * nearest-even.  Inputs must be finite and the partial sums must not
 * overflow (always true for the fields of this problem). */
typedef struct { double p[256]; int n; } xsum;

static void xs_init(xsum *s) { s->n = 0; }

static void xs_add(xsum *s, double x)
{
    int i = 0;
    for (int j = 0; j < s->n; j++) {
        double y = s->p[j];
        if (fabs(x) < fabs(y)) { double t = x; x = y; y = t; }
        double hi = x + y;
        double lo = y - (hi - x);
        if (lo != 0.0) s->p[i++] = lo;
        x = hi;
    }
    s->n = i;
    s->p[s->n++] = x;
}

static double xs_round(const xsum *s)
{
    int n = s->n;
    double hi = 0.0, lo = 0.0;
    if (n > 0) {
        hi = s->p[--n];
        while (n > 0) {
            double x = hi, y = s->p[--n];
            hi = x + y;
            double yr = hi - x;
            lo = y - yr;
            if (lo != 0.0) break;
        }
        /* round-half-even correction when the remainder is exactly half an ulp */
        if (n > 0 && ((lo < 0.0 && s->p[n - 1] < 0.0) || (lo > 0.0 && s->p[n - 1] > 0.0))) {
            double y = lo * 2.0;
            double x = hi + y;
            double yr = x - hi;
            if (y == yr) hi = x;
        }
    }
    return hi + 0.0; /* an exact zero is +0 */
}

static void xs_merge(xsum *dst, const xsum *src)
{
    for (int j = 0; j < src->n; j++) xs_add(dst, src->p[j]);
}

/* one correctly rounded sum of the terms term(i, &hi, &lo) (lo may be 0):
 * per-thread exact expansions over contiguous index ranges, merged exactly */
#define OR_EXACT_SUM(n, BODY)                                                        \
    do {                                                                             \
        const int nt_ = (n) >= OR_PAR_MIN ? omp_get_max_threads() : 1;               \
        xsum *part_ = malloc(sizeof(xsum) * (size_t)nt_);                            \
        _Pragma("omp parallel num_threads(nt_)")                                     \
        {                                                                            \
            const int t_ = omp_get_thread_num(), T_ = omp_get_num_threads();         \
            const long lo_ = (long)((n) * (double)t_ / T_), hi_ = (long)((n) * (double)(t_ + 1) / T_); \
            xsum *s = &part_[t_];                                                    \
            xs_init(s);                                                              \
            for (long i = lo_; i < hi_; i++) { BODY }                                \
        }                                                                            \
        xsum tot_; xs_init(&tot_);                                                   \
        for (int t_ = 0; t_ < nt_; t_++) xs_merge(&tot_, &part_[t_]);                \
        free(part_);                                                                 \
        result_ = xs_round(&tot_);                                                   \
    } while (0)

/* plain (naive) sum for the timing mode: sequential within a thread range,
 * thread results added in thread order */
#define OR_PLAIN_SUM(n, TERM)                                                        \
    do {                                                                             \
        const int nt_ = (n) >= OR_PAR_MIN ? omp_get_max_threads() : 1;               \
        double part_[256];                                                           \
        _Pragma("omp parallel num_threads(nt_ < 256 ? nt_ : 256)")                   \
        {                                                                            \
            const int t_ = omp_get_thread_num(), T_ = omp_get_num_threads();         \
            const long lo_ = (long)((n) * (double)t_ / T_), hi_ = (long)((n) * (double)(t_ + 1) / T_); \
            double a_ = 0.0;                                                         \
            for (long i = lo_; i < hi_; i++) a_ = a_ + (TERM);                       \
            part_[t_] = a_;                                                          \
        }                                                                            \
        double r_ = 0.0;                                                             \
        for (int t_ = 0; t_ < (nt_ < 256 ? nt_ : 256); t_++) r_ = r_ + part_[t_];    \
        result_ = r_ + 0.0;                                                          \
    } while (0)

double or_fsum(long n, const double *x)
{
    double result_;
    if (g_naive) { OR_PLAIN_SUM(n, x[i]); return result_; }
    OR_EXACT_SUM(n, xs_add(s, x[i]););
    return result_;
}

/* <a,b> = exact sum of the products a_i b_i, rounded once.  Each product is
 * split exactly as hi + lo with hi = fl(a b), lo = fma(a, b, -hi). */
double or_dot(long n, const double *a, const double *b)
{
    double result_;
    if (g_naive) { OR_PLAIN_SUM(n, a[i] * b[i]); return result_; }
    OR_EXACT_SUM(n, {
        double hi = a[i] * b[i];
        double lo = fma(a[i], b[i], -hi);
        xs_add(s, hi);
        xs_add(s, lo);
    });
    return result_;
}

double or_sumabs(long n, const double *x)
{
    double result_;
    if (g_naive) { OR_PLAIN_SUM(n, fabs(x[i])); return result_; }
    OR_EXACT_SUM(n, xs_add(s, fabs(x[i])););
    return result_;
}

/* ------------------------------------------------------------ helpers */
static long idx(const og_grid *g, int i, int j, int k)
{
    return (long)i + (long)g->nx * ((long)j + (long)g->ny * (long)k);
}
static int ext(const og_grid *g, int a) { return a == 0 ? g->nx : (a == 1 ? g->ny : g->nz); }
static double spacing(const og_grid *g, int a) { return a == 0 ? g->dx : (a == 1 ? g->dy : g->dz); }
static double area(const og_grid *g, int a)
{
    return a == 0 ? g->dy * g->dz : (a == 1 ? g->dx * g->dz : g->dx * g->dy);
}
static double volume(const og_grid *g) { return (g->dx * g->dy) * g->dz; }
static int inside(const og_grid *g, const int q[3])
{
    return q[0] >= 0 && q[0] < g->nx && q[1] >= 0 && q[1] < g->ny && q[2] >= 0 && q[2] < g->nz;
}
static long at(const og_grid *g, const int q[3]) { return idx(g, q[0], q[1], q[2]); }
static double maxp(double f) { return f > 0.0 ? f : 0.0; }
static long ncell(const og_grid *g) { return (long)g->nx * g->ny * g->nz; }
/* §3.10: Q is a BLOCKED cell (inside the domain and flagged) */
static int blk(const og_grid *g, const og_state *st, const int Q[3])
{
    return st->blocked && inside(g, Q) && st->blocked[at(g, Q)] != 0;
}
/* the face between X and X + e_a touches a BLOCKED cell: an internal wall */
static int wall_face(const og_grid *g, const og_state *st, int a, const int X[3])
{
    int Y[3] = {X[0], X[1], X[2]};
    Y[a] += 1;
    return blk(g, st, X) || blk(g, st, Y);
}

static int grid_ok(const og_grid *g)
{
    if (g->nx < 2 || g->ny < 2 || g->nz < 2) return 0;
    if (!(g->dx > 0 && g->dy > 0 && g->dz > 0)) return 0;
    if (g->bc_zlo != OG_WALL && g->bc_zlo != OG_INLET) return 0;
    if (g->bc_zhi != OG_WALL && g->bc_zhi != OG_OUTLET && g->bc_zhi != OG_DIRICHLET_TEST) return 0;
    return 1;
}

/* ------------------------------------------------------------------ §3.2 */
/* y = A x, row by row: y = aP x_P, then y = fma(-a_nb, x_nb, y) for nb in
 * W, E, S, N, B, T.  Out-of-domain neighbours contribute a_nb = 0, x_nb = 0.
 * Symmetric (p') storage: a_W(n) = c_x[n - 1], a_E(n) = c_x[n], etc. */
void or_spmv(const og_grid *g, const og_eqsys *A, const double *x, double *y)
{
    const int sym = (A->aW == NULL);
    const long sx = 1, sy = g->nx, sz = (long)g->nx * g->ny;
#pragma omp parallel for collapse(2) schedule(static) if (ncell(g) >= OR_PAR_MIN)
    for (int k = 0; k < g->nz; k++)
        for (int j = 0; j < g->ny; j++)
            for (int i = 0; i < g->nx; i++) {
                long n = idx(g, i, j, k);
                double aW, aE, aS, aN, aB, aT;
                if (sym) {
                    aW = i > 0 ? A->aE[n - sx] : 0.0;
                    aE = A->aE[n];
                    aS = j > 0 ? A->aN[n - sy] : 0.0;
                    aN = A->aN[n];
                    aB = k > 0 ? A->aT[n - sz] : 0.0;
                    aT = A->aT[n];
                } else {
                    aW = A->aW[n]; aE = A->aE[n]; aS = A->aS[n];
                    aN = A->aN[n]; aB = A->aB[n]; aT = A->aT[n];
                }
                double xW = i > 0 ? x[n - sx] : 0.0;
                double xE = i < g->nx - 1 ? x[n + sx] : 0.0;
                double xS = j > 0 ? x[n - sy] : 0.0;
                double xN = j < g->ny - 1 ? x[n + sy] : 0.0;
                double xB = k > 0 ? x[n - sz] : 0.0;
                double xT = k < g->nz - 1 ? x[n + sz] : 0.0;
                double r = A->aP[n] * x[n];
                r = fma(-aW, xW, r);
                r = fma(-aE, xE, r);
                r = fma(-aS, xS, r);
                r = fma(-aN, xN, r);
                r = fma(-aB, xB, r);
                r = fma(-aT, xT, r);
                y[n] = r;
            }
}

/* ------------------------------------------------------------------ §3.3 */
/* Momentum row for staggered component c (0=u,1=v,2=w) at cell P: the face
 * between P and E = P + e_c.  Convection first-order upwind in
 * non-conservative form, diffusion mu*eps (Q12), implicit
 * drag beta V plus explicit S V (Q11), pressure -eps grad p (Eq. 2 gauge),
 * gravity eps rho g, implicit under-relaxation.
 * Boundary rules B1 (known value at distance h), B2 (known value at h/2,
 * mirror ghost), B3 (zero gradient, dropped) as in DESIGN.md §3.3. */

enum { ROW_INTERIOR = 0, ROW_IDENTITY = 1, ROW_OUTLET = 2 };

static int mom_row_type(const og_grid *g, const og_state *st, int c, const int P[3])
{
    if (blk(g, st, P)) return ROW_IDENTITY;                     /* §3.10 */
    if (P[c] < ext(g, c) - 1) return wall_face(g, st, c, P) ? ROW_IDENTITY : ROW_INTERIOR;
    if (c == 2 && g->bc_zhi == OG_OUTLET) return ROW_OUTLET;
    return ROW_IDENTITY;
}

static const double *comp_field(const og_state *st, int a)
{
    return a == 0 ? st->u : (a == 1 ? st->v : st->w);
}

/* velocity of component c on the face Q + e_c/2 (Q may be one step outside) */
static double vel_c(const og_grid *g, const og_state *st, int c, const int Q[3])
{
    if (Q[c] == -1) return (c == 2 && g->bc_zlo == OG_INLET) ? g->w_in : 0.0;
    if (mom_row_type(g, st, c, Q) == ROW_IDENTITY) return 0.0;   /* domain or internal wall face */
    return comp_field(st, c)[at(g, Q)];
}

/* mass flux through the +t face of cell X, the face being interior */
/* §3.12: eps on the +a face of X for a convective mass flux: the central
 * average (reading Q9), or with face_eps_upwind the upwind cell's value by
 * the sign of the snapshot velocity on that face (>= 0: X). */
static double conv_face_eps(const og_grid *g, const og_params *pr, const og_state *st, int a, const int X[3])
{
    int Y[3] = {X[0], X[1], X[2]};
    Y[a] += 1;
    if (pr->face_eps_upwind)
        return comp_field(st, a)[at(g, X)] >= 0.0 ? st->eps[at(g, X)] : st->eps[at(g, Y)];
    return 0.5 * (st->eps[at(g, X)] + st->eps[at(g, Y)]);
}

static double mflux_t(const og_grid *g, const og_params *pr, const og_state *st, int t, const int X[3])
{
    double ef = conv_face_eps(g, pr, st, t, X);
    return ((pr->rho * ef) * area(g, t)) * comp_field(st, t)[at(g, X)];
}

int or_assemble_mom(const og_grid *g, const og_params *pr, int c, const og_state *st,
                    og_eqsys *out, double resid2[2])
{
    if (!grid_ok(g) || c < 0 || c > 2) return OG_ERR_ARG;
    if (g->bc_zhi == OG_DIRICHLET_TEST) return OG_ERR_ARG;
    const double V = volume(g);
    const double rVdt = (pr->rho * V) / pr->dt;
    const double *um = comp_field(st, c);
    const double *uold = c == 0 ? st->u_old : (c == 1 ? st->v_old : st->w_old);
    const double *S = c == 0 ? st->sbeta_u : (c == 1 ? st->sbeta_v : st->sbeta_w);
    double Dc[3];
    for (int a = 0; a < 3; a++) Dc[a] = (pr->mu * area(g, a)) / spacing(g, a);
    const long N = ncell(g);
    double *rnum = malloc(sizeof(double) * N), *rden = malloc(sizeof(double) * N);
    int any_nf = 0, any_zd = 0;

#pragma omp parallel for collapse(2) schedule(static) reduction(|: any_nf, any_zd) if (ncell(g) >= OR_PAR_MIN)
    for (int k = 0; k < g->nz; k++)
        for (int j = 0; j < g->ny; j++)
            for (int i = 0; i < g->nx; i++) {
                const int P[3] = {i, j, k};
                const long n = at(g, P);
                const int type = mom_row_type(g, st, c, P);
                if (type == ROW_IDENTITY) {
                    out->aP[n] = 1.0;
                    out->aW[n] = out->aE[n] = out->aS[n] = out->aN[n] = out->aB[n] = out->aT[n] = 0.0;
                    out->b[n] = 0.0;
                    out->d[n] = 0.0;
                    rnum[n] = 0.0;   /* identity rows are excluded from the residual: exact zeros */
                    rden[n] = 0.0;
                    continue;
                }
                /* E: the other cell of the face, clamped onto P at the outlet row */
                int E[3] = {i, j, k};
                if (type == ROW_INTERIOR) E[c] += 1;
                const long nE = at(g, E);

                /* six sides in geometric order x-,x+,y-,y+,z-,z+ */
                double a_side[6], phi_b[6];
                int kept[6], inP[6];
                for (int s6 = 0; s6 < 6; s6++) { a_side[s6] = 0.0; phi_b[s6] = 0.0; kept[s6] = 0; inP[s6] = 0; }

                for (int t = 0; t < 3; t++) {
                    if (t == c) {
                        /* main axis, minus side: face at the centre of P */
                        int Qm[3] = {i, j, k}; Qm[c] -= 1;
                        double Fm = ((pr->rho * st->eps[n]) * area(g, c)) *
                                    (0.5 * (vel_c(g, st, c, Qm) + vel_c(g, st, c, P)));
                        double Dm = Dc[c] * st->eps[n];
                        a_side[2 * c] = Dm + maxp(Fm);
                        inP[2 * c] = 1;
                        if (P[c] >= 1 && !blk(g, st, Qm)) kept[2 * c] = 1;
                        else phi_b[2 * c] = vel_c(g, st, c, Qm); /* B1 (domain or internal wall face: 0) */
                        /* plus side: face at the centre of E */
                        if (type == ROW_OUTLET) {
                            a_side[2 * c + 1] = 0.0; /* B3 */
                        } else {
                            double Fp = ((pr->rho * st->eps[nE]) * area(g, c)) *
                                        (0.5 * (vel_c(g, st, c, P) + vel_c(g, st, c, E)));
                            double Dp = Dc[c] * st->eps[nE];
                            a_side[2 * c + 1] = Dp + maxp(-Fp);
                            inP[2 * c + 1] = 1;
                            if (mom_row_type(g, st, c, E) == ROW_IDENTITY) phi_b[2 * c + 1] = 0.0; /* B1 */
                            else kept[2 * c + 1] = 1;
                        }
                        continue;
                    }
                    for (int s = -1; s <= 1; s += 2) {
                        const int side = 2 * t + (s > 0);
                        int Pt[3] = {i, j, k}; Pt[t] += s;
                        int Et[3] = {E[0], E[1], E[2]}; Et[t] += s;
                        if (inside(g, Pt) && !blk(g, st, Pt) && !blk(g, st, Et)) {
                            const int *Q = s > 0 ? P : Pt;
                            const int *R = s > 0 ? E : Et;
                            double F = 0.5 * (mflux_t(g, pr, st, t, Q) + mflux_t(g, pr, st, t, R));
                            double e4 = 0.25 * (((st->eps[n] + st->eps[nE]) + st->eps[at(g, Pt)]) +
                                                st->eps[at(g, Et)]);
                            double D = Dc[t] * e4;
                            a_side[side] = D + maxp(s > 0 ? -F : F);
                            inP[side] = 1;
                            kept[side] = 1;
                        } else {
                            int bc = OG_WALL;                    /* domain wall or internal wall (§3.10) */
                            if (t == 2 && !inside(g, Pt)) bc = s < 0 ? g->bc_zlo : g->bc_zhi;
                            if (bc == OG_OUTLET) { a_side[side] = 0.0; continue; } /* B3 */
                            double F = 0.0;
                            if (bc == OG_INLET)
                                F = 0.5 * (((pr->rho * st->eps[n]) * area(g, 2)) * g->w_in +
                                           ((pr->rho * st->eps[nE]) * area(g, 2)) * g->w_in);
                            double e2 = 0.5 * (st->eps[n] + st->eps[nE]);
                            double D = Dc[t] * e2;
                            a_side[side] = 2.0 * D + maxp(s > 0 ? -F : F); /* B2, phi_b = 0 */
                            inP[side] = 1;
                            phi_b[side] = 0.0;
                        }
                    }
                }

                double sum = ((((a_side[0] + a_side[1]) + a_side[2]) + a_side[3]) + a_side[4]) + a_side[5];
                double bcb = 0.0;
                for (int s6 = 0; s6 < 6; s6++)
                    if (inP[s6] && !kept[s6]) bcb = bcb + a_side[s6] * phi_b[s6];
                const double ef = 0.5 * (st->eps[n] + st->eps[nE]);
                const double e0f = 0.5 * (st->eps_old[n] + st->eps_old[nE]);
                const double bf = 0.5 * (st->beta[n] + st->beta[nE]);
                const double Sf = 0.5 * (S[n] + S[nE]);
                const double pE = type == ROW_OUTLET ? 0.0 : st->p[nE];
                const double a0 = rVdt * e0f;
                const double aP = (sum + a0) + bf * V;
                const double b = ((((a0 * uold[n]) + (ef * area(g, c)) * (st->p[n] - pE)) +
                                   ((pr->rho * ef) * pr->g[c]) * V) + Sf * V) + bcb;
                const double aPr = aP / pr->urf_mom;
                const double bR = b + (aPr - aP) * um[n];
                const double d = (ef * area(g, c)) / aPr;

                double st6[6];
                for (int s6 = 0; s6 < 6; s6++) st6[s6] = kept[s6] ? a_side[s6] : 0.0;
                out->aW[n] = st6[0]; out->aE[n] = st6[1];
                out->aS[n] = st6[2]; out->aN[n] = st6[3];
                out->aB[n] = st6[4]; out->aT[n] = st6[5];
                out->aP[n] = aPr;
                out->b[n] = bR;
                out->d[n] = d;
                if (!isfinite(aPr) || !isfinite(bR) || !isfinite(d)) any_nf = 1;
                else if (aPr == 0.0) any_zd = 1;

                /* snapshot residual, un-relaxed row */
                double res = b - aP * um[n];
                for (int s6 = 0; s6 < 6; s6++) {
                    int Q[3] = {i, j, k};
                    Q[s6 / 2] += (s6 & 1) ? 1 : -1;
                    double unb = inside(g, Q) ? um[at(g, Q)] : 0.0;
                    res = res + st6[s6] * unb;
                }
                rnum[n] = fabs(res);
                rden[n] = fabs(aP * um[n]);
            }
    const int status = any_nf ? OG_ERR_NONFINITE : (any_zd ? OG_ERR_ZERO_DIAG : OG_OK);
    if (resid2) {
        resid2[0] = or_sumabs(N, rnum);
        resid2[1] = or_sumabs(N, rden);
    }
    free(rnum); free(rden);
    return status;
}

/* ------------------------------------------------------------------ §3.4 */
/* p' row (SIMPLE): face coefficient c_f = rho eps_f A_f d_f,
 * one stored value per face (A symmetric), a_P = sum of the six faces; the
 * outlet face stays in a_P with ghost p' = 0 (Q13).  b = mass imbalance of
 * the starred field minus the transient term (Eq. 1 discretised). */


/* coefficient-like quantity rho eps_f A_f q on the +a face of X */
static double plus_face(const og_grid *g, const og_params *pr, const og_state *st, int a,
                        const int X[3], const double *q)
{
    if (X[a] <= ext(g, a) - 2) {
        if (wall_face(g, st, a, X)) return 0.0;                   /* internal wall (§3.10) */
        return ((pr->rho * conv_face_eps(g, pr, st, a, X)) * area(g, a)) * q[at(g, X)];
    }
    if (a == 2 && g->bc_zhi == OG_OUTLET && !blk(g, st, X))
        return ((pr->rho * st->eps[at(g, X)]) * area(g, 2)) * q[at(g, X)];
    return 0.0;
}

int or_assemble_pp(const og_grid *g, const og_params *pr, const og_state *st,
                   const double *us, const double *vs, const double *ws,
                   const double *dxv, const double *dyv, const double *dzv,
                   og_eqsys *out, double *cont)
{
    if (!grid_ok(g) || g->bc_zhi == OG_DIRICHLET_TEST) return OG_ERR_ARG;
    const double V = volume(g);
    const double rVdt = (pr->rho * V) / pr->dt;
    const double *vel[3] = {us, vs, ws};
    const double *dd[3] = {dxv, dyv, dzv};
    double *cf[3] = {out->aE, out->aN, out->aT};
    int any_nf = 0, any_zd = 0;
#pragma omp parallel for collapse(2) schedule(static) reduction(|: any_nf, any_zd) if (ncell(g) >= OR_PAR_MIN)
    for (int k = 0; k < g->nz; k++)
        for (int j = 0; j < g->ny; j++)
            for (int i = 0; i < g->nx; i++) {
                const int P[3] = {i, j, k};
                const long n = at(g, P);
                double cm[3], cpl[3], mm[3], mp[3];
                for (int a = 0; a < 3; a++) {
                    cpl[a] = plus_face(g, pr, st, a, P, dd[a]);
                    mp[a] = plus_face(g, pr, st, a, P, vel[a]);
                    if (P[a] >= 1) {
                        int Q[3] = {i, j, k}; Q[a] -= 1;
                        cm[a] = plus_face(g, pr, st, a, Q, dd[a]);
                        mm[a] = plus_face(g, pr, st, a, Q, vel[a]);
                    } else {
                        cm[a] = 0.0;
                        mm[a] = (a == 2 && g->bc_zlo == OG_INLET && !blk(g, st, P))
                                    ? ((pr->rho * st->eps[n]) * area(g, 2)) * g->w_in : 0.0;
                    }
                }
                double aP = ((((cm[0] + cpl[0]) + cm[1]) + cpl[1]) + cm[2]) + cpl[2];
                double b = (((mm[0] - mp[0]) + (mm[1] - mp[1])) + (mm[2] - mp[2])) -
                           rVdt * (st->eps[n] - st->eps_old[n]);
                if (blk(g, st, P)) b = 0.0;                               /* empty row: p' stays 0 */
                out->aP[n] = aP;
                for (int a = 0; a < 3; a++) cf[a][n] = cpl[a];
                out->b[n] = b;
                if (!isfinite(aP) || !isfinite(b)) any_nf = 1;
                else if (aP == 0.0 && !blk(g, st, P)) any_zd = 1;
            }
    const int status = any_nf ? OG_ERR_NONFINITE : (any_zd ? OG_ERR_ZERO_DIAG : OG_OK);
    if (cont) *cont = or_sumabs(ncell(g), out->b);
    return status;
}

/* ------------------------------------------------------------------ §3.5 */
/* Cell-centred scalar (energy / species): FOUP convection-
 * diffusion with transient; Dirichlet inlet (B2), zero-gradient outlet (B3),
 * zero-flux walls; test-only Dirichlet top (B2 with phi_out). */
int or_assemble_scalar(const og_grid *g, const og_params *pr, int sid, const og_state *st,
                       og_eqsys *out, double resid2[2])
{
    if (!grid_ok(g) || sid < 0 || sid > 3) return OG_ERR_ARG;
    const double V = volume(g);
    const double rVdt = (pr->rho * V) / pr->dt;
    const double gam = pr->gamma_phi[sid];
    const double *phim = st->phi[sid], *phi0 = st->phi_old[sid];
    const double *vel[3] = {st->u, st->v, st->w};
    double Dc[3];
    for (int a = 0; a < 3; a++) Dc[a] = (gam * area(g, a)) / spacing(g, a);
    const long N = ncell(g);
    double *rnum = malloc(sizeof(double) * N), *rden = malloc(sizeof(double) * N);
    int any_nf = 0, any_zd = 0;
#pragma omp parallel for collapse(2) schedule(static) reduction(|: any_nf, any_zd) if (ncell(g) >= OR_PAR_MIN)
    for (int k = 0; k < g->nz; k++)
        for (int j = 0; j < g->ny; j++)
            for (int i = 0; i < g->nx; i++) {
                const int P[3] = {i, j, k};
                const long n = at(g, P);
                double a_side[6], phib[6];
                int kept[6], inP[6];
                for (int a = 0; a < 3; a++) {
                    /* minus side */
                    int sm = 2 * a, sp = 2 * a + 1;
                    a_side[sm] = a_side[sp] = 0.0; phib[sm] = phib[sp] = 0.0;
                    kept[sm] = kept[sp] = 0; inP[sm] = inP[sp] = 0;
                    int Qm_[3] = {i, j, k}; Qm_[a] -= 1;
                    int Qp_[3] = {i, j, k}; Qp_[a] += 1;
                    if (P[a] >= 1 && blk(g, st, Qm_)) {
                        /* internal zero-flux wall (§3.10): a = 0 */
                    } else if (P[a] >= 1) {
                        int Q[3] = {i, j, k}; Q[a] -= 1;
                        double e = 0.5 * (st->eps[at(g, Q)] + st->eps[n]);
                        double F = ((pr->rho * conv_face_eps(g, pr, st, a, Q)) * area(g, a)) * vel[a][at(g, Q)];
                        a_side[sm] = Dc[a] * e + maxp(F);
                        kept[sm] = inP[sm] = 1;
                    } else if (a == 2 && g->bc_zlo == OG_INLET) {
                        double F = ((pr->rho * st->eps[n]) * area(g, 2)) * g->w_in;
                        a_side[sm] = 2.0 * (Dc[2] * st->eps[n]) + maxp(F);
                        inP[sm] = 1;
                        phib[sm] = g->phi_in;
                    }
                    /* plus side */
                    if (P[a] <= ext(g, a) - 2 && blk(g, st, Qp_)) {
                        /* internal zero-flux wall (§3.10) */
                    } else if (P[a] <= ext(g, a) - 2) {
                        double e = 0.5 * (st->eps[n] + st->eps[at(g, (int[3]){i + (a == 0), j + (a == 1), k + (a == 2)})]);
                        double F = ((pr->rho * conv_face_eps(g, pr, st, a, P)) * area(g, a)) * vel[a][n];
                        a_side[sp] = Dc[a] * e + maxp(-F);
                        kept[sp] = inP[sp] = 1;
                    } else if (a == 2 && g->bc_zhi == OG_DIRICHLET_TEST) {
                        double F = ((pr->rho * st->eps[n]) * area(g, 2)) * vel[2][n];
                        a_side[sp] = 2.0 * (Dc[2] * st->eps[n]) + maxp(-F);
                        inP[sp] = 1;
                        phib[sp] = g->phi_out;
                    }
                }
                if (blk(g, st, P)) {
                    /* BLOCKED cell: identity row phi = 0 (no scalar inside an obstacle), no residual */
                    out->aP[n] = 1.0;
                    out->aW[n] = out->aE[n] = out->aS[n] = out->aN[n] = out->aB[n] = out->aT[n] = 0.0;
                    out->b[n] = 0.0;
                    if (out->d) out->d[n] = 0.0;
                    rnum[n] = 0.0;
                    rden[n] = 0.0;
                    continue;
                }
                double sum = ((((a_side[0] + a_side[1]) + a_side[2]) + a_side[3]) + a_side[4]) + a_side[5];
                double bcb = 0.0;
                for (int s6 = 0; s6 < 6; s6++)
                    if (inP[s6] && !kept[s6]) bcb = bcb + a_side[s6] * phib[s6];
                const double a0 = rVdt * st->eps_old[n];
                const double aP = sum + a0;
                const double b = (a0 * phi0[n]) + bcb;
                const double aPr = aP / pr->urf_phi;
                const double bR = b + (aPr - aP) * phim[n];
                double st6[6];
                for (int s6 = 0; s6 < 6; s6++) st6[s6] = kept[s6] ? a_side[s6] : 0.0;
                out->aW[n] = st6[0]; out->aE[n] = st6[1];
                out->aS[n] = st6[2]; out->aN[n] = st6[3];
                out->aB[n] = st6[4]; out->aT[n] = st6[5];
                out->aP[n] = aPr;
                out->b[n] = bR;
                if (out->d) out->d[n] = 0.0;
                if (!isfinite(aPr) || !isfinite(bR)) any_nf = 1;
                else if (aPr == 0.0) any_zd = 1;
                double res = b - aP * phim[n];
                for (int s6 = 0; s6 < 6; s6++) {
                    int Q[3] = {i, j, k};
                    Q[s6 / 2] += (s6 & 1) ? 1 : -1;
                    double unb = inside(g, Q) ? phim[at(g, Q)] : 0.0;
                    res = res + st6[s6] * unb;
                }
                rnum[n] = fabs(res);
                rden[n] = fabs(aP * phim[n]);
            }
    const int status = any_nf ? OG_ERR_NONFINITE : (any_zd ? OG_ERR_ZERO_DIAG : OG_OK);
    if (resid2) {
        resid2[0] = or_sumabs(N, rnum);
        resid2[1] = or_sumabs(N, rden);
    }
    free(rnum); free(rden);
    return status;
}

/* ------------------------------------------------------------------ §3.6 */
/* Unpreconditioned BiCGSTAB (van der Vorst), "No preconditioners";
 * SPEC.md:370-378; readings Q1-Q5, Q17. */
int or_bicgstab(const og_grid *g, const og_eqsys *A, double *x, double tol, int maxit,
                og_solve_info *info, double *trace)
{
    const long N = ncell(g);
    double *r = calloc(N, sizeof(double)), *rh = calloc(N, sizeof(double));
    double *p = calloc(N, sizeof(double)), *v = calloc(N, sizeof(double));
    double *s = calloc(N, sizeof(double)), *t = calloc(N, sizeof(double));
    double *y = calloc(N, sizeof(double));
    int status = OG_NOT_CONVERGED, iters = 0, restarts = 0;
    double rel = 0.0;

    or_spmv(g, A, x, y);
    #pragma omp parallel for schedule(static) if (N >= OR_PAR_MIN)
    for (long n = 0; n < N; n++) r[n] = A->b[n] - y[n];
    const double bn = sqrt(or_dot(N, A->b, A->b));
    double rr = or_dot(N, r, r);
    double rn = sqrt(rr);
    if (bn == 0.0) {
        #pragma omp parallel for schedule(static) if (N >= OR_PAR_MIN)
        for (long n = 0; n < N; n++) x[n] = 0.0;
        status = OG_OK; iters = 0; rel = 0.0;
        goto done;
    }
    if (rn <= tol * bn) { status = OG_OK; iters = 0; rel = rn / bn; goto done; }

    #pragma omp parallel for schedule(static) if (N >= OR_PAR_MIN)
    for (long n = 0; n < N; n++) rh[n] = r[n];
    double rhn = rn;
    double rho = or_dot(N, rh, r);
    double rho_prev = 1.0, alpha = 1.0, omega = 1.0;
    int restarted = 0;

    for (int it = 1; it <= maxit; it++) {
        double *tr = trace ? trace + 8 * (long)(it - 1) : NULL;
        if (fabs(rho) <= (1e-14 * rhn) * rn) {
            if (restarted) { status = OG_ERR_BREAKDOWN; iters = it - 1; goto done_rel; }
            #pragma omp parallel for schedule(static) if (N >= OR_PAR_MIN)
            for (long n = 0; n < N; n++) { rh[n] = r[n]; p[n] = 0.0; v[n] = 0.0; }
            rhn = rn; rho = or_dot(N, rh, r);
            rho_prev = alpha = omega = 1.0; restarted = 1; restarts++;
        }
        const double beta = (rho / rho_prev) * (alpha / omega);
        #pragma omp parallel for schedule(static) if (N >= OR_PAR_MIN)
        for (long n = 0; n < N; n++) p[n] = fma(beta, fma(-omega, v[n], p[n]), r[n]);
        or_spmv(g, A, p, v);
        const double sigma = or_dot(N, rh, v);
        if (tr) { tr[0] = rho; tr[1] = sigma; }
        if (sigma == 0.0) {
            if (restarted) { status = OG_ERR_BREAKDOWN; iters = it; goto done_rel; }
            #pragma omp parallel for schedule(static) if (N >= OR_PAR_MIN)
            for (long n = 0; n < N; n++) { rh[n] = r[n]; p[n] = 0.0; v[n] = 0.0; }
            rhn = rn; rho = or_dot(N, rh, r);
            rho_prev = alpha = omega = 1.0; restarted = 1; restarts++;
            continue;
        }
        alpha = rho / sigma;
        #pragma omp parallel for schedule(static) if (N >= OR_PAR_MIN)
        for (long n = 0; n < N; n++) s[n] = fma(-alpha, v[n], r[n]);
        const double ss = or_dot(N, s, s);
        if (tr) { tr[2] = alpha; tr[3] = ss; }
        if (sqrt(ss) <= tol * bn) {
            #pragma omp parallel for schedule(static) if (N >= OR_PAR_MIN)
            for (long n = 0; n < N; n++) { x[n] = fma(alpha, p[n], x[n]); r[n] = s[n]; }
            rn = sqrt(ss);
            status = OG_OK; iters = it; goto done_rel;
        }
        or_spmv(g, A, s, t);
        const double ts = or_dot(N, t, s);
        const double tt = or_dot(N, t, t);
        const double om = tt == 0.0 ? 0.0 : ts / tt;
        if (tr) { tr[4] = ts; tr[5] = tt; tr[6] = om; }
        if (tt == 0.0 || om == 0.0) {
            if (restarted) { status = OG_ERR_BREAKDOWN; iters = it; goto done_rel; }
            #pragma omp parallel for schedule(static) if (N >= OR_PAR_MIN)
            for (long n = 0; n < N; n++) { rh[n] = r[n]; p[n] = 0.0; v[n] = 0.0; }
            rhn = rn; rho = or_dot(N, rh, r);
            rho_prev = alpha = omega = 1.0; restarted = 1; restarts++;
            continue;
        }
        omega = om;
        #pragma omp parallel for schedule(static) if (N >= OR_PAR_MIN)
        for (long n = 0; n < N; n++) {
            x[n] = fma(omega, s[n], fma(alpha, p[n], x[n]));
            r[n] = fma(-omega, t[n], s[n]);
        }
        rho_prev = rho;
        rho = or_dot(N, rh, r);
        rr = or_dot(N, r, r);
        rn = sqrt(rr);
        if (tr) tr[7] = rr;
        if (rn <= tol * bn) { status = OG_OK; iters = it; goto done_rel; }
    }
    iters = maxit;
    status = OG_NOT_CONVERGED;
done_rel:
    rel = rn / bn;
done:
    if (info) { info->iters = iters; info->status = status; info->restarts = restarts; info->rel_resid = rel; }
    free(r); free(rh); free(p); free(v); free(s); free(t); free(y);
    return status;
}

/* ------------------------------------------------------------------ §3.7 */
/* u_e = u*_e + d_e (p'_P - p'_E) on interior and outlet faces (outlet ghost
 * p' = 0, Q13/Q27); identity (wall) faces are copied; p = p + urf_p p'. */
void or_correct(const og_grid *g, const og_params *pr,
                const double *us, const double *vs, const double *ws,
                const double *dxv, const double *dyv, const double *dzv,
                const double *pp, const double *p,
                double *u, double *v, double *w, double *pnew)
{
    const double *vin[3] = {us, vs, ws};
    const double *dd[3] = {dxv, dyv, dzv};
    double *vout[3] = {u, v, w};
#pragma omp parallel for collapse(2) schedule(static) if (ncell(g) >= OR_PAR_MIN)
    for (int k = 0; k < g->nz; k++)
        for (int j = 0; j < g->ny; j++)
            for (int i = 0; i < g->nx; i++) {
                const int P[3] = {i, j, k};
                const long n = at(g, P);
                for (int a = 0; a < 3; a++) {
                    if (P[a] <= ext(g, a) - 2) {
                        int E[3] = {i, j, k}; E[a] += 1;
                        vout[a][n] = vin[a][n] + dd[a][n] * (pp[n] - pp[at(g, E)]);
                    } else if (a == 2 && g->bc_zhi == OG_OUTLET) {
                        vout[a][n] = vin[a][n] + dd[a][n] * (pp[n] - 0.0);
                    } else {
                        vout[a][n] = vin[a][n];
                    }
                }
                pnew[n] = p[n] + pr->urf_p * pp[n];
            }
}

/* ------------------------------------------------------------------ §3.8 */
static og_eqsys alloc_sys(long N, int sym)
{
    og_eqsys e;
    e.aP = calloc(N, sizeof(double)); e.aE = calloc(N, sizeof(double));
    e.aN = calloc(N, sizeof(double)); e.aT = calloc(N, sizeof(double));
    e.b = calloc(N, sizeof(double)); e.d = calloc(N, sizeof(double));
    if (sym) { e.aW = e.aS = e.aB = NULL; }
    else { e.aW = calloc(N, sizeof(double)); e.aS = calloc(N, sizeof(double)); e.aB = calloc(N, sizeof(double)); }
    return e;
}
static void free_sys(og_eqsys *e)
{
    free(e->aP); free(e->aE); free(e->aN); free(e->aT); free(e->b); free(e->d);
    free(e->aW); free(e->aS); free(e->aB);
}

int or_simple_iter(const og_grid *g, const og_params *pr, int n_scalars, og_state *st,
                   double resid[4], int iters[8], int status[8])
{
    if (!grid_ok(g) || n_scalars < 0 || n_scalars > 4) return OG_ERR_ARG;
    const long N = ncell(g);
    double *star[3], *dv[3];
    double R[3];
    int worst = OG_OK;
    for (int q = 0; q < 8; q++) { iters[q] = 0; status[q] = OG_OK; }
    /* momentum predictors from the snapshot (u, v, w solved independently) */
    for (int c = 0; c < 3; c++) {
        og_eqsys e = alloc_sys(N, 0);
        double r2[2];
        int rc = or_assemble_mom(g, pr, c, st, &e, r2);
        if (rc < 0) { free_sys(&e); return rc; }
        R[c] = r2[0] / (r2[1] > 1e-30 ? r2[1] : 1e-30);
        star[c] = malloc(sizeof(double) * N);
        memcpy(star[c], c == 0 ? st->u : (c == 1 ? st->v : st->w), sizeof(double) * N);
        og_solve_info inf;
        or_bicgstab(g, &e, star[c], pr->lin_tol_mom, pr->lin_maxit_mom, &inf, NULL);
        iters[c] = inf.iters; status[c] = inf.status;
        if (inf.status < 0) worst = inf.status;
        dv[c] = e.d; e.d = NULL;
        free_sys(&e);
    }
    /* scalars from the same snapshot (Q22) */
    double *phinew[4] = {NULL, NULL, NULL, NULL};
    for (int s = 0; s < n_scalars; s++) {
        og_eqsys e = alloc_sys(N, 0);
        double r2[2];
        int rc = or_assemble_scalar(g, pr, s, st, &e, r2);
        if (rc < 0) { free_sys(&e); return rc; }
        phinew[s] = malloc(sizeof(double) * N);
        memcpy(phinew[s], st->phi[s], sizeof(double) * N);
        og_solve_info inf;
        or_bicgstab(g, &e, phinew[s], pr->lin_tol_phi, pr->lin_maxit_phi, &inf, NULL);
        iters[4 + s] = inf.iters; status[4 + s] = inf.status;
        if (inf.status < 0) worst = inf.status;
        free_sys(&e);
    }
    /* pressure correction */
    og_eqsys e = alloc_sys(N, 1);
    double cont;
    int rc = or_assemble_pp(g, pr, st, star[0], star[1], star[2], dv[0], dv[1], dv[2], &e, &cont);
    if (rc < 0) { free_sys(&e); return rc; }
    double *pp = calloc(N, sizeof(double));
    og_solve_info inf;
    or_bicgstab(g, &e, pp, pr->lin_tol_pp, pr->lin_maxit_pp, &inf, NULL);
    iters[3] = inf.iters; status[3] = inf.status;
    if (inf.status < 0) worst = inf.status;
    free_sys(&e);
    double *pn = malloc(sizeof(double) * N);
    or_correct(g, pr, star[0], star[1], star[2], dv[0], dv[1], dv[2], pp, st->p, st->u, st->v, st->w, pn);
    memcpy(st->p, pn, sizeof(double) * N);
    for (int s = 0; s < n_scalars; s++) { memcpy(st->phi[s], phinew[s], sizeof(double) * N); free(phinew[s]); }
    resid[0] = R[0]; resid[1] = R[1]; resid[2] = R[2]; resid[3] = cont;
    for (int c = 0; c < 3; c++) { free(star[c]); free(dv[c]); }
    free(pp); free(pn);
    return worst;
}

/* ------------------------------------------------------------------ §3.9 */
/* Particle -> grid coupling on the PIC device (NEXT-2; "F is the
 * interpolated force from the parcel location to the corresponding fluid
 * cell", PAPER.md:97 explicit vs implicit refresh, "bilinear
 * numerical interpolation" of eps_p; SPEC.md:200-208 deposit
 * Syamlal-O'Brien drag).  Plain definition: parcels in ascending index order,
 * the 8 nodes of each parcel in (kk, jj, ii) order, every expression exactly
 * as DESIGN.md §3.9 writes it.
 *
 * Weights along one axis:
 *   cell-centred lattice: xi = x/h - 0.5, node positions (i + 0.5) h;
 *   face lattice of the velocity component along its own axis: xi = x/h - 1.0,
 *   node positions (i + 1) h, node -1 = the unstored boundary face.
 *   i0 = floor(xi), f = xi - i0; nodes i0 (weight 1 - f) and i0 + 1 (weight f).
 *   Cell nodes are clamped into [0, n-1] (a parcel within half a cell of a
 *   wall folds both weights onto the boundary cell: partition of unity kept);
 *   face nodes are clamped into [-1, n-1]. */
static double pic_vs(double dp) { return (((OG_PI / 6.0) * dp) * dp) * dp; }

static void pic_axis(double x, double h, int n, int face, int node[2], double w[2])
{
    const double xi = face ? x / h - 1.0 : x / h - 0.5;
    const double fl = floor(xi);
    const double f = xi - fl;
    int i0 = (int)fl, i1 = i0 + 1;
    const int lo = face ? -1 : 0;
    i0 = i0 < lo ? lo : (i0 > n - 1 ? n - 1 : i0);
    i1 = i1 < lo ? lo : (i1 > n - 1 ? n - 1 : i1);
    node[0] = i0; node[1] = i1;
    w[0] = 1.0 - f; w[1] = f;
}

/* 8 nodes and weights of parcel position X for the lattice whose face axis is
 * `fa` (-1: cell-centred on every axis). */
static void pic_stencil(const og_grid *g, const double X[3], int fa, int nd[3][2], double w[3][2])
{
    for (int a = 0; a < 3; a++) pic_axis(X[a], spacing(g, a), ext(g, a), a == fa, nd[a], w[a]);
}

/* value of velocity component c at face node (i, j, k); index -1 along c is
 * the unstored boundary face: w_in for the z INLET, else 0 (wall). */
static double pic_face_value(const og_grid *g, const double *f, int c, const int q[3])
{
    if (q[c] == -1) return (c == 2 && g->bc_zlo == OG_INLET) ? g->w_in : 0.0;
    return f[at(g, q)];
}

static double pic_interp(const og_grid *g, const double *f, int fa, const double X[3])
{
    int nd[3][2];
    double w[3][2];
    pic_stencil(g, X, fa, nd, w);
    double val = 0.0;
    for (int kk = 0; kk < 2; kk++)
        for (int jj = 0; jj < 2; jj++)
            for (int ii = 0; ii < 2; ii++) {
                const int q[3] = {nd[0][ii], nd[1][jj], nd[2][kk]};
                const double W = (w[0][ii] * w[1][jj]) * w[2][kk];
                const double v = fa < 0 ? f[at(g, q)] : pic_face_value(g, f, fa, q);
                val = val + W * v;
            }
    return val;
}

static int pic_ok(const og_grid *g, const og_parcels *pc, const og_pic_params *pp)
{
    if (!grid_ok(g) || !pc || !pp || pc->n < 0) return 0;
    if (!(pp->d_p > 0.0)) return 0;
    const double L[3] = {g->nx * g->dx, g->ny * g->dy, g->nz * g->dz};
    for (long p = 0; p < pc->n; p++) {
        const double X[3] = {pc->x[p], pc->y[p], pc->z[p]};
        for (int a = 0; a < 3; a++)
            if (!(X[a] >= 0.0 && X[a] <= L[a])) return 0;
        if (!(pc->omega[p] >= 0.0)) return 0;
    }
    return 1;
}

/* D1: eps_g[c] = max(1 - (sum_p W_pc (omega_p Vs)) / V, eps_min) */
int or_pic_deposit_eps(const og_grid *g, const og_pic_params *pp, const og_parcels *pc, double *eps_g)
{
    if (!pic_ok(g, pc, pp)) return OG_ERR_ARG;
    const long N = ncell(g);
    const double Vs = pic_vs(pp->d_p), V = volume(g);
    for (long n = 0; n < N; n++) eps_g[n] = 0.0;
    for (long p = 0; p < pc->n; p++) {
        const double X[3] = {pc->x[p], pc->y[p], pc->z[p]};
        const double vol = pc->omega[p] * Vs;
        int nd[3][2];
        double w[3][2];
        pic_stencil(g, X, -1, nd, w);
        for (int kk = 0; kk < 2; kk++)
            for (int jj = 0; jj < 2; jj++)
                for (int ii = 0; ii < 2; ii++) {
                    const int q[3] = {nd[0][ii], nd[1][jj], nd[2][kk]};
                    const double W = (w[0][ii] * w[1][jj]) * w[2][kk];
                    eps_g[at(g, q)] += W * vol;
                }
    }
    for (long n = 0; n < N; n++) {
        const double e = 1.0 - eps_g[n] / V;
        eps_g[n] = e < pp->eps_min ? pp->eps_min : e;
    }
    return OG_OK;
}

/* x^y for x > 0, CORRECTLY ROUNDED (DESIGN.md §3.9 reading, the same contract
 * as the dots of §3.1): the exact real x^y rounded once to nearest-even.
 * Evaluated with libquadmath's powq on the exactly converted binary64
 * arguments (113-bit significand, error well below 2^-100 relative), then
 * rounded to binary64.  That rounding is the correctly rounded value unless
 * the quad result lies within the quad error of a binary64 rounding boundary
 * (a midpoint between neighbouring doubles); that case is detected and
 * reported as NaN plus the or_pow_ambiguous counter, never silently rounded. */
static long g_pow_ambiguous = 0;

long or_pow_ambiguous(void) { return g_pow_ambiguous; }

double or_pow(double x, double y)
{
    const __float128 q = powq((__float128)x, (__float128)y);
    const double d = (double)q;                       /* round to nearest-even */
    /* distance of q from the nearer of the two midpoints around d */
    const double up = nextafter(d, INFINITY), dn = nextafter(d, -INFINITY);
    const __float128 mid_hi = ((__float128)d + (__float128)up) / 2, mid_lo = ((__float128)d + (__float128)dn) / 2;
    const __float128 dist = fminq(fabsq(q - mid_hi), fabsq(q - mid_lo));
    if (dist <= fabsq(q) * 0x1p-100Q) {
        g_pow_ambiguous++;
        return NAN;
    }
    return d;
}

/* Syamlal-O'Brien per-parcel drag coefficient K (N s / m): the force on the
 * gas is -K (u_g - u_p); K = beta_d (omega Vs) / eps_s with beta_d of
 * SPEC.md:285-289, written without the eps_s that cancels. */
double or_pic_drag_coef(const og_params *pr, const og_pic_params *pp, double eg, double slip, double omega)
{
    double Re = ((pr->rho * pp->d_p) * slip) / pr->mu;
    Re = Re < 1e-12 ? 1e-12 : Re;
    const double A = or_pow(eg, 4.14);
    const double B = eg <= 0.85 ? 0.8 * or_pow(eg, 1.28) : or_pow(eg, 2.65);
    const double q = 0.06 * Re;
    const double Vr = 0.5 * ((A - q) + sqrt((q * q + (0.12 * Re) * (2.0 * B - A)) + A * A));
    double Cd = 0.63 + 4.8 / sqrt(Re / Vr);
    Cd = Cd * Cd;
    return (omega * pic_vs(pp->d_p)) * ((((0.75 * Cd) * eg) * pr->rho) * slip) / ((Vr * Vr) * pp->d_p);
}

/* D2: per parcel interpolate eps_g (cell lattice) and u_g (staggered
 * lattices), slip, K; deposit beta = sum_p W (K / V) and
 * sbeta_c = sum_p W ((K u_p,c) / V) (the division is per parcel, so the sums
 * are the fields: no pass over the grid after the deposit).
 * diag (optional, may be NULL): per parcel {eps_g@p, u_g@p, v_g@p, w_g@p, K}.
 * sabs (optional, may be NULL): 3 x N, sum W |(K u_p,c) / V| (error scale of sbeta). */
int or_pic_drag(const og_grid *g, const og_params *pr, const og_pic_params *pp, const og_parcels *pc,
                const double *eps_g, const double *u, const double *v, const double *w,
                double *beta, double *sbu, double *sbv, double *sbw, double *diag, double *sabs)
{
    if (!pic_ok(g, pc, pp)) return OG_ERR_ARG;
    const long N = ncell(g);
    const double V = volume(g);
    const double *vel[3] = {u, v, w};
    double *sb[3] = {sbu, sbv, sbw};
    for (long n = 0; n < N; n++) {
        beta[n] = 0.0; sbu[n] = 0.0; sbv[n] = 0.0; sbw[n] = 0.0;
        if (sabs) { sabs[n] = 0.0; sabs[N + n] = 0.0; sabs[2 * N + n] = 0.0; }
    }
    for (long p = 0; p < pc->n; p++) {
        const double X[3] = {pc->x[p], pc->y[p], pc->z[p]};
        const double up[3] = {pc->u[p], pc->v[p], pc->w[p]};
        const double eg = pic_interp(g, eps_g, -1, X);
        double ug[3];
        for (int c = 0; c < 3; c++) ug[c] = pic_interp(g, vel[c], c, X);
        const double sx = ug[0] - up[0], sy = ug[1] - up[1], sz = ug[2] - up[2];
        const double slip = sqrt((sx * sx + sy * sy) + sz * sz);
        const double K = or_pic_drag_coef(pr, pp, eg, slip, pc->omega[p]);
        if (diag) {
            diag[5 * p + 0] = eg; diag[5 * p + 1] = ug[0]; diag[5 * p + 2] = ug[1]; diag[5 * p + 3] = ug[2];
            diag[5 * p + 4] = K;
        }
        const double KV = K / V;
        double KuV[3];
        for (int c = 0; c < 3; c++) KuV[c] = (K * up[c]) / V;
        int nd[3][2];
        double wt[3][2];
        pic_stencil(g, X, -1, nd, wt);
        for (int kk = 0; kk < 2; kk++)
            for (int jj = 0; jj < 2; jj++)
                for (int ii = 0; ii < 2; ii++) {
                    const int q[3] = {nd[0][ii], nd[1][jj], nd[2][kk]};
                    const double W = (wt[0][ii] * wt[1][jj]) * wt[2][kk];
                    const long n = at(g, q);
                    beta[n] += W * KV;
                    for (int c = 0; c < 3; c++) {
                        sb[c][n] += W * KuV[c];
                        if (sabs) sabs[c * N + n] += W * fabs(KuV[c]);
                    }
                }
    }
    return OG_OK;
}

/* ------------------------------------------------------------------ §3.11 */
/* Time loop (NEXT-3; "initial time step was set to 1 ms and
 * varied depending on the convergence of SIMPLE iterations with the given
 * tolerance and maximum number of iterations"; PAPER.md:165 gradual growth
 * to the maximum 5e-4 s; SPEC.md:388-396 adapt_dt).  Plain definition:
 *   converged within grow_threshold outer iterations -> dt = min(dt*grow, dt_max)
 *   converged later                                  -> dt unchanged
 *   not converged in max_outer, dt > dt_min          -> reject: restore the
 *        step's initial state, dt = max(dt*shrink, dt_min), retry
 *   not converged at dt_min                          -> accept (flagged)
 * On acceptance: time += dt_used, u_old, v_old, w_old <- u, v, w,
 * eps_old <- eps, phi_old <- phi. */
int or_adapt_dt(og_time_ctrl *tc, int outer_iters, int converged)
{
    if (converged) {
        if (outer_iters <= tc->grow_threshold) {
            double d = tc->dt * tc->grow;
            tc->dt = d < tc->dt_max ? d : tc->dt_max;
        }
        return 1;
    }
    if (tc->dt > tc->dt_min) {
        double d = tc->dt * tc->shrink;
        tc->dt = d > tc->dt_min ? d : tc->dt_min;
        return 0;
    }
    return 1; /* accepted at dt_min although not converged */
}

int or_time_step(const og_grid *g, const og_params *pr0, int n_scalars, og_state *st, og_time_ctrl *tc,
                 int *outer_used, double resid[4])
{
    const long N = ncell(g);
    const size_t vb = sizeof(double) * (size_t)N;
    double *save[8];
    double *fld[8] = {st->u, st->v, st->w, st->p, NULL, NULL, NULL, NULL};
    for (int s = 0; s < n_scalars; s++) fld[4 + s] = st->phi[s];
    for (int q = 0; q < 8; q++) {
        save[q] = NULL;
        if (fld[q]) { save[q] = malloc(vb); memcpy(save[q], fld[q], vb); }
    }
    og_params pr = *pr0;
    int rc = OG_OK, accepted = 0, its = 0, conv = 0;
    double dt_used = tc->dt;
    while (!accepted) {
        pr.dt = tc->dt;
        dt_used = tc->dt;
        conv = 0;
        its = 0;
        for (int it = 1; it <= tc->max_outer; it++) {
            int iters[8], status[8];
            rc = or_simple_iter(g, &pr, n_scalars, st, resid, iters, status);
            its = it;
            if (rc < 0 && rc != OG_ERR_BREAKDOWN) goto out;
            double mx = resid[0];
            for (int q = 1; q < 4; q++) mx = resid[q] > mx ? resid[q] : mx;
            if (mx < pr.tol) { conv = 1; break; }
        }
        accepted = or_adapt_dt(tc, its, conv);
        if (!accepted) {
            tc->rejected += 1;
            for (int q = 0; q < 8; q++)
                if (fld[q]) memcpy(fld[q], save[q], vb);
        }
    }
    tc->time += dt_used;
    tc->steps += 1;
    memcpy(st->u_old, st->u, vb); memcpy(st->v_old, st->v, vb); memcpy(st->w_old, st->w, vb);
    memcpy(st->eps_old, st->eps, vb);
    for (int s = 0; s < n_scalars; s++) memcpy(st->phi_old[s], st->phi[s], vb);
    rc = conv ? OG_OK : OG_NOT_CONVERGED;
out:
    if (outer_used) *outer_used = its;
    for (int q = 0; q < 8; q++) free(save[q]);
    return rc;
}
