/* oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, CPU fp64 reference of the SIMPLE + BiCGSTAB hot path of
 * arXiv 2211.15605 (§2.1 Eqs. 1-2, §2.2.2, §3 "No preconditioners").
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  It shares no code with the CUDA path
 * (paper_2211_15605_b200/csrc) and never includes include/mfx.h.
 *
 * Every formula follows DESIGN.md §3 ("Discrete definitions"), which restates
 * the paper's equations plus the readings Q1-Q27 of SURVEY.md §8(c).
 */
#ifndef MFX_ORACLE_H
#define MFX_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

enum { OG_WALL = 0, OG_INLET = 1, OG_OUTLET = 2, OG_DIRICHLET_TEST = 3 };
enum { OG_OK = 0, OG_NOT_CONVERGED = 1, OG_ERR_ARG = -1, OG_ERR_NONFINITE = -2,
       OG_ERR_ZERO_DIAG = -3, OG_ERR_BREAKDOWN = -4 };

typedef struct {
    int nx, ny, nz;
    double dx, dy, dz;
    int bc_zlo, bc_zhi;          /* x and y sides are always no-slip walls */
    double w_in, phi_in, phi_out;
} og_grid;

typedef struct {
    double rho, mu, gamma_phi[4], g[3], dt, urf_mom, urf_p, urf_phi;
    double tol, lin_tol_mom, lin_tol_pp, lin_tol_phi;
    int lin_maxit_mom, lin_maxit_pp, lin_maxit_phi;
    int face_eps_upwind;        /* §3.12: 1 = convective face eps upwinded by the snapshot velocity */
} og_params;

typedef struct {
    double *eps, *eps_old, *u, *v, *w, *u_old, *v_old, *w_old, *p;
    double *beta, *sbeta_u, *sbeta_v, *sbeta_w;
    double *phi[4], *phi_old[4];
    const unsigned char *blocked;   /* NULL or N flags: 1 = BLOCKED cell (internal obstacle, §3.10) */
} og_state;

/* Momentum / scalar systems use all 7 coefficient arrays; the p' system is
 * stored symmetrically: aE/aN/aT hold c_x/c_y/c_z and aW/aS/aB are NULL. */
typedef struct { double *aP, *aE, *aW, *aN, *aS, *aT, *aB, *b, *d; } og_eqsys;

typedef struct {
    int iters, status, restarts;
    double rel_resid;          /* recursive ||r|| / ||b|| at exit */
} og_solve_info;

/* correctly rounded sums (exact sum, rounded once) */
double or_fsum(long n, const double *x);
double or_dot(long n, const double *a, const double *b);
double or_sumabs(long n, const double *x);

void or_spmv(const og_grid *g, const og_eqsys *A, const double *x, double *y);

int or_assemble_mom(const og_grid *g, const og_params *pr, int comp, const og_state *st,
                    og_eqsys *out, double resid2[2]);
int or_assemble_pp(const og_grid *g, const og_params *pr, const og_state *st,
                   const double *us, const double *vs, const double *ws,
                   const double *dxv, const double *dyv, const double *dzv,
                   og_eqsys *out, double *cont);
int or_assemble_scalar(const og_grid *g, const og_params *pr, int sid, const og_state *st,
                       og_eqsys *out, double resid2[2]);

/* trace (optional, may be NULL): per iteration 8 doubles
 * {rho, sigma, alpha, ss, ts, tt, omega, rr}; capacity maxit rows. */
int or_bicgstab(const og_grid *g, const og_eqsys *A, double *x, double tol, int maxit,
                og_solve_info *info, double *trace);

void or_correct(const og_grid *g, const og_params *pr,
                const double *us, const double *vs, const double *ws,
                const double *dxv, const double *dyv, const double *dzv,
                const double *pp, const double *p,
                double *u, double *v, double *w, double *pnew);

/* One SIMPLE outer iteration (serial definition; equation decomposition does
 * not change the discrete result).
 * st->u,v,w,p (and phi[s]) are updated in place.  resid[4] = R_u,R_v,R_w,R_cont;
 * iters[8] = u,v,w,pp,phi0..3 ; status[8] likewise. */
int or_simple_iter(const og_grid *g, const og_params *pr, int n_scalars, og_state *st,
                   double resid[4], int iters[8], int status[8]);

/* §3.9 particle -> grid coupling (NEXT-2).  Parcels: SoA, positions in
 * [0, L] per axis, velocities, statistical weight omega >= 0. */
#define OG_PI 3.14159265358979323846
typedef struct { const double *x, *y, *z, *u, *v, *w, *omega; long n; } og_parcels;
typedef struct { double d_p, eps_min; } og_pic_params;

int or_pic_deposit_eps(const og_grid *g, const og_pic_params *pp, const og_parcels *pc, double *eps_g);
void or_set_mode(int threads, int naive);   /* threads (<= 0: keep), naive = plain sums (timing only) */
int or_max_threads(void);
double or_pow(double x, double y);   /* correctly rounded x^y */
long or_pow_ambiguous(void);           /* calls whose rounding could not be decided (NaN returned) */
double or_pic_drag_coef(const og_params *pr, const og_pic_params *pp, double eg, double slip, double omega);
int or_pic_drag(const og_grid *g, const og_params *pr, const og_pic_params *pp, const og_parcels *pc,
                const double *eps_g, const double *u, const double *v, const double *w,
                double *beta, double *sbu, double *sbv, double *sbw, double *diag, double *sabs);

/* §3.11 time loop: adaptive dt controller */
typedef struct {
    double dt, dt_min, dt_max, grow, shrink;
    int grow_threshold, max_outer;
    double time;
    int steps, rejected;
} og_time_ctrl;
/* returns 1 if the step is accepted; updates tc->dt */
int or_adapt_dt(og_time_ctrl *tc, int outer_iters, int converged);
/* one accepted time step (retries included); returns OG_OK (converged),
 * OG_NOT_CONVERGED (accepted at dt_min) or an error */
int or_time_step(const og_grid *g, const og_params *pr, int n_scalars, og_state *st, og_time_ctrl *tc,
                 int *outer_used, double resid[4]);

#ifdef __cplusplus
}
#endif
#endif
