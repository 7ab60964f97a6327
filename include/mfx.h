/* mfx.h -- C ABI of libmfx.so: the B200-native hot path of arXiv 2211.15605
 * ("equation decomposition" of the MP-PIC gas phase, §2.2.2).
 *
 * One SIMPLE outer iteration = assemble the
 * 7-point finite-volume stencil of u, v, w momentum (Eq. 2) and of the
 * pressure correction p' (Eq. 1), plus optional transported scalars
 * (P:85), solve each with unpreconditioned BiCGSTAB, correct, and
 * exchange the state between equation-owning GPUs once.
 * The discrete definitions are written out in DESIGN.md §3.
 *
 * Conventions for every entry point:
 *  - Fields are caller-owned, contiguous IEEE binary64 DEVICE buffers of
 *    N = nx*ny*nz elements on the calling thread's current device, linear
 *    index n = i + nx*(j + ny*k) (x fastest).  Staggered velocities: u[n] sits
 *    on the +x face of cell n, v on +y, w on +z.
 *  - All calls are stream-ordered on `stream` (a cudaStream_t passed as
 *    void*; NULL = legacy default stream) and never allocate device memory,
 *    except mfx_ctx_create.  Nothing throws; every call returns mfx_status.
 *  - Argument errors (NULL pointer, bad sizes, unsupported boundary
 *    combination, workspace too small) return MFX_ERR_ARG before any launch;
 *    mfx_last_error() (thread-local) describes the first error.
 *  - Device-side problems (non-finite coefficient, zero diagonal) are latched
 *    in the workspace and reported by mfx_ws_check() (synchronises `stream`)
 *    with the first offending linear cell index in mfx_last_error().
 *  - Requirements: nx, ny, nz >= 2 (an odd nx is accepted; its rows are not
 *    16-byte aligned, so the TMA kernels give way to the grid-stride ones,
 *    which produce the same bits), device arrays 16-byte aligned,
 *    x/y sides are no-slip walls, z- INLET or WALL, z+ OUTLET or WALL
 *    (DIRICHLET_TEST: scalar equations only).
 */
#ifndef MFX_H
#define MFX_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MFX_OK = 0,
    MFX_NOT_CONVERGED = 1,     /* status, not an error: last iterate returned (Q5) */
    MFX_ERR_ARG = -1,
    MFX_ERR_NONFINITE = -2,
    MFX_ERR_ZERO_DIAG = -3,
    MFX_ERR_BREAKDOWN = -4,    /* SPEC.md:374, after one restart */
    MFX_ERR_CUDA = -5,
    MFX_ERR_NCCL = -6
} mfx_status;

typedef enum { MFX_EQ_U = 0, MFX_EQ_V = 1, MFX_EQ_W = 2, MFX_EQ_PP = 3, MFX_EQ_SCALAR = 4 } mfx_eq_kind;

typedef enum { MFX_BC_WALL = 0, MFX_BC_INLET = 1, MFX_BC_OUTLET = 2, MFX_BC_DIRICHLET_TEST = 3 } mfx_bc;

typedef struct {
    int nx, ny, nz;
    double dx, dy, dz;          /* uniform spacing (m) */
    int bc_zlo, bc_zhi;         /* mfx_bc; x/y sides are walls */
    double w_in;                /* inlet normal velocity (m/s) */
    double phi_in, phi_out;     /* scalar Dirichlet values (inlet; test-only top) */
} mfx_grid;

typedef struct {
    double rho, mu;             /* gas density, viscosity */
    double gamma_phi[4];        /* scalar diffusivities (Q21) */
    double g[3];                /* gravity (m/s^2); paper: -z */
    double dt;                  /* time step (s) */
    double urf_mom, urf_p, urf_phi;  /* under-relaxation */
    double tol;                 /* SIMPLE residual tolerance */
    double lin_tol_mom, lin_tol_pp, lin_tol_phi;
    int lin_maxit_mom, lin_maxit_pp, lin_maxit_phi;
    int face_eps_upwind;        /* 0: central face eps in convective fluxes (reading Q9); 1: upwind cell
                                   by the sign of the snapshot velocity (MFiX-style) */
    int packed_state;           /* multi-rank contexts: 1 = on every rank u, v, w, p are ONE contiguous
                                   [u|v|w|p] block (v = u + N, w = u + 2N, p = u + 3N), so the BCAST
                                   phase sends them as one broadcast of 4N doubles (mfx_simple_iter
                                   returns MFX_ERR_ARG if they are not).  Like every parameter it must
                                   be identical on all ranks; 0 = four grouped broadcasts. */
} mfx_params;

/* Snapshot state (device pointers, N each).  Read-only to assembly; u, v, w,
 * p, phi[] are overwritten by mfx_simple_iter. */
typedef struct {
    double *eps, *eps_old;                /* gas volume fraction now / old time */
    double *u, *v, *w;                    /* staggered velocities, snapshot m */
    double *u_old, *v_old, *w_old;        /* old-time velocities */
    double *p;                            /* gauge pressure */
    double *beta;                         /* implicit drag coefficient per cell (Q11) */
    double *sbeta_u, *sbeta_v, *sbeta_w;  /* explicit drag source beta*u_s per cell */
    double *phi[4], *phi_old[4];          /* optional scalars (NULL if unused) */
    const unsigned char *blocked;         /* NULL, or N flags, 1 = BLOCKED cell (internal obstacle,
                                             NEXT-3): faces touching it are walls;
                                             velocities on those faces and scalars inside must be 0 */
} mfx_state;

/* Equation system (device pointers, N each).  Momentum/scalar: all seven
 * coefficient arrays, row a_P x_P - sum a_nb x_nb = b.  p': symmetric
 * storage, aE/aN/aT hold the face coefficients c_x/c_y/c_z and aW/aS/aB must
 * be NULL; its diagonal is by definition the ordered row sum
 * a_P = ((((c_W + c_E) + c_S) + c_N) + c_B) + c_T, which
 * mfx_spmv / the solvers rebuild on the fly: they never read aP (may be NULL;
 * mfx_assemble_eq still writes it).  d (momentum only) = eps_f A_f /
 * a_P,relaxed (Q16, Q27). */
typedef struct { double *aP, *aE, *aW, *aN, *aS, *aT, *aB, *b, *d; } mfx_eqsys;

typedef struct {
    int iters;                 /* BiCGSTAB iterations (half-step exit counts 1, Q3) */
    int status;                /* mfx_status */
    int restarts;              /* breakdown restarts taken (0 or 1) */
    double rel_resid;          /* recursive ||r|| / ||b|| at exit */
    double true_rel_resid;     /* ||b - A x|| / ||b|| of the returned iterate, from one extra correctly
                                  rounded apply at exit (reading Q2; 0 when b = 0); with info == NULL
                                  it is not computed */
} mfx_solve_info;

typedef struct {
    double R_u, R_v, R_w, R_cont;   /* SIMPLE residuals (Norm_g = 1 P:157) */
    double R_phi[4];
    int iters[8];                   /* u, v, w, pp, phi0..3 */
    int status[8];
    int converged;                  /* max(R_u,R_v,R_w,R_cont) < tol */
    double rel_resid[8];            /* per equation: recursive ||r||/||b|| at solver exit */
    double true_rel_resid[8];       /* per equation: ||b - A x||/||b|| of the returned iterate */
} mfx_resid;

const char *mfx_last_error(void);
const char *mfx_version(void);

/* Initialise a freshly allocated workspace (clears reduction tickets and the
 * error latch).  Must be called once before first use. */
mfx_status mfx_ws_init(void *ws, size_t ws_bytes, void *stream);

/* Bytes of device workspace needed to assemble and solve one equation of
 * `kind` on `grid` (solver vectors r, r^, p x2, v x2, t + reduction scratch). */
size_t mfx_workspace_bytes(const mfx_grid *grid, int kind);

/* Reads and clears the device-side error latch of `ws` (synchronises stream). */
mfx_status mfx_ws_check(void *ws, size_t ws_bytes, void *stream);

/* a-1/a-2/a-3: assemble one equation's coefficients.
 *  kind MFX_EQ_U/V/W: momentum; needs state->eps..sbeta_*; out->d required.
 *  kind MFX_EQ_PP: star = {u*, v*, w*, d_x, d_y, d_z} (device); out aW/aS/aB NULL.
 *  kind MFX_EQ_SCALAR: scalar_id 0..3, uses phi[scalar_id], phi_old[scalar_id].
 *  resid2 (device, may be NULL): momentum/scalar {sum|res|, sum|aP u|};
 *  p': {sum|b|, 0}.  Sums are correctly rounded. */
mfx_status mfx_assemble_eq(int kind, int scalar_id, const mfx_grid *grid, const mfx_params *params,
                           const mfx_state *state, const double *const star[6], mfx_eqsys *out,
                           double *resid2, void *ws, size_t ws_bytes, void *stream);

/* a-4: y = A x with the canonical term order of DESIGN.md §3.2. */
mfx_status mfx_spmv(int kind, const mfx_grid *grid, const mfx_eqsys *A, const double *x, double *y,
                    void *stream);

/* a-5/a-6: unpreconditioned BiCGSTAB on A x = A->b.
 * x: in x0, out solution (last iterate if not converged).  info (host) may be
 * NULL: then the call is fully asynchronous and runs the device loop to
 * convergence without host round trips; otherwise it synchronises `stream`
 * once at exit.  Returns the solve status (MFX_OK / MFX_NOT_CONVERGED /
 * MFX_ERR_BREAKDOWN) when info != NULL, else MFX_OK after launching. */
mfx_status mfx_bicgstab_solve(int kind, const mfx_grid *grid, const mfx_eqsys *A, double *x,
                              double tol, int maxit, void *ws, size_t ws_bytes,
                              mfx_solve_info *info, void *stream);

/* a-7: SIMPLE correction: u = u* + d (p'_P - p'_E), p = p + urf_p p'.
 * star = {u*, v*, w*, d_x, d_y, d_z}; outputs may alias nothing in star. */
mfx_status mfx_correct(const mfx_grid *grid, const mfx_params *params, const double *const star[6],
                       const double *pp, const double *p, double *u, double *v, double *w,
                       double *p_new, void *stream);

/* ---------------------------------------------------------------- particle -> grid coupling (NEXT-2) */
/* The PIC device's coupling terms: "F is the
 * interpolated force from the parcel location to the corresponding fluid
 * cell"; PAPER.md:97 explicit (once per time step) or implicit (head of every
 * SIMPLE iteration) refresh; PAPER.md:131 interpolation of eps_p; closure of
 * SPEC.md:285-289 (Syamlal-O'Brien).
 * Parcels: caller-owned DEVICE arrays of n doubles each (structure of arrays):
 * position x, y, z (m, inside [0, nx dx] x [0, ny dy] x [0, nz dz]), velocity
 * u, v, w (m/s), statistical weight omega (real particles per parcel, >= 0).
 * A parcel outside the domain, or with a negative/NaN weight, is skipped and
 * latched in `ws` (mfx_ws_check then returns MFX_ERR_ARG with its index). */
typedef struct { const double *x, *y, *z, *u, *v, *w, *omega; long long n; } mfx_parcels;
typedef struct {
    double d_p;        /* particle diameter (m) */
    double eps_min;    /* floor of the deposited gas fraction */
} mfx_pic_params;

/* eps_g[c] = max(1 - sum_p W_pc (omega_p Vs) / V, eps_min), Vs = pi d_p^3 / 6,
 * W_pc = trilinear weight of cell centre c (nodes clamped into the grid).
 * eps_g (device, N) is overwritten.  Sums in arrival order (fp64 atomics):
 * equal to the parcel-ordered definition within (m - 1) u sum|terms| per cell. */
mfx_status mfx_pic_deposit_eps(const mfx_grid *grid, const mfx_pic_params *pic, const mfx_parcels *parcels,
                               double *eps_g, void *ws, size_t ws_bytes, void *stream);

/* Per parcel p: eps_g and the staggered u, v, w interpolated to the parcel
 * (trilinear; the unstored boundary face carries 0 at walls and w_in at the
 * inlet), slip = |u_g - u_p|, K_p = Syamlal-O'Brien beta_d omega_p Vs / eps_s
 * (N s/m); then beta[c] = sum_p W_pc (K_p / V) and
 * sbeta_a[c] = sum_p W_pc ((K_p u_p,a) / V): the cell-centred implicit drag
 * coefficient and explicit source of mfx_state (reading Q11).  Outputs
 * (device, N each) are overwritten; K (device, n, may be NULL) receives K_p. */
mfx_status mfx_pic_drag(const mfx_grid *grid, const mfx_params *params, const mfx_pic_params *pic,
                        const mfx_parcels *parcels, const double *eps_g, const double *u, const double *v,
                        const double *w, double *beta, double *sbeta_u, double *sbeta_v, double *sbeta_w,
                        double *K, void *ws, size_t ws_bytes, void *stream);

/* Binned copy of the parcels: a deterministic counting sort by BASE cell (the
 * clamped lower corner floor(x/h - 0.5) of the parcel's trilinear stencil),
 * ascending original index inside a bin, so the binned order is unique.
 * out = 7 device arrays x, y, z, u, v, w, omega of n (must not alias the
 * input); orig (device, n, may be NULL) = original index of each binned
 * parcel; bin_start (device, N + 1, may be NULL) = first binned position of
 * each base cell (bin_start[N] = n).  scratch: device buffer of at least
 * mfx_pic_sort_scratch_bytes(grid, n) bytes.  Parcels move once per time step,
 * so one binning serves every SIMPLE iteration of an implicit coupling. */
size_t mfx_pic_sort_scratch_bytes(const mfx_grid *grid, long long n_parcels);
mfx_status mfx_pic_sort(const mfx_grid *grid, const mfx_pic_params *pic, const mfx_parcels *parcels,
                        double *const out[7], unsigned int *orig, unsigned int *bin_start, void *scratch,
                        size_t scratch_bytes, void *stream);

/* The two deposits on binned parcels, as gathers: every node sums, in
 * ascending ORIGINAL parcel index, the contributions of the parcels whose
 * stencil contains it -- the exact sequence of additions of the parcel-ordered
 * definition, so the fields are bitwise those of the
 * definition and do not depend on scheduling (no atomics).  vals: device
 * scratch of 4 n (eps) or 7 n (drag) doubles, n = parcel count: the
 * per-parcel deposit values, then each parcel's lattice coordinates (computed
 * once, read by the up to 8 nodes that gather the parcel).  K (may be NULL) is per binned
 * parcel.  Invalid parcels contribute nothing and are latched in ws by their
 * original index. */
mfx_status mfx_pic_deposit_eps_binned(const mfx_grid *grid, const mfx_pic_params *pic,
                                      const mfx_parcels *binned, const unsigned int *orig,
                                      const unsigned int *bin_start, double *eps_g, double *vals, void *ws,
                                      size_t ws_bytes, void *stream);
mfx_status mfx_pic_drag_binned(const mfx_grid *grid, const mfx_params *params, const mfx_pic_params *pic,
                               const mfx_parcels *binned, const unsigned int *orig, const unsigned int *bin_start,
                               const double *eps_g, const double *u, const double *v, const double *w,
                               double *beta, double *sbeta_u, double *sbeta_v, double *sbeta_w, double *K,
                               double *vals, void *ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------- dump / restart (NEXT-4) */
/* MPXD state dumps (PAPER.md:119 restarts, PAPER.md:121
 * Eq. 6 comparisons; layout in DESIGN.md §13): a packed little-endian header
 * {"MPXD", version 1, nx, ny, nz, n_parcels, time, dt, n_fields}, a table of
 * named fields (8-byte name, kind 0 = cell field of N, 1 = parcel array),
 * then the binary64 arrays.  Dumped fields: eps, eps_old, u, v, w, u_old,
 * v_old, w_old, p, beta, sbu, sbv, sbw, phi<s>/phio<s> for s < n_scalars, and
 * px..pomega when parcels (may be NULL) are given.  Device buffers are copied
 * on `stream` (synchronises it); the file is written / read with stdio.
 * Errors (unwritable path, bad magic/version, grid mismatch, truncated file,
 * missing field, too small parcel capacity) return MFX_ERR_ARG with the
 * reason in mfx_last_error().  Load of a dump is bitwise: a run continued
 * from a reloaded state equals the uninterrupted run. */
mfx_status mfx_state_dump(const char *path, const mfx_grid *grid, const mfx_state *state, int n_scalars,
                          const mfx_parcels *parcels, double time, double dt, void *stream);
/* Header query without a GPU (host only): grid extents, parcel count, number
 * of scalar fields, time and dt.  Any output pointer may be NULL. */
mfx_status mfx_dump_info(const char *path, int dims[3], long long *n_parcels, int *n_scalars, double *time,
                         double *dt);
/* Loads the state fields into `state` (device buffers of N) and, if
 * parcel_out (7 device arrays x, y, z, u, v, w, omega of parcel_capacity) is
 * given, the parcels; n_parcels / time / dt outputs may be NULL. */
mfx_status mfx_state_load(const char *path, const mfx_grid *grid, mfx_state *state, int n_scalars,
                          double *const parcel_out[7], long long parcel_capacity, long long *n_parcels,
                          double *time, double *dt, void *stream);

/* ---------------------------------------------------------------- equation decomposition */
/* Assignment string: three 1-based GPU ids for U, V, W,
 * a bracketed P list, then optional scalar owners, e.g. "111[1]", "234[1]",
 * "234[1]5678", "234[1234]", "234[23]".  A multi-entry P list is any set of
 * distinct ranks ("a set of devices"): the pressure correction is
 * then solved by the domain-decomposed solver over exactly those ranks (the
 * paper's multi-GPU pressure solver), slab i on rank p_rank[i]
 * (a sub-communicator of the context's); owner[3] = p_rank[0] is P0, which
 * corrects and broadcasts. */
typedef struct {
    int owner[8];       /* 0-based rank owning u, v, w, pp, phi0..phi3; -1 = absent */
    int n_scalars;
    int n_ranks_used;   /* max id */
    int n_p;            /* entries of the P list (1 .. 9, distinct ranks) */
    int p_rank[9];      /* 0-based ranks of the P list in the order written; -1 past n_p */
} mfx_assignment;

mfx_status mfx_parse_assignment(const char *text, int nranks, mfx_assignment *out);

/* Exchange schedule for `rank` (host logic, no device work).  phase 0 =
 * GATHER (momentum owners -> p' owner(s): u*, d per component, plus a
 * 16-double residual record), phase 1 = BCAST (p' owner -> all: u, v, w, p,
 * residual record; scalar owners -> all: phi), phase 2 = PSLAB (multi-GPU p':
 * the slab of every P-list rank -> P0; k0/k1 give the plane range), phase 3 = PIC
 * (the PIC device, rank 0 = "GPU 1" of P:95, broadcasts the refreshed drag
 * fields beta, sbeta_u, sbeta_v, sbeta_w).  Ops are returned in the order they
 * are issued inside one NCCL group. */
enum { MFX_OP_SEND = 0, MFX_OP_RECV = 1, MFX_OP_BCAST = 2 };
enum { MFX_BUF_U = 0, MFX_BUF_V, MFX_BUF_W, MFX_BUF_DX, MFX_BUF_DY, MFX_BUF_DZ,
       MFX_BUF_P, MFX_BUF_PHI0, MFX_BUF_PHI1, MFX_BUF_PHI2, MFX_BUF_PHI3,
       MFX_BUF_META, MFX_BUF_PP, MFX_BUF_BETA, MFX_BUF_SBU, MFX_BUF_SBV, MFX_BUF_SBW, MFX_NBUF };
/* buf MFX_BUF_META moves nslots 16-double residual records starting at slot;
 * other buffers move planes [k0, k1) (k1 = 0: the whole field of N doubles).
 * peer = root for BCAST. */
typedef struct { int op, peer, buf, slot, nslots, k0, k1; } mfx_xfer;
mfx_status mfx_exchange_plan(const mfx_assignment *a, int rank, int phase, mfx_xfer *ops, int max_ops,
                             int *n_ops, int nz /* grid extent, used by PSLAB */);

/* NCCL bootstrap: rank 0 calls mfx_nccl_unique_id and ships the 128 bytes to
 * the other ranks (e.g. torch.distributed.broadcast_object_list). */
mfx_status mfx_nccl_unique_id(unsigned char out[128]);

typedef struct mfx_ctx mfx_ctx;
typedef struct mfx_local_group mfx_local_group;

/* Creates the per-rank context: parses the assignment, allocates the solver
 * workspaces and exchange buffers for the equations this rank owns, and (for
 * nranks > 1) an NCCL communicator from `uid`.  uid may be NULL when nranks == 1. */
mfx_status mfx_ctx_create(const char *assignment, int rank, int nranks, const unsigned char *uid,
                          const mfx_grid *grid, const mfx_params *params, mfx_ctx **out);
void mfx_ctx_destroy(mfx_ctx *ctx);

/* In-process transport (no NCCL): the ranks of a group are host threads of
 * one process, each calling mfx_simple_iter on its own stream (same or
 * different GPUs).  The exchange plan runs as device-to-device pull copies
 * ordered by CUDA events and host barriers.  Used to exercise the multi-rank
 * path on one GPU and for single-node runs without NCCL. */
mfx_status mfx_local_group_create(int nranks, mfx_local_group **out);
void mfx_local_group_destroy(mfx_local_group *group);
mfx_status mfx_ctx_create_local(const char *assignment, int rank, int nranks, mfx_local_group *group,
                                const mfx_grid *grid, const mfx_params *params, mfx_ctx **out);

/* a-8: execute `phase` of the exchange plan on the context's buffers
 * (fields = MFX_NBUF device pointers indexed by MFX_BUF_*; unused may be NULL;
 * MFX_BUF_PP is the p' solution). */
mfx_status mfx_exchange_state(mfx_ctx *ctx, int phase, double *const fields[MFX_NBUF], void *stream);

/* Domain-decomposed (z-slab) BiCGSTAB over all ranks of `ctx`: the
 * "domain-decomposed allreduce-dot baseline" of configuration 5 (the MPI
 * strategy of P:87, Fig. 2a) and the basis of a multi-GPU pressure solve
 * (P:85).  Rank r owns global planes [k0, k1) of mfx_dist_slab(); its
 * A_slab / x_slab arrays hold only those planes (nx*ny*(k1-k0) each, same
 * storage conventions as a global system).  Per iteration one halo plane is
 * exchanged per stencil apply and the double-double dot partials of all ranks
 * are all-gathered and folded in rank order, so every rank takes identical
 * decisions and the iterates equal the single-GPU mfx_bicgstab_solve bitwise.
 * Requires nz >= number of ranks.  Synchronises `stream` once per chunk. */
mfx_status mfx_dist_solve(mfx_ctx *ctx, int kind, const mfx_grid *grid, const mfx_eqsys *A_slab, double *x_slab,
                          double tol, int maxit, mfx_solve_info *info, void *stream);
void mfx_dist_slab(int nz, int rank, int nranks, int *k0, int *k1);

/* a-9: one SIMPLE outer iteration on this rank's share of the equations.
 * state: in snapshot m, out m+1 (u, v, w, p and owned/broadcast phi on every
 * rank).  out (host) receives the residual record (identical on all ranks).
 * Synchronises `stream` once at the end (residual record to host). */
mfx_status mfx_simple_iter(mfx_ctx *ctx, mfx_state *state, mfx_resid *out, void *stream);

/* Particle -> fluid coupling inside the SIMPLE loop (NEXT-2).
 * mode MFX_PIC_IMPLICIT: the drag fields of mfx_state (beta, sbeta_*) are
 * recomputed by mfx_pic_drag from the current snapshot (eps, u, v, w) at the
 * head of every mfx_simple_iter; MFX_PIC_EXPLICIT: only at the next
 * mfx_simple_iter (call again at the start of each time step: "calculated
 * before the first SIMPLE iteration and not updated during subsequent SIMPLE
 * iterations"); MFX_PIC_OFF: never.  The PIC device is rank 0 ("PICdev
 * is always on GPU 1"): only rank 0 needs `parcels` (device arrays, kept by
 * pointer until the next call; other ranks pass NULL) and, for nranks > 1, it
 * broadcasts the four drag fields (exchange phase 3) before the momentum
 * assembly.  The context keeps a cell-ordered copy of the parcels, made by
 * mfx_pic_sort during this call (synchronises the device), so call it again
 * whenever the parcels move. */
enum { MFX_PIC_OFF = 0, MFX_PIC_EXPLICIT = 1, MFX_PIC_IMPLICIT = 2 };
mfx_status mfx_ctx_set_pic(mfx_ctx *ctx, const mfx_parcels *parcels, const mfx_pic_params *pic, int mode);

/* Time loop (NEXT-3; "initial time step was set
 * to 1 ms and varied depending on the convergence of SIMPLE iterations",
 * PAPER.md:165).  mfx_adapt_dt (host, pure): converged within
 * grow_threshold outer iterations -> dt = min(dt*grow, dt_max); converged
 * later -> unchanged; not converged and dt > dt_min -> returns *accept = 0
 * with dt = max(dt*shrink, dt_min); not converged at dt_min -> accepted.
 * mfx_time_step: one accepted time step on this rank's context: params.dt is
 * set to tc->dt, up to max_outer mfx_simple_iter calls until the residual
 * record converges, a rejected attempt restores u, v, w, p, phi to the step's
 * start (device copies) and retries; on acceptance time += dt_used, steps++,
 * and u_old, v_old, w_old, eps_old, phi_old <- u, v, w, eps, phi.  Every rank
 * takes identical decisions (the residual record is exchanged).  Returns
 * MFX_OK (converged) or MFX_NOT_CONVERGED (accepted at dt_min). */
typedef struct {
    double dt, dt_min, dt_max, grow, shrink;
    int grow_threshold, max_outer;
    double time;            /* in/out: simulated time */
    int steps, rejected;    /* in/out: accepted steps, rejected attempts */
} mfx_time_ctrl;
mfx_status mfx_adapt_dt(mfx_time_ctrl *tc, int outer_iters, int converged, int *accept);
mfx_status mfx_time_step(mfx_ctx *ctx, mfx_state *state, mfx_time_ctrl *tc, mfx_resid *last, int *outer_iters,
                         void *stream);

/* Device pointers to the context's internal buffers from the last
 * mfx_simple_iter (NULL where this rank does not hold them): which =
 * 0..2 u*, v*, w* (momentum predictors), 3..5 d_x, d_y, d_z, 6 p' solution. */
double *mfx_ctx_buffer(mfx_ctx *ctx, int which);

/* Per-phase device times of the last mfx_simple_iter on this rank (ms):
 * [0] momentum+scalars (including a PIC drag refresh and its broadcast),
 * [1] GATHER, [2] p' assemble+solve, [3] correction, [4] BCAST, [5] total. */
mfx_status mfx_ctx_phase_times(const mfx_ctx *ctx, double ms[6]);

/* ---------------------------------------------------------------- instrumentation */
/* Kernel timing with CUDA events recorded on the launching stream around
 * every hot kernel launch (off by default).  ids: 0 spmv/setup, 1 K1 (momentum/
 * scalar), 2 K2 (momentum/scalar), 3 K3, 4 momentum assembly, 5 correct, 6 K1 (p'), 7 K2 (p'),
 * 8 p' assembly, 9 scalar assembly, 10 PIC eps deposit, 11 PIC drag deposit (the single-cluster
 * solve is timed under id 0).  mfx_prof_read synchronises the device and
 * returns, per id, launches and total milliseconds since mfx_prof_reset. */
void mfx_prof_enable(int on);
void mfx_prof_reset(void);
mfx_status mfx_prof_read(int counts[16], double ms[16]);
/* Runtime options (process-wide).  "solver_path": 0 = auto (the
 * single-cluster kernel when the system fits one cluster's shared memory;
 * else, for a p' system with even nx whose working set is <= 112 MiB (L2-
 * resident, MFX_PERSIST_MB overrides), the persistent row-warp solver (path
 * 5); else the TMA z-marching kernels; the grid-synchronous kernel is chosen
 * automatically only when MFX_GRID_SOLVER_MB sets an L2 budget -- off by
 * default, measured slower at configuration 3), 1 = TMA z-marching kernels,
 * 2 = single-cluster persistent kernel, 3 = v1 grid-stride reference kernels,
 * 4 = grid-synchronous persistent kernel (one cooperative launch per solve),
 * 5 = persistent row-warp TMA solver (p' only, even nx: the whole iteration
 * loop in one cooperative launch; other systems take path 1).
 * "graphs": 1/0 enables CUDA-graph replay of the iteration loop.  "pdl": 1/0
 * enables programmatic dependent launch between the BiCGSTAB kernels.
 * "asm_tma": 1/0 selects the TMA z-marching momentum assembly (default) or
 * the grid-stride kernel (both give identical bits).  "cluster_size": 16 or 8
 * CTAs for the single-cluster solver (default 16, the non-portable maximum,
 * when the device can place such a cluster; MFX_CLUSTER=8 forces 8); the
 * systems that fit it follow from the size (mfx_get_option reports the one in
 * use).  Every path gives the same bits.  Returns MFX_ERR_ARG for an unknown
 * key. */
mfx_status mfx_set_option(const char *key, int value);
int mfx_get_option(const char *key);

/* Number of libmfx kernel launches issued since process start. */
long long mfx_launch_count(void);

/* CUDA-graph cache of the BiCGSTAB iteration loop.  A graph is
 * keyed on every array pointer it bakes in plus nx, ny, nz, the p' flag, the
 * PDL option and the device, so a replay always matches the launches it
 * replaces.  mfx_ctx_destroy evicts the graphs of its workspaces; callers that
 * free their own workspaces may call mfx_graph_cache_clear (releases every
 * cached graph; stream-ordered, in-flight replays complete).  The cache holds
 * at most 64 graphs (least recently used out first). */
void mfx_graph_cache_clear(void);
size_t mfx_graph_cache_size(void);

#ifdef __cplusplus
}
#endif
#endif /* MFX_H */
