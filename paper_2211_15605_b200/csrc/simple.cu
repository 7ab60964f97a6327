// simple.cu -- a-8 state exchange and a-9 the equation-decomposed SIMPLE
// outer iteration (§2.2.2: Udev/Vdev/Wdev/Pdev, P:85, P:95;
// "infrequent movement of entire field variables").
//
// Each equation is owned by one rank (assignment string); its assembly,
// every BiCGSTAB dot product and its convergence test stay on that GPU.  The
// only inter-GPU traffic per outer iteration is one NCCL group of
// point-to-point sends into the p' owner (GATHER: u*, d per component) and one
// group of broadcasts out of it (BCAST: corrected u, v, w, p; scalar owners
// broadcast phi).  Payloads are copied, never reduced, so any assignment gives
// bitwise the same state as "111[1]".
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace mfx {

void graph_cache_evict(const void *ws);
bool grid_valid(const mfx_grid *g, bool scalar);
mfx_status assemble_eq(int kind, int sid, const mfx_grid *grid, const mfx_params *pr, const mfx_state *st,
                       const double *const star[6], mfx_eqsys *out, double *resid2, void *ws, size_t wsb,
                       cudaStream_t s);
mfx_status bicgstab_solve(int kind, const mfx_grid *grid, const mfx_eqsys *A, double *x, double tol, int maxit,
                          void *ws, size_t wsb, mfx_solve_info *info, cudaStream_t s);
mfx_status correct(const mfx_grid *grid, const mfx_params *pr, const double *const star[6], const double *pp,
                   const double *p, double *u, double *v, double *w, double *pnew, cudaStream_t s);

// ------------------------------------------------------------------ assignment
mfx_status parse_assignment(const char *text, int nranks, mfx_assignment *out)
{
    MFX_ARG_CHECK(text && out, "NULL assignment/out");
    MFX_ARG_CHECK(nranks >= 1 && nranks <= 64, "nranks %d out of range", nranks);
    mfx_assignment a;
    for (int q = 0; q < 8; q++) a.owner[q] = -1;
    a.n_scalars = 0;
    a.n_ranks_used = 0;
    a.n_p = 1;
    const char *c = text;
    auto digit = [&](int &id) -> bool {
        if (*c < '1' || *c > '9') return false;
        id = *c - '0';
        c++;
        return true;
    };
    int id;
    for (int q = 0; q < 3; q++) {
        MFX_ARG_CHECK(digit(id), "assignment '%s': expected a digit 1-9 for %c", text, "UVW"[q]);
        a.owner[q] = id - 1;
    }
    MFX_ARG_CHECK(*c == '[', "assignment '%s': expected '['", text);
    c++;
    int np = 0;
    for (int q = 0; q < 9; q++) a.p_rank[q] = -1;
    while (*c && *c != ']') {
        MFX_ARG_CHECK(np < 9, "assignment '%s': P list longer than 9", text);
        MFX_ARG_CHECK(digit(id), "assignment '%s': bad P list", text);
        for (int q = 0; q < np; q++)
            MFX_ARG_CHECK(a.p_rank[q] != id - 1, "assignment '%s': device %d twice in the P list", text, id);
        if (np == 0) a.owner[3] = id - 1;
        a.p_rank[np++] = id - 1;
    }
    MFX_ARG_CHECK(*c == ']' && np >= 1, "assignment '%s': expected non-empty [P] list", text);
    for (int q = 0; q < np; q++)
        MFX_ARG_CHECK(a.p_rank[q] < nranks, "assignment '%s': device id %d exceeds %d ranks (S:448)", text,
                      a.p_rank[q] + 1, nranks);
    a.n_p = np;
    c++;
    while (*c) {
        MFX_ARG_CHECK(a.n_scalars < 4, "assignment '%s': at most 4 scalar equations", text);
        MFX_ARG_CHECK(digit(id), "assignment '%s': bad scalar owner", text);
        a.owner[4 + a.n_scalars++] = id - 1;
    }
    for (int q = 0; q < 8; q++) {
        if (a.owner[q] < 0) continue;
        MFX_ARG_CHECK(a.owner[q] < nranks, "assignment '%s': device id %d exceeds %d ranks (S:448)", text,
                      a.owner[q] + 1, nranks);
        if (a.owner[q] + 1 > a.n_ranks_used) a.n_ranks_used = a.owner[q] + 1;
    }
    for (int q = 0; q < a.n_p; q++)
        if (a.p_rank[q] + 1 > a.n_ranks_used) a.n_ranks_used = a.p_rank[q] + 1;
    *out = a;
    return MFX_OK;
}

// ------------------------------------------------------------------ exchange plan
// GATHER: momentum owners -> p' owner (u*, d, meta slot); BCAST: p' owner ->
// all (u, v, w, p, meta slots 0-3), scalar owner -> all (phi, its meta slot).
void dist_slab(int nz, int rank, int nranks, int *k0, int *k1);
mfx_status dist_solve(mfx_ctx *ctx, int kind, const mfx_grid *grid, const mfx_eqsys *A, double *x, double tol,
                      int maxit, mfx_solve_info *info, cudaStream_t s);

mfx_status exchange_plan(const mfx_assignment *a, int rank, int phase, mfx_xfer *ops, int max_ops, int *n_ops,
                         int nz)
{
    MFX_ARG_CHECK(a && n_ops && (ops || max_ops == 0), "NULL argument");
    MFX_ARG_CHECK(phase != 2 || a->n_p == 1 || nz >= a->n_p, "PSLAB plan needs nz >= number of p' ranks");
    MFX_ARG_CHECK(phase >= 0 && phase <= 3, "phase must be 0 (GATHER), 1 (BCAST), 2 (PSLAB) or 3 (PIC)");
    std::vector<mfx_xfer> v;
    const int P = a->owner[3];
    const bool multi_p = a->n_p > 1;   // the P-list ranks solve p' together
    if (phase == 0) {
        for (int c = 0; c < 3; c++) {
            const int o = a->owner[c];
            for (int dst = 0; dst < (multi_p ? a->n_p : 1); dst++) {
                const int pr = multi_p ? a->p_rank[dst] : P;
                if (pr == o) continue;
                if (rank == o) {
                    v.push_back({MFX_OP_SEND, pr, MFX_BUF_U + c, 0, 0, 0, 0});
                    v.push_back({MFX_OP_SEND, pr, MFX_BUF_DX + c, 0, 0, 0, 0});
                    v.push_back({MFX_OP_SEND, pr, MFX_BUF_META, c, 1, 0, 0});
                } else if (rank == pr) {
                    v.push_back({MFX_OP_RECV, o, MFX_BUF_U + c, 0, 0, 0, 0});
                    v.push_back({MFX_OP_RECV, o, MFX_BUF_DX + c, 0, 0, 0, 0});
                    v.push_back({MFX_OP_RECV, o, MFX_BUF_META, c, 1, 0, 0});
                }
            }
        }
    } else if (phase == 1) {
        v.push_back({MFX_OP_BCAST, P, MFX_BUF_U, 0, 0, 0, 0});
        v.push_back({MFX_OP_BCAST, P, MFX_BUF_V, 0, 0, 0, 0});
        v.push_back({MFX_OP_BCAST, P, MFX_BUF_W, 0, 0, 0, 0});
        v.push_back({MFX_OP_BCAST, P, MFX_BUF_P, 0, 0, 0, 0});
        v.push_back({MFX_OP_BCAST, P, MFX_BUF_META, 0, 4, 0, 0});
        for (int s = 0; s < a->n_scalars; s++) {
            v.push_back({MFX_OP_BCAST, a->owner[4 + s], MFX_BUF_PHI0 + s, 0, 0, 0, 0});
            v.push_back({MFX_OP_BCAST, a->owner[4 + s], MFX_BUF_META, 4 + s, 1, 0, 0});
        }
    } else if (phase == 3) {
        // PIC: the PIC device (rank 0) broadcasts the refreshed drag fields
        for (int b = MFX_BUF_BETA; b <= MFX_BUF_SBW; b++) v.push_back({MFX_OP_BCAST, 0, b, 0, 0, 0, 0});
        v.push_back({MFX_OP_BCAST, 0, MFX_BUF_META, 8, 1, 0, 0});   // the PIC record (error latch)
    } else if (multi_p) {
        // PSLAB: slab i of the domain-decomposed p' solution (on p_rank[i]) -> P0 = p_rank[0]
        for (int i = 1; i < a->n_p; i++) {
            const int q = a->p_rank[i];
            int k0, k1;
            dist_slab(nz, i, a->n_p, &k0, &k1);
            if (rank == q) v.push_back({MFX_OP_SEND, P, MFX_BUF_PP, 0, 0, k0, k1});
            else if (rank == P) v.push_back({MFX_OP_RECV, q, MFX_BUF_PP, 0, 0, k0, k1});
        }
    }
    *n_ops = (int)v.size();
    MFX_ARG_CHECK((int)v.size() <= max_ops || !ops, "plan needs %d ops, buffer holds %d", (int)v.size(), max_ops);
    if (ops)
        for (size_t q = 0; q < v.size(); q++) ops[q] = v[q];
    return MFX_OK;
}

// ------------------------------------------------------------------ NCCL (dlopen)
namespace {
struct Nccl {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t *, ncclConfig_t *) = nullptr;
    bool load()
    {
        if (h) return true;
        const char *env = getenv("MFX_NCCL_PATH");
        if (env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // torch's, if already loaded
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) { set_error("cannot dlopen libnccl.so.2: %s", dlerror()); return false; }
#define SYM(name) name = (decltype(name))dlsym(h, "nccl" #name); if (!name) { set_error("nccl%s missing", #name); return false; }
        SYM(GetUniqueId) SYM(CommInitRank) SYM(CommDestroy) SYM(GroupStart) SYM(GroupEnd) SYM(Send) SYM(Recv)
        SYM(Broadcast) SYM(AllGather) SYM(GetErrorString) SYM(CommSplit)
#undef SYM
        return true;
    }
};
Nccl g_nccl;

#define MFX_NCCL_TRY(expr)                                                                     \
    do {                                                                                       \
        ncclResult_t r_ = (expr);                                                              \
        if (r_ != ncclSuccess) {                                                               \
            set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, g_nccl.GetErrorString(r_));    \
            return MFX_ERR_NCCL;                                                               \
        }                                                                                      \
    } while (0)

size_t round256(size_t b) { return (b + 255) & ~(size_t)255; }
constexpr size_t kMetaBytes = 9 * 16 * sizeof(double);

// Residual record of one equation (16 doubles, exchanged with the state so
// every rank sees the same record): [0] residual numerator, [1] denominator,
// [2] iterations, [3] solve status, [4] restarts, [5] recursive rel. residual,
// [6] present, [7] true rel. residual at exit, [8] device error (0, or
// MFX_ERR_NONFINITE / MFX_ERR_ZERO_DIAG / MFX_ERR_ARG for a bad parcel),
// [9] first offending cell (or parcel) index.  The error latch of the
// equation's workspace is read here on the device and cleared, so the status
// every rank returns derives from the exchanged record (identical decisions).
__device__ void meta_error(WsHeader *h, double *slot)
{
    const unsigned long long nf = h->bad_nonfinite, zd = h->bad_zerodiag;
    slot[8] = 0.0;
    slot[9] = 0.0;
    if (nf != ~0ull) { slot[8] = (double)MFX_ERR_NONFINITE; slot[9] = (double)nf; }
    else if (zd != ~0ull) { slot[8] = (double)MFX_ERR_ZERO_DIAG; slot[9] = (double)zd; }
    h->bad_nonfinite = ~0ull;
    h->bad_zerodiag = ~0ull;
}

__global__ void k_meta_vals(const double *resid2, double *slot, int iters, int status, int restarts, double rel,
                            WsHeader *h)
{
    if (threadIdx.x != 0) return;
    slot[0] = resid2[0];
    slot[1] = resid2[1];
    slot[2] = (double)iters;
    slot[3] = (double)status;
    slot[4] = (double)restarts;
    slot[5] = rel;
    slot[6] = 1.0;
    slot[7] = h->true_rel;
    meta_error(h, slot);
}

__global__ void k_meta(WsHeader *h, const double *resid2, double *slot, int solved)
{
    if (threadIdx.x != 0) return;
    const SolverScalars &S = h->sc;
    slot[0] = resid2 ? resid2[0] : 0.0;
    slot[1] = resid2 ? resid2[1] : 0.0;
    slot[2] = solved ? (double)S.it : 0.0;
    slot[3] = solved ? (double)S.status : 0.0;
    slot[4] = solved ? (double)S.restarts : 0.0;
    slot[5] = solved && S.bn != 0.0 ? S.rn / S.bn : 0.0;
    slot[6] = 1.0;   // present
    slot[7] = solved ? h->true_rel : 0.0;
    meta_error(h, slot);
}

// PIC record (meta slot 8, broadcast with the drag fields): a parcel latched
// outside the domain by the refresh on the PIC device
__global__ void k_meta_pic(WsHeader *h, double *slot)
{
    if (threadIdx.x != 0) return;
    const unsigned long long bp = h->bad_parcel;
    slot[6] = 1.0;
    slot[8] = bp != ~0ull ? (double)MFX_ERR_ARG : 0.0;
    slot[9] = bp != ~0ull ? (double)bp : 0.0;
    h->bad_parcel = ~0ull;
}
}  // namespace

mfx_status nccl_unique_id(unsigned char out[128])
{
    MFX_ARG_CHECK(out, "NULL out");
    if (!g_nccl.load()) return MFX_ERR_NCCL;
    ncclUniqueId id;
    MFX_NCCL_TRY(g_nccl.GetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    memcpy(out, &id, 128);
    return MFX_OK;
}

}  // namespace mfx

// ------------------------------------------------------------------ local transport
// In-process transport: ranks are host threads of one process (same or
// different GPUs), each with its own stream.  The exchange plan is executed as
// pull copies: every rank publishes its buffer pointers and records a "ready"
// event, a host barrier orders publication before use, receivers/non-roots
// wait on the producer's event and copy peer-to-peer, and a second barrier +
// "done" events keep producers from overwriting a buffer still being read.
struct mfx_local_group {
    int nranks;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long gen = 0;
    double *fields[64][MFX_NBUF];
    const void *dptr[64];     // distributed solver: published slab / partials pointer
    long long dlen[64];       // ... and its length (planes or values)
    cudaEvent_t ready[64];
    cudaEvent_t done[64];
    // sub-groups for a multi-GPU p' solve over a subset of the ranks (the P
    // list, in its order), created once by the first rank that asks
    std::vector<std::pair<std::vector<int>, mfx_local_group *>> subs;
    void barrier()
    {
        std::unique_lock<std::mutex> lk(mu);
        const unsigned long g = gen;
        if (++arrived == nranks) {
            arrived = 0;
            gen++;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

// ------------------------------------------------------------------ context
struct mfx_ctx {
    int rank, nranks;
    mfx_assignment asg;
    mfx_grid grid;
    mfx_params params;
    long long N;
    std::vector<void *> allocs;
    mfx_eqsys sys[8];        // per equation (owned ones allocated)
    void *ws[8];
    size_t ws_bytes;
    double *resid2;          // device [8][2]
    double *star[3], *dv[3]; // u*, v*, w*, d_x, d_y, d_z (owned or received)
    double *pp;              // p' solution
    double *phinew[4];
    double *meta;            // device [9][16]: 8 equation records + the PIC record
    double *meta_host;       // pinned [9][16]
    ncclComm_t comm;
    mfx_local_group *group;  // non-NULL: in-process transport instead of NCCL
    int prank;               // index of this rank in the P list (-1: not a p' rank)
    ncclComm_t pcomm;        // the P-list ranks (multi-GPU p'); == comm when the list is every rank in order
    mfx_local_group *pgroup; // ... in-process transport
    int dist_sub;            // 1 while the distributed solver runs over the P list
    void *dist_scratch;      // distributed-solver workspace (allocated on first use)
    size_t dist_bytes;
    cudaEvent_t ev[6];
    double phase_ms[6];
    // GATHER / BCAST run on a dedicated communication stream, ordered against
    // the compute stream by events (fork/join); xt[] time them on that stream
    cudaStream_t cs;
    cudaEvent_t xfork, xjoin, xt[4];
    double *ts_save[8];       // time loop: state at the start of the step (allocated on first use)
    // particle -> fluid coupling: parcels live on the PIC device (rank 0)
    int pic_mode, pic_pending;
    mfx_parcels pic_pc;            // the caller's parcels, or the context's cell-sorted copy
    mfx_pic_params pic_pp;
    void *pic_ws;
    double *pic_sorted[7];         // binned copy (mfx_pic_sort), capacity pic_cap
    unsigned int *pic_orig;        // original index per binned parcel
    unsigned int *pic_start;       // bin starts (N + 1)
    double *pic_vals;              // 7 x pic_cap: per-parcel deposit values + lattice coordinates
    long long pic_cap;
    void *pic_scratch;
    size_t pic_scratch_bytes;
};

namespace mfx {

static mfx_status ctx_alloc(mfx_ctx *c, void **p, size_t bytes)
{
    MFX_CUDA_TRY(cudaMalloc(p, bytes));
    c->allocs.push_back(*p);
    return MFX_OK;
}

mfx_status ctx_create(const char *assignment, int rank, int nranks, const unsigned char *uid, const mfx_grid *grid,
                      const mfx_params *params, mfx_ctx **out, mfx_local_group *group = nullptr)
{
    MFX_ARG_CHECK(out && params, "NULL out/params");
    *out = nullptr;
    if (!grid_valid(grid, false)) return MFX_ERR_ARG;
    MFX_ARG_CHECK(rank >= 0 && rank < nranks, "rank %d of %d", rank, nranks);
    mfx_assignment a;
    mfx_status st = parse_assignment(assignment, nranks, &a);
    if (st != MFX_OK) return st;
    MFX_ARG_CHECK(nranks == 1 || uid || group, "uid (NCCL) or a local group required for nranks > 1");
    MFX_ARG_CHECK(!group || group->nranks == nranks, "local group has %d ranks, expected %d",
                  group ? group->nranks : 0, nranks);
    MFX_ARG_CHECK(a.n_p == 1 || grid->nz >= a.n_p, "multi-GPU p' needs nz >= number of p' ranks");
    mfx_ctx *c = new mfx_ctx();
    c->prank = -1;
    for (int q = 0; q < a.n_p; q++)
        if (a.p_rank[q] == rank) c->prank = q;
    c->rank = rank; c->nranks = nranks; c->asg = a; c->grid = *grid; c->params = *params;
    c->N = (long long)grid->nx * grid->ny * grid->nz;
    c->comm = nullptr;
    c->group = group;
    c->dist_scratch = nullptr;
    c->dist_bytes = 0;
    const size_t vb = round256(sizeof(double) * c->N);
    c->ws_bytes = ws_total_bytes(c->N);
    auto fail = [&](mfx_status s) { mfx_ctx_destroy(c); return s; };
    for (int q = 0; q < 8; q++) { memset(&c->sys[q], 0, sizeof(mfx_eqsys)); c->ws[q] = nullptr; }
    const int P = a.owner[3];
    const bool multi_p = a.n_p > 1 && c->prank >= 0;   // this rank solves a slab of p'
    auto holds = [&](int q) { return a.owner[q] == rank || (q == 3 && multi_p); };
    for (int q = 0; q < 8; q++) {
        if (!holds(q)) continue;
        const int narr = q == 3 ? 5 : 9;
        void *blk;
        if ((st = ctx_alloc(c, &blk, vb * narr)) != MFX_OK) return fail(st);
        double *b0 = (double *)blk;
        auto arr = [&](int k) { return (double *)((char *)b0 + vb * k); };
        mfx_eqsys &e = c->sys[q];
        e.aP = arr(0); e.aE = arr(1); e.aN = arr(2); e.aT = arr(3); e.b = arr(4);
        if (q != 3) { e.aW = arr(5); e.aS = arr(6); e.aB = arr(7); e.d = arr(8); }
        if ((st = ctx_alloc(c, &c->ws[q], c->ws_bytes)) != MFX_OK) return fail(st);
        if (cudaMemset(c->ws[q], 0, ws_header_bytes()) != cudaSuccess) return fail(MFX_ERR_CUDA);
        WsView W;
        ws_view(c->ws[q], c->ws_bytes, c->N, false, W);
        const unsigned long long none = ~0ull;
        cudaMemcpy(&W.hdr->bad_nonfinite, &none, 8, cudaMemcpyHostToDevice);
        cudaMemcpy(&W.hdr->bad_zerodiag, &none, 8, cudaMemcpyHostToDevice);
        cudaMemcpy(&W.hdr->bad_parcel, &none, 8, cudaMemcpyHostToDevice);
    }
    // starred velocities and d: on the owner of each component and on the p' owner
    for (int q = 0; q < 3; q++) {
        c->star[q] = c->dv[q] = nullptr;
        if (a.owner[q] == rank || P == rank || multi_p) {
            void *blk;
            if ((st = ctx_alloc(c, &blk, vb)) != MFX_OK) return fail(st);
            c->star[q] = (double *)blk;
            if (a.owner[q] == rank) c->dv[q] = c->sys[q].d;
            else {
                if ((st = ctx_alloc(c, &blk, vb)) != MFX_OK) return fail(st);
                c->dv[q] = (double *)blk;
            }
        }
    }
    c->pp = nullptr;
    if (P == rank || multi_p) {
        void *blk;
        if ((st = ctx_alloc(c, &blk, vb)) != MFX_OK) return fail(st);
        c->pp = (double *)blk;
    }
    for (int s = 0; s < 4; s++) {
        c->phinew[s] = nullptr;
        if (s < a.n_scalars && a.owner[4 + s] == rank) {
            void *blk;
            if ((st = ctx_alloc(c, &blk, vb)) != MFX_OK) return fail(st);
            c->phinew[s] = (double *)blk;
        }
    }
    {
        void *blk;
        if ((st = ctx_alloc(c, &blk, 256 + kMetaBytes)) != MFX_OK) return fail(st);
        c->resid2 = (double *)blk;
        c->meta = (double *)((char *)blk + 256);
        if (cudaMemset(blk, 0, 256 + kMetaBytes) != cudaSuccess) return fail(MFX_ERR_CUDA);
    }
    if (cudaMallocHost(&c->meta_host, kMetaBytes) != cudaSuccess) {
        c->meta_host = nullptr;
        return fail(MFX_ERR_CUDA);
    }
    for (int q = 0; q < 6; q++) {
        if (cudaEventCreate(&c->ev[q]) != cudaSuccess) return fail(MFX_ERR_CUDA);
        c->phase_ms[q] = 0.0;
    }
    if (cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->xfork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->xjoin, cudaEventDisableTiming) != cudaSuccess)
        return fail(MFX_ERR_CUDA);
    for (int q = 0; q < 4; q++)
        if (cudaEventCreate(&c->xt[q]) != cudaSuccess) return fail(MFX_ERR_CUDA);
    if (nranks > 1 && !group) {
        if (!g_nccl.load()) return fail(MFX_ERR_NCCL);
        ncclUniqueId id;
        memcpy(&id, uid, 128);
        ncclResult_t r = g_nccl.CommInitRank(&c->comm, nranks, id, rank);
        if (r != ncclSuccess) {
            set_error("ncclCommInitRank: %s", g_nccl.GetErrorString(r));
            c->comm = nullptr;
            return fail(MFX_ERR_NCCL);
        }
    }
    // the P-list communicator of a multi-GPU p' solve (slab i on p_rank[i])
    if (a.n_p > 1) {
        bool every_in_order = a.n_p == nranks;
        for (int q = 0; q < a.n_p; q++) every_in_order = every_in_order && a.p_rank[q] == q;
        if (group) {
            std::vector<int> key(a.p_rank, a.p_rank + a.n_p);
            std::unique_lock<std::mutex> lk(group->mu);
            for (auto &e : group->subs)
                if (e.first == key) c->pgroup = e.second;
            if (!c->pgroup) {
                mfx_local_group *sg = nullptr;
                if (mfx_local_group_create(a.n_p, &sg) != MFX_OK) { lk.unlock(); return fail(MFX_ERR_CUDA); }
                group->subs.push_back({key, sg});
                c->pgroup = sg;
            }
        } else if (nranks > 1) {
            if (every_in_order) c->pcomm = c->comm;
            else {
                ncclResult_t r = g_nccl.CommSplit(c->comm, c->prank >= 0 ? 0 : -1 /* NCCL_SPLIT_NOCOLOR */,
                                                  c->prank >= 0 ? c->prank : 0, &c->pcomm, nullptr);
                if (r != ncclSuccess) {
                    set_error("ncclCommSplit: %s", g_nccl.GetErrorString(r));
                    c->pcomm = nullptr;
                    return fail(MFX_ERR_NCCL);
                }
            }
        }
    }
    *out = c;
    return MFX_OK;
}

mfx_status exchange_state(mfx_ctx *c, int phase, double *const fields[MFX_NBUF], cudaStream_t s)
{
    MFX_ARG_CHECK(c && fields, "NULL ctx/fields");
    if (c->nranks == 1) return MFX_OK;
    mfx_xfer ops[64];
    int n = 0;
    mfx_status st = exchange_plan(&c->asg, c->rank, phase, ops, 64, &n, c->grid.nz);
    if (st != MFX_OK) return st;
    const long long plane = (long long)c->grid.nx * c->grid.ny;
    // element offset and count of op o in its buffer
    size_t packed_count[64] = {0};   // > 0: op q carries the whole [u|v|w|p] block
    auto span = [&](int q, size_t &off, size_t &count) {
        const mfx_xfer &o = ops[q];
        if (packed_count[q]) { off = 0; count = packed_count[q]; }
        else if (o.buf == MFX_BUF_META) { off = 16 * (size_t)o.slot; count = 16 * (size_t)o.nslots; }
        else if (o.k1 > o.k0) { off = (size_t)(o.k0 * plane); count = (size_t)((o.k1 - o.k0) * plane); }
        else { off = 0; count = (size_t)c->N; }
    };
    // packed BCAST (mfx_params.packed_state, identical on every rank): the four
    // broadcasts of u, v, w, p from the p' owner become one of 4N doubles
    bool skip[64] = {false};
    mfx_status local_err = MFX_OK;
    if (phase == 1 && c->params.packed_state) {
        auto contiguous = [&](double *const *f) {
            return f[MFX_BUF_U] && f[MFX_BUF_V] == f[MFX_BUF_U] + c->N && f[MFX_BUF_W] == f[MFX_BUF_U] + 2 * c->N &&
                   f[MFX_BUF_P] == f[MFX_BUF_U] + 3 * c->N;
        };
        if (!contiguous(fields)) {
            set_error("packed_state: u, v, w, p are not one [u|v|w|p] block on rank %d", c->rank);
            if (!c->group) return MFX_ERR_ARG;
            local_err = MFX_ERR_ARG;   // in-process transport: keep the barriers, fail after them
        }
        for (int q = 0; q < n; q++) {
            if (ops[q].op != MFX_OP_BCAST || ops[q].buf < MFX_BUF_U || ops[q].buf > MFX_BUF_P) continue;
            if (ops[q].buf == MFX_BUF_U) packed_count[q] = 4 * (size_t)c->N;
            else skip[q] = true;
        }
    }
    if (c->group) {
        mfx_local_group &g = *c->group;
        for (int b = 0; b < MFX_NBUF; b++) g.fields[c->rank][b] = fields[b];
        MFX_CUDA_TRY(cudaEventRecord(g.ready[c->rank], s));
        g.barrier();
        // a rank-local argument error must not strand the other ranks in the
        // barriers below: it is reported after them
        for (int q = 0; q < n && local_err == MFX_OK; q++) {
            const mfx_xfer &o = ops[q];
            if (skip[q] || o.op == MFX_OP_SEND || (o.op == MFX_OP_BCAST && o.peer == c->rank)) continue;
            double *dst = fields[o.buf];
            const double *src = g.fields[o.peer][o.buf];
            size_t off, count;
            span(q, off, count);
            if (packed_count[q] && !(g.fields[o.peer][MFX_BUF_V] == src + c->N &&
                                     g.fields[o.peer][MFX_BUF_P] == src + 3 * c->N)) {
                set_error("packed_state: the root's [u|v|w|p] block is not contiguous");
                local_err = MFX_ERR_ARG;
                break;
            }
            if (dst) dst += off;
            if (src) src += off;
            if (!dst || !src) {
                set_error("local exchange: buffer %d missing (rank %d <- %d)", o.buf, c->rank, o.peer);
                local_err = MFX_ERR_ARG;
                break;
            }
            MFX_CUDA_TRY(cudaStreamWaitEvent(s, g.ready[o.peer], 0));
            MFX_CUDA_TRY(cudaMemcpyAsync(dst, src, count * sizeof(double), cudaMemcpyDefault, s));
        }
        MFX_CUDA_TRY(cudaEventRecord(g.done[c->rank], s));
        g.barrier();
        for (int q = 0; q < g.nranks; q++)
            if (q != c->rank) MFX_CUDA_TRY(cudaStreamWaitEvent(s, g.done[q], 0));
        g.barrier();   // every rank has enqueued its waits before any event is re-recorded
        return local_err;
    }
    MFX_NCCL_TRY(g_nccl.GroupStart());
    for (int q = 0; q < n; q++) {
        const mfx_xfer &o = ops[q];
        if (skip[q]) continue;
        double *buf = fields[o.buf];
        size_t off, count;
        span(q, off, count);
        if (buf) buf += off;
        if (!buf) {
            g_nccl.GroupEnd();
            set_error("exchange: buffer %d is NULL on rank %d", o.buf, c->rank);
            return MFX_ERR_ARG;
        }
        if (o.op == MFX_OP_SEND) MFX_NCCL_TRY(g_nccl.Send(buf, count, ncclDouble, o.peer, c->comm, s));
        else if (o.op == MFX_OP_RECV) MFX_NCCL_TRY(g_nccl.Recv(buf, count, ncclDouble, o.peer, c->comm, s));
        else MFX_NCCL_TRY(g_nccl.Broadcast(buf, buf, count, ncclDouble, o.peer, c->comm, s));
    }
    MFX_NCCL_TRY(g_nccl.GroupEnd());
    return MFX_OK;
}

// ------------------------------------------------------------------ distributed-solver transport
// the distributed solver's group: every rank of the context (mfx_dist_solve),
// or the P list while mfx_simple_iter runs a multi-GPU p' solve (dist_sub)
int ctx_rank(const mfx_ctx *c) { return c->dist_sub ? c->prank : c->rank; }
int ctx_nranks(const mfx_ctx *c) { return c->dist_sub ? c->asg.n_p : c->nranks; }
static ncclComm_t ctx_comm(const mfx_ctx *c) { return c->dist_sub ? c->pcomm : c->comm; }
static mfx_local_group *ctx_group(const mfx_ctx *c) { return c->dist_sub ? c->pgroup : c->group; }
// the distributed solver may capture its iterations in a CUDA graph: NCCL (or
// one rank), not the in-process transport, whose phases synchronise host threads
bool ctx_capturable(const mfx_ctx *c)
{
    static const int allowed = [] { const char *e = getenv("MFX_DIST_GRAPH"); return e ? atoi(e) : 1; }();
    return allowed && (ctx_nranks(c) == 1 || !ctx_group(c));
}

void *ctx_dist_scratch(mfx_ctx *c, size_t bytes)
{
    if (c->dist_bytes < bytes) {
        if (c->dist_scratch) cudaFree(c->dist_scratch);
        c->dist_scratch = nullptr;
        c->dist_bytes = 0;
        if (cudaMalloc(&c->dist_scratch, bytes) != cudaSuccess) {
            set_error("cudaMalloc(%zu) for the distributed solver failed", bytes);
            return nullptr;
        }
        c->dist_bytes = bytes;
    }
    return c->dist_scratch;
}

// local transport: publish (ptr, len), barrier, pull, done-events, barrier
template <class Pull>
static mfx_status local_phase(mfx_ctx *c, const void *ptr, long long len, cudaStream_t s, Pull pull)
{
    mfx_local_group &g = *ctx_group(c);
    const int me = ctx_rank(c);
    g.dptr[me] = ptr;
    g.dlen[me] = len;
    MFX_CUDA_TRY(cudaEventRecord(g.ready[me], s));
    g.barrier();
    mfx_status st = pull(g);
    if (st != MFX_OK) return st;
    MFX_CUDA_TRY(cudaEventRecord(g.done[me], s));
    g.barrier();
    for (int q = 0; q < g.nranks; q++)
        if (q != me) MFX_CUDA_TRY(cudaStreamWaitEvent(s, g.done[q], 0));
    g.barrier();
    return MFX_OK;
}

// hb <- last plane of rank-1's slab, ha <- first plane of rank+1's slab
mfx_status ctx_halo_exchange(mfx_ctx *c, const double *slab, int npl, long long plane, double *hb, double *ha,
                             cudaStream_t s)
{
    const int r = ctx_rank(c), R = ctx_nranks(c);
    if (R == 1) return MFX_OK;
    const size_t pb = sizeof(double) * (size_t)plane;
    ncclComm_t comm = ctx_comm(c);
    if (c->group) {
        return local_phase(c, slab, npl, s, [&](mfx_local_group &g) -> mfx_status {
            if (r > 0) {
                MFX_CUDA_TRY(cudaStreamWaitEvent(s, g.ready[r - 1], 0));
                const double *src = (const double *)g.dptr[r - 1] + (g.dlen[r - 1] - 1) * plane;
                MFX_CUDA_TRY(cudaMemcpyAsync(hb, src, pb, cudaMemcpyDefault, s));
            }
            if (r < R - 1) {
                MFX_CUDA_TRY(cudaStreamWaitEvent(s, g.ready[r + 1], 0));
                MFX_CUDA_TRY(cudaMemcpyAsync(ha, g.dptr[r + 1], pb, cudaMemcpyDefault, s));
            }
            return MFX_OK;
        });
    }
    MFX_NCCL_TRY(g_nccl.GroupStart());
    if (r > 0) {
        MFX_NCCL_TRY(g_nccl.Send(slab, (size_t)plane, ncclDouble, r - 1, comm, s));
        MFX_NCCL_TRY(g_nccl.Recv(hb, (size_t)plane, ncclDouble, r - 1, comm, s));
    }
    if (r < R - 1) {
        MFX_NCCL_TRY(g_nccl.Send(slab + (size_t)(npl - 1) * plane, (size_t)plane, ncclDouble, r + 1, comm, s));
        MFX_NCCL_TRY(g_nccl.Recv(ha, (size_t)plane, ncclDouble, r + 1, comm, s));
    }
    MFX_NCCL_TRY(g_nccl.GroupEnd());
    return MFX_OK;
}

// all[q*K .. q*K+K) <- rank q's K double-double partials, for every rank q
mfx_status ctx_allgather_dd(mfx_ctx *c, const dd *mine, int K, dd *all, cudaStream_t s)
{
    const int R = ctx_nranks(c);
    const size_t kb = sizeof(dd) * (size_t)K;
    if (R == 1) {
        MFX_CUDA_TRY(cudaMemcpyAsync(all, mine, kb, cudaMemcpyDeviceToDevice, s));
        return MFX_OK;
    }
    if (c->group) {
        return local_phase(c, mine, K, s, [&](mfx_local_group &g) -> mfx_status {
            for (int q = 0; q < R; q++) {
                if (q != ctx_rank(c)) MFX_CUDA_TRY(cudaStreamWaitEvent(s, g.ready[q], 0));
                MFX_CUDA_TRY(cudaMemcpyAsync(all + (size_t)q * K, g.dptr[q], kb, cudaMemcpyDefault, s));
            }
            return MFX_OK;
        });
    }
    MFX_NCCL_TRY(g_nccl.AllGather(mine, all, 2 * (size_t)K, ncclDouble, ctx_comm(c), s));
    return MFX_OK;
}

// exchange phase on the communication stream: fork from s, time it with
// (t0, t1) on cs, and join back into s at the caller's chosen point
static mfx_status exchange_fork(mfx_ctx *c, int phase, double *const fields[MFX_NBUF], cudaStream_t s,
                                cudaEvent_t t0, cudaEvent_t t1)
{
    if (c->nranks == 1) {
        MFX_CUDA_TRY(cudaEventRecord(t0, s));
        MFX_CUDA_TRY(cudaEventRecord(t1, s));
        return MFX_OK;
    }
    MFX_CUDA_TRY(cudaEventRecord(c->xfork, s));
    MFX_CUDA_TRY(cudaStreamWaitEvent(c->cs, c->xfork, 0));
    MFX_CUDA_TRY(cudaEventRecord(t0, c->cs));
    mfx_status rc = exchange_state(c, phase, fields, c->cs);
    if (rc != MFX_OK) return rc;
    MFX_CUDA_TRY(cudaEventRecord(t1, c->cs));
    return MFX_OK;
}
static mfx_status exchange_join(mfx_ctx *c, cudaStream_t s)
{
    if (c->nranks == 1) return MFX_OK;
    MFX_CUDA_TRY(cudaEventRecord(c->xjoin, c->cs));
    MFX_CUDA_TRY(cudaStreamWaitEvent(s, c->xjoin, 0));
    return MFX_OK;
}

mfx_status simple_iter(mfx_ctx *c, mfx_state *st, mfx_resid *out, cudaStream_t s)
{
    MFX_ARG_CHECK(c && st && out, "NULL argument");
    const mfx_assignment &a = c->asg;
    const mfx_params &pr = c->params;
    const int r = c->rank, P = a.owner[3];
    const size_t vbytes = sizeof(double) * (size_t)c->N;
    mfx_status rc;
    MFX_CUDA_TRY(cudaMemsetAsync(c->meta, 0, kMetaBytes, s));
    MFX_CUDA_TRY(cudaEventRecord(c->ev[0], s));
    // head of the SIMPLE iteration: particle -> fluid drag refresh
    if (c->pic_mode == MFX_PIC_IMPLICIT || (c->pic_mode == MFX_PIC_EXPLICIT && c->pic_pending)) {
        if (r == 0) {
            // deterministic gather deposit on the binned parcels (bitwise the parcel-ordered definition)
            double *outs[4] = {st->beta, st->sbeta_u, st->sbeta_v, st->sbeta_w};
            rc = pic_deposit_binned(1, &c->grid, &pr, &c->pic_pp, &c->pic_pc, c->pic_orig, c->pic_start, st->eps,
                                    st->u, st->v, st->w, outs, nullptr, c->pic_vals, c->pic_ws, ws_header_bytes(), s);
            if (rc != MFX_OK) return rc;
            k_meta_pic<<<1, 32, 0, s>>>((WsHeader *)c->pic_ws, c->meta + 16 * 8);
        }
        double *D[MFX_NBUF] = {0};
        D[MFX_BUF_BETA] = st->beta; D[MFX_BUF_SBU] = st->sbeta_u;
        D[MFX_BUF_SBV] = st->sbeta_v; D[MFX_BUF_SBW] = st->sbeta_w;
        D[MFX_BUF_META] = c->meta;   // slot 8: the PIC record (error latch of the refresh)
        if ((rc = exchange_fork(c, 3, D, s, c->xt[0], c->xt[1])) != MFX_OK) return rc;
        if ((rc = exchange_join(c, s)) != MFX_OK) return rc;
        c->pic_pending = 0;
    }
    // momentum predictors (snapshot) on their owners
    for (int q = 0; q < 3; q++) {
        if (a.owner[q] != r) continue;
        if ((rc = assemble_eq(q, 0, &c->grid, &pr, st, nullptr, &c->sys[q], c->resid2 + 2 * q, c->ws[q],
                              c->ws_bytes, s)) != MFX_OK) return rc;
        const double *snap = q == 0 ? st->u : (q == 1 ? st->v : st->w);
        MFX_CUDA_TRY(cudaMemcpyAsync(c->star[q], snap, vbytes, cudaMemcpyDeviceToDevice, s));
        mfx_solve_info info;
        rc = bicgstab_solve(q, &c->grid, &c->sys[q], c->star[q], pr.lin_tol_mom, pr.lin_maxit_mom, c->ws[q],
                            c->ws_bytes, &info, s);
        if (rc < 0 && rc != MFX_ERR_BREAKDOWN) return rc;
        k_meta<<<1, 32, 0, s>>>((WsHeader *)c->ws[q], c->resid2 + 2 * q, c->meta + 16 * q, 1);
    }
    // GATHER (u*, d -> the p' owner) on the communication stream, overlapping
    // the scalar equations below (they read only the snapshot)
    double *F[MFX_NBUF] = {0};
    F[MFX_BUF_U] = c->star[0]; F[MFX_BUF_V] = c->star[1]; F[MFX_BUF_W] = c->star[2];
    F[MFX_BUF_DX] = c->dv[0]; F[MFX_BUF_DY] = c->dv[1]; F[MFX_BUF_DZ] = c->dv[2];
    F[MFX_BUF_META] = c->meta;
    if ((rc = exchange_fork(c, 0, F, s, c->xt[0], c->xt[1])) != MFX_OK) return rc;
    // scalars (same snapshot, Q22)
    for (int sc = 0; sc < a.n_scalars; sc++) {
        const int q = 4 + sc;
        if (a.owner[q] != r) continue;
        if ((rc = assemble_eq(MFX_EQ_SCALAR, sc, &c->grid, &pr, st, nullptr, &c->sys[q], c->resid2 + 2 * q,
                              c->ws[q], c->ws_bytes, s)) != MFX_OK) return rc;
        MFX_CUDA_TRY(cudaMemcpyAsync(c->phinew[sc], st->phi[sc], vbytes, cudaMemcpyDeviceToDevice, s));
        mfx_solve_info info;
        rc = bicgstab_solve(MFX_EQ_SCALAR, &c->grid, &c->sys[q], c->phinew[sc], pr.lin_tol_phi, pr.lin_maxit_phi,
                            c->ws[q], c->ws_bytes, &info, s);
        if (rc < 0 && rc != MFX_ERR_BREAKDOWN) return rc;
        k_meta<<<1, 32, 0, s>>>((WsHeader *)c->ws[q], c->resid2 + 2 * q, c->meta + 16 * q, 1);
    }
    MFX_CUDA_TRY(cudaEventRecord(c->ev[1], s));
    if ((rc = exchange_join(c, s)) != MFX_OK) return rc;
    MFX_CUDA_TRY(cudaEventRecord(c->ev[2], s));
    if (a.n_p > 1) {
        // multi-GPU pressure correction: every rank of the P list
        // assembles p' (cheap, from the gathered u*, d), solves its z-slab with
        // the domain-decomposed BiCGSTAB over the P list, and the slabs are
        // gathered to P0 = p_rank[0]
        const double *star6[6] = {c->star[0], c->star[1], c->star[2], c->dv[0], c->dv[1], c->dv[2]};
        if (c->prank >= 0) {
            if ((rc = assemble_eq(MFX_EQ_PP, 0, &c->grid, &pr, st, star6, &c->sys[3], c->resid2 + 6, c->ws[3],
                                  c->ws_bytes, s)) != MFX_OK) return rc;
            MFX_CUDA_TRY(cudaMemsetAsync(c->pp, 0, vbytes, s));
            int k0, k1;
            dist_slab(c->grid.nz, c->prank, a.n_p, &k0, &k1);
            const size_t off = (size_t)k0 * c->grid.nx * c->grid.ny;
            mfx_eqsys sl;
            memset(&sl, 0, sizeof(sl));
            sl.aP = c->sys[3].aP + off; sl.aE = c->sys[3].aE + off; sl.aN = c->sys[3].aN + off;
            sl.aT = c->sys[3].aT + off; sl.b = c->sys[3].b + off;
            mfx_solve_info info;
            c->dist_sub = 1;
            rc = dist_solve(c, MFX_EQ_PP, &c->grid, &sl, c->pp + off, pr.lin_tol_pp, pr.lin_maxit_pp, &info, s);
            c->dist_sub = 0;
            if (rc < 0 && rc != MFX_ERR_BREAKDOWN) return rc;
            // P0 holds the whole p' after PSLAB: its true residual over the full system
            WsView W3;
            ws_view(c->ws[3], c->ws_bytes, c->N, false, W3);
            double *Fp[MFX_NBUF] = {0};
            Fp[MFX_BUF_PP] = c->pp;
            if ((rc = exchange_state(c, 2, Fp, s)) != MFX_OK) return rc;
            if (r == P) {
                const Geo G = make_geo(c->grid);
                if ((rc = true_resid_launch(true, G, &c->sys[3], c->pp, W3.hdr, W3.part, s)) != MFX_OK) return rc;
            }
            k_meta_vals<<<1, 32, 0, s>>>(c->resid2 + 6, c->meta + 48, info.iters, info.status, info.restarts,
                                         info.rel_resid, W3.hdr);
        } else {
            double *Fp[MFX_NBUF] = {0};
            if ((rc = exchange_state(c, 2, Fp, s)) != MFX_OK) return rc;   // no ops; keeps the phase collective
        }
        MFX_CUDA_TRY(cudaEventRecord(c->ev[3], s));
        if (r == P && (rc = correct(&c->grid, &pr, star6, c->pp, st->p, st->u, st->v, st->w, st->p, s)) != MFX_OK)
            return rc;
    } else if (r == P) {
        const double *star6[6] = {c->star[0], c->star[1], c->star[2], c->dv[0], c->dv[1], c->dv[2]};
        if ((rc = assemble_eq(MFX_EQ_PP, 0, &c->grid, &pr, st, star6, &c->sys[3], c->resid2 + 6, c->ws[3],
                              c->ws_bytes, s)) != MFX_OK) return rc;
        MFX_CUDA_TRY(cudaMemsetAsync(c->pp, 0, vbytes, s));
        mfx_solve_info info;
        rc = bicgstab_solve(MFX_EQ_PP, &c->grid, &c->sys[3], c->pp, pr.lin_tol_pp, pr.lin_maxit_pp, c->ws[3],
                            c->ws_bytes, &info, s);
        if (rc < 0 && rc != MFX_ERR_BREAKDOWN) return rc;
        k_meta<<<1, 32, 0, s>>>((WsHeader *)c->ws[3], c->resid2 + 6, c->meta + 48, 1);
        MFX_CUDA_TRY(cudaEventRecord(c->ev[3], s));
        if ((rc = correct(&c->grid, &pr, star6, c->pp, st->p, st->u, st->v, st->w, st->p, s)) != MFX_OK) return rc;
    } else {
        MFX_CUDA_TRY(cudaEventRecord(c->ev[3], s));
    }
    for (int sc = 0; sc < a.n_scalars; sc++)
        if (a.owner[4 + sc] == r)
            MFX_CUDA_TRY(cudaMemcpyAsync(st->phi[sc], c->phinew[sc], vbytes, cudaMemcpyDeviceToDevice, s));
    MFX_CUDA_TRY(cudaEventRecord(c->ev[4], s));
    double *B[MFX_NBUF] = {0};
    B[MFX_BUF_U] = st->u; B[MFX_BUF_V] = st->v; B[MFX_BUF_W] = st->w; B[MFX_BUF_P] = st->p;
    for (int sc = 0; sc < a.n_scalars; sc++) B[MFX_BUF_PHI0 + sc] = st->phi[sc];
    B[MFX_BUF_META] = c->meta;
    if ((rc = exchange_fork(c, 1, B, s, c->xt[2], c->xt[3])) != MFX_OK) return rc;
    if ((rc = exchange_join(c, s)) != MFX_OK) return rc;
    MFX_CUDA_TRY(cudaEventRecord(c->ev[5], s));
    MFX_CUDA_TRY(cudaMemcpyAsync(c->meta_host, c->meta, kMetaBytes, cudaMemcpyDeviceToHost, s));
    MFX_CUDA_TRY(cudaStreamSynchronize(s));
    float ms;
    // [0] momentum+scalars, [1] GATHER (comm stream, overlaps the scalars), [2] p' assemble+solve,
    // [3] correction, [4] BCAST (comm stream), [5] total
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]); c->phase_ms[0] = ms;
    cudaEventElapsedTime(&ms, c->xt[0], c->xt[1]); c->phase_ms[1] = ms;
    cudaEventElapsedTime(&ms, c->ev[2], c->ev[3]); c->phase_ms[2] = ms;
    cudaEventElapsedTime(&ms, c->ev[3], c->ev[4]); c->phase_ms[3] = ms;
    cudaEventElapsedTime(&ms, c->xt[2], c->xt[3]); c->phase_ms[4] = ms;
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[5]); c->phase_ms[5] = ms;
    const double *m = c->meta_host;
    auto R = [&](int q) { const double den = m[16 * q + 1]; return m[16 * q] / (den > 1e-30 ? den : 1e-30); };
    memset(out, 0, sizeof(*out));
    out->R_u = R(0); out->R_v = R(1); out->R_w = R(2); out->R_cont = m[16 * 3];
    for (int sc = 0; sc < 4; sc++) out->R_phi[sc] = sc < a.n_scalars ? R(4 + sc) : 0.0;
    int worst = MFX_OK;
    for (int q = 0; q < 8; q++) {
        out->iters[q] = (int)m[16 * q + 2];
        out->status[q] = (int)m[16 * q + 3];
        out->rel_resid[q] = m[16 * q + 5];
        out->true_rel_resid[q] = m[16 * q + 7];
        if (out->status[q] < 0) worst = out->status[q];
    }
    // device errors latched by any equation's assembly or by the PIC refresh
    // (SPEC.md:356, 365), taken from the exchanged records: every rank returns
    // the same status (a rank-local latch let ranks diverge)
    for (int q = 0; q < 9; q++) {
        const double e = m[16 * q + 8];
        if (e == 0.0) continue;
        const unsigned long long at = (unsigned long long)m[16 * q + 9];
        if (q == 8) set_error("PIC drag refresh: parcel %llu outside the domain (or negative / NaN weight)", at);
        else set_error("equation %d: %s at cell %llu", q, e == (double)MFX_ERR_NONFINITE ? "non-finite coefficient"
                                                                                      : "zero diagonal", at);
        worst = (int)e;
        break;
    }
    double mx = out->R_u;
    if (out->R_v > mx) mx = out->R_v;
    if (out->R_w > mx) mx = out->R_w;
    if (out->R_cont > mx) mx = out->R_cont;
    out->converged = mx < pr.tol;
    return (mfx_status)worst;
}

}  // namespace mfx

mfx_status mfx_local_group_create(int nranks, mfx_local_group **out)
{
    MFX_ARG_CHECK(out && nranks >= 1 && nranks <= 64, "bad arguments");
    mfx_local_group *g = new mfx_local_group();
    g->nranks = nranks;
    for (int q = 0; q < nranks; q++) {
        for (int b = 0; b < MFX_NBUF; b++) g->fields[q][b] = nullptr;
        if (cudaEventCreateWithFlags(&g->ready[q], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&g->done[q], cudaEventDisableTiming) != cudaSuccess) {
            mfx::set_error("cudaEventCreate failed");
            delete g;
            return MFX_ERR_CUDA;
        }
    }
    *out = g;
    return MFX_OK;
}

void mfx_local_group_destroy(mfx_local_group *g)
{
    if (!g) return;
    for (auto &e : g->subs) mfx_local_group_destroy(e.second);
    for (int q = 0; q < g->nranks; q++) {
        cudaEventDestroy(g->ready[q]);
        cudaEventDestroy(g->done[q]);
    }
    delete g;
}

mfx_status mfx_ctx_create_local(const char *assignment, int rank, int nranks, mfx_local_group *group,
                                const mfx_grid *grid, const mfx_params *params, mfx_ctx **out)
{
    MFX_ARG_CHECK(group, "NULL group");
    return mfx::ctx_create(assignment, rank, nranks, nullptr, grid, params, out, group);
}

void mfx_ctx_destroy(mfx_ctx *c)
{
    if (!c) return;
    for (int q = 0; q < 8; q++)
        if (c->ws[q]) mfx::graph_cache_evict(c->ws[q]);   // graphs captured on this context's workspaces
    if (c->pcomm && c->pcomm != c->comm && mfx::g_nccl.CommDestroy) mfx::g_nccl.CommDestroy(c->pcomm);
    if (c->comm && mfx::g_nccl.CommDestroy) mfx::g_nccl.CommDestroy(c->comm);
    for (void *p : c->allocs) cudaFree(p);
    if (c->dist_scratch) cudaFree(c->dist_scratch);
    if (c->meta_host) cudaFreeHost(c->meta_host);
    for (int q = 0; q < 6; q++)
        if (c->ev[q]) cudaEventDestroy(c->ev[q]);
    for (int q = 0; q < 4; q++)
        if (c->xt[q]) cudaEventDestroy(c->xt[q]);
    if (c->xfork) cudaEventDestroy(c->xfork);
    if (c->xjoin) cudaEventDestroy(c->xjoin);
    if (c->cs) cudaStreamDestroy(c->cs);
    delete c;
}

namespace mfx {
mfx_status dist_solve(mfx_ctx *ctx, int kind, const mfx_grid *grid, const mfx_eqsys *A, double *x, double tol,
                      int maxit, mfx_solve_info *info, cudaStream_t s);
void dist_slab(int nz, int rank, int nranks, int *k0, int *k1);
}

mfx_status mfx_dist_solve(mfx_ctx *ctx, int kind, const mfx_grid *grid, const mfx_eqsys *A_slab, double *x_slab,
                          double tol, int maxit, mfx_solve_info *info, void *stream)
{
    return mfx::dist_solve(ctx, kind, grid, A_slab, x_slab, tol, maxit, info, (cudaStream_t)stream);
}

void mfx_dist_slab(int nz, int rank, int nranks, int *k0, int *k1) { mfx::dist_slab(nz, rank, nranks, k0, k1); }

mfx_status mfx_adapt_dt(mfx_time_ctrl *tc, int outer_iters, int converged, int *accept)
{
    MFX_ARG_CHECK(tc && accept, "NULL argument");
    MFX_ARG_CHECK(tc->dt > 0.0 && tc->dt_min > 0.0 && tc->dt_max >= tc->dt_min, "bad dt bounds");
    // a shrink factor >= 1 (or NaN) would never reach dt_min: mfx_time_step would retry forever
    MFX_ARG_CHECK(tc->shrink > 0.0 && tc->shrink < 1.0, "shrink must lie in (0, 1), got %g", tc->shrink);
    MFX_ARG_CHECK(tc->grow >= 1.0 && tc->dt_max < 1e300, "grow must be >= 1 and dt_max finite");
    if (converged) {
        if (outer_iters <= tc->grow_threshold) {
            const double d = tc->dt * tc->grow;
            tc->dt = d < tc->dt_max ? d : tc->dt_max;
        }
        *accept = 1;
        return MFX_OK;
    }
    if (tc->dt > tc->dt_min) {
        const double d = tc->dt * tc->shrink;
        tc->dt = d > tc->dt_min ? d : tc->dt_min;
        *accept = 0;
        return MFX_OK;
    }
    *accept = 1;   // accepted at dt_min although not converged
    return MFX_OK;
}

mfx_status mfx_time_step(mfx_ctx *c, mfx_state *st, mfx_time_ctrl *tc, mfx_resid *last, int *outer_iters,
                         void *stream)
{
    MFX_ARG_CHECK(c && st && tc, "NULL argument");
    MFX_ARG_CHECK(tc->max_outer >= 1, "max_outer must be >= 1");
    cudaStream_t s = (cudaStream_t)stream;
    const size_t vb = sizeof(double) * (size_t)c->N;
    const int ns = c->asg.n_scalars;
    double *fld[8] = {st->u, st->v, st->w, st->p, nullptr, nullptr, nullptr, nullptr};
    for (int q = 0; q < ns; q++) fld[4 + q] = st->phi[q];
    for (int q = 0; q < 4 + ns; q++) {
        MFX_ARG_CHECK(fld[q], "state field %d is NULL", q);
        if (!c->ts_save[q]) {
            mfx_status rc = mfx::ctx_alloc(c, (void **)&c->ts_save[q], vb);
            if (rc != MFX_OK) return rc;
        }
        MFX_CUDA_TRY(cudaMemcpyAsync(c->ts_save[q], fld[q], vb, cudaMemcpyDeviceToDevice, s));
    }
    const double dt0 = c->params.dt;
    mfx_resid R;
    memset(&R, 0, sizeof(R));
    int accepted = 0, its = 0, conv = 0;
    double dt_used = tc->dt;
    mfx_status rc = MFX_OK;
    while (!accepted) {
        c->params.dt = tc->dt;
        dt_used = tc->dt;
        conv = 0;
        its = 0;
        for (int it = 1; it <= tc->max_outer; it++) {
            rc = mfx::simple_iter(c, st, &R, s);
            its = it;
            if (rc < 0 && rc != MFX_ERR_BREAKDOWN) { c->params.dt = dt0; return rc; }
            if (R.converged) { conv = 1; break; }
        }
        rc = mfx_adapt_dt(tc, its, conv, &accepted);
        if (rc != MFX_OK) { c->params.dt = dt0; return rc; }
        if (!accepted) {
            tc->rejected += 1;
            for (int q = 0; q < 4 + ns; q++)
                MFX_CUDA_TRY(cudaMemcpyAsync(fld[q], c->ts_save[q], vb, cudaMemcpyDeviceToDevice, s));
        }
    }
    c->params.dt = dt0;
    tc->time += dt_used;
    tc->steps += 1;
    MFX_CUDA_TRY(cudaMemcpyAsync(st->u_old, st->u, vb, cudaMemcpyDeviceToDevice, s));
    MFX_CUDA_TRY(cudaMemcpyAsync(st->v_old, st->v, vb, cudaMemcpyDeviceToDevice, s));
    MFX_CUDA_TRY(cudaMemcpyAsync(st->w_old, st->w, vb, cudaMemcpyDeviceToDevice, s));
    MFX_CUDA_TRY(cudaMemcpyAsync(st->eps_old, st->eps, vb, cudaMemcpyDeviceToDevice, s));
    for (int q = 0; q < ns; q++)
        MFX_CUDA_TRY(cudaMemcpyAsync(st->phi_old[q], st->phi[q], vb, cudaMemcpyDeviceToDevice, s));
    MFX_CUDA_TRY(cudaStreamSynchronize(s));
    if (last) *last = R;
    if (outer_iters) *outer_iters = its;
    return conv ? MFX_OK : MFX_NOT_CONVERGED;
}

mfx_status mfx_ctx_set_pic(mfx_ctx *c, const mfx_parcels *parcels, const mfx_pic_params *pic, int mode)
{
    MFX_ARG_CHECK(c, "NULL ctx");
    MFX_ARG_CHECK(mode >= MFX_PIC_OFF && mode <= MFX_PIC_IMPLICIT, "bad PIC mode %d", mode);
    if (mode != MFX_PIC_OFF && c->rank == 0) {
        MFX_ARG_CHECK(parcels && pic, "the PIC device (rank 0) needs parcels and pic params");
        MFX_ARG_CHECK(parcels->n >= 0, "negative parcel count");
        MFX_ARG_CHECK(pic->d_p > 0.0, "d_p must be positive");
        c->pic_pc = *parcels;
        c->pic_pp = *pic;
        // keep a binned copy (deterministic order): the refresh is a gather over
        // it, and the parcels do not move between SIMPLE iterations of a time step
        {
            const long long n = parcels->n;
            if (n > c->pic_cap) {
                // release the smaller buffers first (they stay in c->allocs until then)
                auto release = [&](void *p) {
                    if (!p) return;
                    for (auto it = c->allocs.begin(); it != c->allocs.end(); ++it)
                        if (*it == p) { c->allocs.erase(it); break; }
                    cudaFree(p);
                };
                MFX_CUDA_TRY(cudaDeviceSynchronize());
                for (int f = 0; f < 7; f++) { release(c->pic_sorted[f]); c->pic_sorted[f] = nullptr; }
                release(c->pic_orig); c->pic_orig = nullptr;
                release(c->pic_vals); c->pic_vals = nullptr;
                c->pic_cap = 0;
                for (int f = 0; f < 7; f++) {
                    mfx_status st = mfx::ctx_alloc(c, (void **)&c->pic_sorted[f], sizeof(double) * (size_t)n);
                    if (st != MFX_OK) return st;
                }
                mfx_status st = mfx::ctx_alloc(c, (void **)&c->pic_orig, sizeof(unsigned int) * (size_t)n);
                if (st != MFX_OK) return st;
                st = mfx::ctx_alloc(c, (void **)&c->pic_vals, 7 * sizeof(double) * (size_t)n);
                if (st != MFX_OK) return st;
                c->pic_cap = n;
            }
            if (!c->pic_start) {
                mfx_status st = mfx::ctx_alloc(c, (void **)&c->pic_start, sizeof(unsigned int) * (size_t)(c->N + 1));
                if (st != MFX_OK) return st;
            }
            const size_t need = mfx::pic_sort_scratch_bytes(c->N, n);
            if (need > c->pic_scratch_bytes) {
                if (c->pic_scratch) {
                    for (auto it = c->allocs.begin(); it != c->allocs.end(); ++it)
                        if (*it == c->pic_scratch) { c->allocs.erase(it); break; }
                    cudaFree(c->pic_scratch);
                    c->pic_scratch = nullptr;
                    c->pic_scratch_bytes = 0;
                }
                mfx_status st = mfx::ctx_alloc(c, &c->pic_scratch, need);
                if (st != MFX_OK) return st;
                c->pic_scratch_bytes = need;
            }
            // the parcels may have been written on any stream of this device
            MFX_CUDA_TRY(cudaDeviceSynchronize());
            mfx_status st = mfx::pic_sort(&c->grid, pic, parcels, c->pic_sorted, c->pic_orig, c->pic_start,
                                          c->pic_scratch, c->pic_scratch_bytes, nullptr);
            if (st != MFX_OK) return st;
            MFX_CUDA_TRY(cudaDeviceSynchronize());
            mfx_parcels sp;
            sp.x = c->pic_sorted[0]; sp.y = c->pic_sorted[1]; sp.z = c->pic_sorted[2];
            sp.u = c->pic_sorted[3]; sp.v = c->pic_sorted[4]; sp.w = c->pic_sorted[5];
            sp.omega = c->pic_sorted[6]; sp.n = n;
            c->pic_pc = sp;
        }
        if (!c->pic_ws) {
            mfx_status st = mfx::ctx_alloc(c, &c->pic_ws, mfx::ws_header_bytes());
            if (st != MFX_OK) return st;
            MFX_CUDA_TRY(cudaMemset(c->pic_ws, 0, mfx::ws_header_bytes()));
            MFX_CUDA_TRY(cudaMemset(&((mfx::WsHeader *)c->pic_ws)->bad_nonfinite, 0xff, 16));
            MFX_CUDA_TRY(cudaMemset(&((mfx::WsHeader *)c->pic_ws)->bad_parcel, 0xff, 8));
        }
    }
    c->pic_mode = mode;
    c->pic_pending = mode == MFX_PIC_EXPLICIT;
    return MFX_OK;
}

double *mfx_ctx_buffer(mfx_ctx *c, int which)
{
    if (!c || which < 0 || which > 6) return nullptr;
    if (which < 3) return c->star[which];
    if (which < 6) return c->dv[which - 3];
    return c->pp;
}

mfx_status mfx_ctx_phase_times(const mfx_ctx *c, double ms[6])
{
    if (!c || !ms) return MFX_ERR_ARG;
    for (int q = 0; q < 6; q++) ms[q] = c->phase_ms[q];
    return MFX_OK;
}
