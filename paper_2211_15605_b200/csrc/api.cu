// api.cu -- the extern "C" boundary of libmfx.so (include/mfx.h): argument
// marshalling, workspace layout, error reporting and launch instrumentation.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace mfx {

// ------------------------------------------------------------------ errors
static thread_local char g_err[1024] = "";

void set_error(const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

// ------------------------------------------------------------------ workspace
static size_t r256(size_t b) { return (b + 255) & ~(size_t)255; }
size_t ws_header_bytes() { return r256(sizeof(WsHeader)); }
static size_t ws_part_bytes() { return r256(sizeof(dd) * kPartCap); }
size_t ws_total_bytes(long long N) { return ws_header_bytes() + ws_part_bytes() + 7 * r256(sizeof(double) * N); }

bool ws_view(void *ws, size_t bytes, long long N, bool need_vectors, WsView &W)
{
    if (!ws) { set_error("workspace is NULL"); return false; }
    if (((uintptr_t)ws) & 255) { set_error("workspace must be 256-byte aligned"); return false; }
    const size_t need = need_vectors ? ws_total_bytes(N) : ws_header_bytes() + ws_part_bytes();
    if (bytes < need) { set_error("workspace too small: %zu < %zu bytes", bytes, need); return false; }
    char *b = (char *)ws;
    W.hdr = (WsHeader *)b;
    W.part = (dd *)(b + ws_header_bytes());
    char *v = b + ws_header_bytes() + ws_part_bytes();
    const size_t vb = r256(sizeof(double) * N);
    double *vec[7];
    for (int q = 0; q < 7; q++) vec[q] = need_vectors ? (double *)(v + vb * q) : nullptr;
    W.r = vec[0]; W.rh = vec[1]; W.p[0] = vec[2]; W.p[1] = vec[3]; W.v[0] = vec[4]; W.v[1] = vec[5]; W.t = vec[6];
    return true;
}

int reduce_grid(long long N)
{
    // fixed, device-independent grid -> fixed reduction order
    long long b = (N + 255) / 256;
    if (b > 148 * 8) b = 148 * 8;
    if (b < 1) b = 1;
    return (int)b;
}

// ------------------------------------------------------------------ instrumentation
static std::atomic<long long> g_launches{0};
static std::atomic<int> g_prof{0};
struct ProfRec { int id; cudaEvent_t a, b; };
static std::mutex g_mu;
static std::vector<ProfRec> g_recs;
static std::vector<cudaEvent_t> g_pool;
static thread_local cudaEvent_t g_pending = nullptr;

static cudaEvent_t get_event()
{
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_pool.empty()) {
        cudaEvent_t e = g_pool.back();
        g_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

void count_launch(int id, cudaStream_t s, bool start)
{
    if (!start) g_launches.fetch_add(1, std::memory_order_relaxed);
    if (!g_prof.load(std::memory_order_relaxed) || id >= 12) return;
    if (start) {
        g_pending = get_event();
        cudaEventRecord(g_pending, s);
    } else if (g_pending) {
        cudaEvent_t e = get_event();
        cudaEventRecord(e, s);
        std::lock_guard<std::mutex> lk(g_mu);
        g_recs.push_back({id, g_pending, e});
        g_pending = nullptr;
    }
}

bool prof_enabled() { return g_prof.load(std::memory_order_relaxed) != 0; }

// ------------------------------------------------------------------ options
static int env_default(const char *name, int dflt)
{
    const char *e = getenv(name);
    return e ? atoi(e) : dflt;
}
static std::atomic<int> g_opt_path{-1};
static std::atomic<int> g_opt_graphs{-1};
static std::atomic<int> g_opt_pdl{-1};
static std::atomic<int> g_opt_asm{-1};
int opt_asm_tma()
{
    int v = g_opt_asm.load();
    if (v < 0) {
        const char *e = getenv("MFX_KERNELS");
        v = (e && e[0] == 'v' && e[1] == '1') ? 0 : env_default("MFX_ASM_TMA", 1);
        g_opt_asm.store(v);
    }
    return v;
}
int opt_pdl()
{
    int v = g_opt_pdl.load();
    if (v < 0) {
        v = env_default("MFX_PDL", 0);   // off: measured slower (early dependent CTAs unbalance the persistent grids)
        g_opt_pdl.store(v);
    }
    return v;
}
int opt_solver_path()
{
    int v = g_opt_path.load();
    if (v < 0) {
        const char *e = getenv("MFX_KERNELS");
        v = (e && e[0] == 'v' && e[1] == '1') ? 3 : env_default("MFX_SOLVER_PATH", 0);
        g_opt_path.store(v);
    }
    return v;
}
int opt_graphs()
{
    int v = g_opt_graphs.load();
    if (v < 0) {
        v = env_default("MFX_GRAPH", 1);
        g_opt_graphs.store(v);
    }
    return v;
}
long long launch_count_get() { return g_launches.load(); }
void launch_count_set(long long v) { g_launches.store(v); }
void launch_count_add(long long v) { g_launches.fetch_add(v); }

// forward declarations (other translation units)
bool grid_valid(const mfx_grid *g, bool scalar);
mfx_status assemble_eq(int, int, const mfx_grid *, const mfx_params *, const mfx_state *, const double *const[6],
                       mfx_eqsys *, double *, void *, size_t, cudaStream_t);
mfx_status spmv(int, const mfx_grid *, const mfx_eqsys *, const double *, double *, cudaStream_t);
mfx_status bicgstab_solve(int, const mfx_grid *, const mfx_eqsys *, double *, double, int, void *, size_t,
                          mfx_solve_info *, cudaStream_t);
mfx_status correct(const mfx_grid *, const mfx_params *, const double *const[6], const double *, const double *,
                   double *, double *, double *, double *, cudaStream_t);
mfx_status parse_assignment(const char *, int, mfx_assignment *);
mfx_status exchange_plan(const mfx_assignment *, int, int, mfx_xfer *, int, int *, int);
mfx_status nccl_unique_id(unsigned char out[128]);
mfx_status ctx_create(const char *, int, int, const unsigned char *, const mfx_grid *, const mfx_params *,
                      mfx_ctx **, mfx_local_group *);
mfx_status exchange_state(mfx_ctx *, int, double *const[MFX_NBUF], cudaStream_t);
mfx_status simple_iter(mfx_ctx *, mfx_state *, mfx_resid *, cudaStream_t);

}  // namespace mfx

using namespace mfx;

#define API extern "C" __attribute__((visibility("default")))

API const char *mfx_last_error(void) { return g_err; }
API const char *mfx_version(void) { return "mfx 0.2 (sm_100a, fp64; TMA z-marching BiCGSTAB, cluster solver, PIC coupling)"; }

API size_t mfx_workspace_bytes(const mfx_grid *grid, int kind)
{
    (void)kind;
    if (!grid) return 0;
    return ws_total_bytes((long long)grid->nx * grid->ny * grid->nz);
}

API mfx_status mfx_ws_init(void *ws, size_t ws_bytes, void *stream)
{
    MFX_ARG_CHECK(ws && ws_bytes >= ws_header_bytes(), "bad workspace");
    cudaStream_t s = (cudaStream_t)stream;
    MFX_CUDA_TRY(cudaMemsetAsync(ws, 0, ws_header_bytes(), s));
    WsHeader *h = (WsHeader *)ws;
    MFX_CUDA_TRY(cudaMemsetAsync(&h->bad_nonfinite, 0xff, 16, s));
    MFX_CUDA_TRY(cudaMemsetAsync(&h->bad_parcel, 0xff, 8, s));
    return MFX_OK;
}

API mfx_status mfx_ws_check(void *ws, size_t ws_bytes, void *stream)
{
    MFX_ARG_CHECK(ws && ws_bytes >= ws_header_bytes(), "bad workspace");
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long bad[2], badp;
    WsHeader *h = (WsHeader *)ws;
    MFX_CUDA_TRY(cudaMemcpyAsync(bad, &h->bad_nonfinite, 16, cudaMemcpyDeviceToHost, s));
    MFX_CUDA_TRY(cudaMemcpyAsync(&badp, &h->bad_parcel, 8, cudaMemcpyDeviceToHost, s));
    MFX_CUDA_TRY(cudaStreamSynchronize(s));
    MFX_CUDA_TRY(cudaMemsetAsync(&h->bad_nonfinite, 0xff, 16, s));
    MFX_CUDA_TRY(cudaMemsetAsync(&h->bad_parcel, 0xff, 8, s));
    if (badp != ~0ull) {
        set_error("parcel %llu outside the domain (or negative / NaN weight)", badp);
        return MFX_ERR_ARG;
    }
    if (bad[0] != ~0ull) {
        set_error("non-finite coefficient at cell %llu", bad[0]);
        return MFX_ERR_NONFINITE;
    }
    if (bad[1] != ~0ull) {
        set_error("zero diagonal at cell %llu", bad[1]);
        return MFX_ERR_ZERO_DIAG;
    }
    return MFX_OK;
}

API mfx_status mfx_assemble_eq(int kind, int scalar_id, const mfx_grid *grid, const mfx_params *params,
                               const mfx_state *state, const double *const star[6], mfx_eqsys *out, double *resid2,
                               void *ws, size_t ws_bytes, void *stream)
{
    return assemble_eq(kind, scalar_id, grid, params, state, star, out, resid2, ws, ws_bytes, (cudaStream_t)stream);
}

API mfx_status mfx_pic_deposit_eps(const mfx_grid *grid, const mfx_pic_params *pic, const mfx_parcels *parcels,
                                   double *eps_g, void *ws, size_t ws_bytes, void *stream)
{
    return pic_deposit_eps(grid, pic, parcels, eps_g, ws, ws_bytes, (cudaStream_t)stream);
}

API size_t mfx_pic_sort_scratch_bytes(const mfx_grid *grid, long long n_parcels)
{
    if (!grid || n_parcels < 0) return 0;
    return pic_sort_scratch_bytes((long long)grid->nx * grid->ny * grid->nz, n_parcels);
}

API mfx_status mfx_pic_sort(const mfx_grid *grid, const mfx_pic_params *pic, const mfx_parcels *parcels,
                            double *const out[7], unsigned int *orig, unsigned int *bin_start, void *scratch,
                            size_t scratch_bytes, void *stream)
{
    return pic_sort(grid, pic, parcels, out, orig, bin_start, scratch, scratch_bytes, (cudaStream_t)stream);
}

API mfx_status mfx_pic_deposit_eps_binned(const mfx_grid *grid, const mfx_pic_params *pic,
                                          const mfx_parcels *binned, const unsigned int *orig,
                                          const unsigned int *bin_start, double *eps_g, double *vals, void *ws,
                                          size_t ws_bytes, void *stream)
{
    double *outs[4] = {eps_g, nullptr, nullptr, nullptr};
    return pic_deposit_binned(0, grid, nullptr, pic, binned, orig, bin_start, nullptr, nullptr, nullptr, nullptr,
                              outs, nullptr, vals, ws, ws_bytes, (cudaStream_t)stream);
}

API mfx_status mfx_pic_drag_binned(const mfx_grid *grid, const mfx_params *params, const mfx_pic_params *pic,
                                   const mfx_parcels *binned, const unsigned int *orig, const unsigned int *bin_start,
                                   const double *eps_g, const double *u, const double *v, const double *w,
                                   double *beta, double *sbeta_u, double *sbeta_v, double *sbeta_w, double *K,
                                   double *vals, void *ws, size_t ws_bytes, void *stream)
{
    double *outs[4] = {beta, sbeta_u, sbeta_v, sbeta_w};
    return pic_deposit_binned(1, grid, params, pic, binned, orig, bin_start, eps_g, u, v, w, outs, K, vals, ws,
                              ws_bytes, (cudaStream_t)stream);
}

API mfx_status mfx_pic_drag(const mfx_grid *grid, const mfx_params *params, const mfx_pic_params *pic,
                            const mfx_parcels *parcels, const double *eps_g, const double *u, const double *v,
                            const double *w, double *beta, double *sbeta_u, double *sbeta_v, double *sbeta_w,
                            double *K, void *ws, size_t ws_bytes, void *stream)
{
    return pic_drag(grid, params, pic, parcels, eps_g, u, v, w, beta, sbeta_u, sbeta_v, sbeta_w, K, ws, ws_bytes,
                    (cudaStream_t)stream);
}

API mfx_status mfx_spmv(int kind, const mfx_grid *grid, const mfx_eqsys *A, const double *x, double *y, void *stream)
{
    return spmv(kind, grid, A, x, y, (cudaStream_t)stream);
}

API mfx_status mfx_bicgstab_solve(int kind, const mfx_grid *grid, const mfx_eqsys *A, double *x, double tol,
                                  int maxit, void *ws, size_t ws_bytes, mfx_solve_info *info, void *stream)
{
    return bicgstab_solve(kind, grid, A, x, tol, maxit, ws, ws_bytes, info, (cudaStream_t)stream);
}

API mfx_status mfx_correct(const mfx_grid *grid, const mfx_params *params, const double *const star[6],
                           const double *pp, const double *p, double *u, double *v, double *w, double *p_new,
                           void *stream)
{
    return correct(grid, params, star, pp, p, u, v, w, p_new, (cudaStream_t)stream);
}

API mfx_status mfx_parse_assignment(const char *text, int nranks, mfx_assignment *out)
{
    return parse_assignment(text, nranks, out);
}

API mfx_status mfx_exchange_plan(const mfx_assignment *a, int rank, int phase, mfx_xfer *ops, int max_ops, int *n_ops,
                                 int nz)
{
    return exchange_plan(a, rank, phase, ops, max_ops, n_ops, nz);
}

API mfx_status mfx_nccl_unique_id(unsigned char out[128]) { return nccl_unique_id(out); }

API mfx_status mfx_ctx_create(const char *assignment, int rank, int nranks, const unsigned char *uid,
                              const mfx_grid *grid, const mfx_params *params, mfx_ctx **out)
{
    return ctx_create(assignment, rank, nranks, uid, grid, params, out, nullptr);
}

API mfx_status mfx_exchange_state(mfx_ctx *ctx, int phase, double *const fields[MFX_NBUF], void *stream)
{
    return exchange_state(ctx, phase, fields, (cudaStream_t)stream);
}

API mfx_status mfx_simple_iter(mfx_ctx *ctx, mfx_state *state, mfx_resid *out, void *stream)
{
    return simple_iter(ctx, state, out, (cudaStream_t)stream);
}

API void mfx_prof_enable(int on) { g_prof.store(on ? 1 : 0); }

API void mfx_prof_reset(void)
{
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto &r : g_recs) { g_pool.push_back(r.a); g_pool.push_back(r.b); }
    g_recs.clear();
}

API mfx_status mfx_prof_read(int counts[16], double ms[16])
{
    MFX_ARG_CHECK(counts && ms, "NULL out");
    MFX_CUDA_TRY(cudaDeviceSynchronize());
    for (int q = 0; q < 16; q++) { counts[q] = 0; ms[q] = 0.0; }
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto &r : g_recs) {
        float t = 0.f;
        if (cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess) {
            counts[r.id] += 1;
            ms[r.id] += t;
        }
    }
    return MFX_OK;
}

API long long mfx_launch_count(void) { return g_launches.load(); }

namespace mfx {
int cluster_size();
void cluster_size_set(int cl);
void graph_cache_evict(const void *ws);
size_t graph_cache_size();
}
API void mfx_graph_cache_clear(void) { graph_cache_evict(nullptr); }
API size_t mfx_graph_cache_size(void) { return graph_cache_size(); }

API mfx_status mfx_set_option(const char *key, int value)
{
    MFX_ARG_CHECK(key, "NULL key");
    if (!strcmp(key, "solver_path")) {
        MFX_ARG_CHECK(value >= 0 && value <= 5, "solver_path must be 0..5");
        g_opt_path.store(value);
        return MFX_OK;
    }
    if (!strcmp(key, "graphs")) {
        g_opt_graphs.store(value ? 1 : 0);
        return MFX_OK;
    }
    if (!strcmp(key, "pdl")) {
        g_opt_pdl.store(value ? 1 : 0);
        return MFX_OK;
    }
    if (!strcmp(key, "asm_tma")) {
        g_opt_asm.store(value ? 1 : 0);
        return MFX_OK;
    }
    if (!strcmp(key, "cluster_size")) {
        MFX_ARG_CHECK(value == 8 || value == 16, "cluster_size must be 8 or 16");
        cluster_size_set(value);
        return MFX_OK;
    }
    set_error("unknown option '%s'", key);
    return MFX_ERR_ARG;
}

API int mfx_get_option(const char *key)
{
    if (!key) return -1;
    if (!strcmp(key, "solver_path")) return opt_solver_path();
    if (!strcmp(key, "graphs")) return opt_graphs();
    if (!strcmp(key, "pdl")) return opt_pdl();
    if (!strcmp(key, "asm_tma")) return opt_asm_tma();
    if (!strcmp(key, "cluster_size")) return cluster_size();
    return -1;
}
