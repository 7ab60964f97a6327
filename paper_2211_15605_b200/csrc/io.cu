// io.cu -- MPXD state dump / restart (NEXT-4; "FieldDump",
// PAPER.md:119 "both simulations were restarted from an MFiX calculation",
// PAPER.md:121 Eq. 6 comparisons of dumped fields).  Host code: the fields
// are copied device -> host on the caller's stream and written with stdio.
//
// File layout (little-endian):
//   char     magic[4] = "MPXD"
//   uint32   version = 1
//   int32    nx, ny, nz
//   int64    n_parcels
//   float64  time, dt
//   uint32   n_fields
//   n_fields x { char name[8] (NUL padded), uint8 kind (0 cell field of N,
//                1 parcel array of n_parcels), pad[7] }
//   payload: the arrays in table order, IEEE binary64.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

namespace mfx {
namespace {

constexpr uint32_t kVersion = 1;

struct FieldRef {
    const char *name;
    int kind;            // 0 cell, 1 parcel
    double *dev;         // device pointer (load target or dump source)
};

#pragma pack(push, 1)
struct Header {
    char magic[4];
    uint32_t version;
    int32_t nx, ny, nz;
    int64_t n_parcels;
    double time, dt;
    uint32_t n_fields;
};

struct TableEntry {
    char name[8];
    uint8_t kind;
    uint8_t pad[7];
};
#pragma pack(pop)
static_assert(sizeof(Header) == 48, "packed MPXD header");
static_assert(sizeof(TableEntry) == 16, "packed MPXD table entry");

const char *kParcelNames[7] = {"px", "py", "pz", "pu", "pv", "pw", "pomega"};

std::vector<FieldRef> state_fields(const mfx_state *st, int n_scalars)
{
    std::vector<FieldRef> f = {
        {"eps", 0, st->eps}, {"eps_old", 0, st->eps_old}, {"u", 0, st->u}, {"v", 0, st->v}, {"w", 0, st->w},
        {"u_old", 0, st->u_old}, {"v_old", 0, st->v_old}, {"w_old", 0, st->w_old}, {"p", 0, st->p},
        {"beta", 0, st->beta}, {"sbu", 0, st->sbeta_u}, {"sbv", 0, st->sbeta_v}, {"sbw", 0, st->sbeta_w}};
    static const char *phin[4] = {"phi0", "phi1", "phi2", "phi3"};
    static const char *phon[4] = {"phio0", "phio1", "phio2", "phio3"};
    for (int s = 0; s < n_scalars; s++) {
        f.push_back({phin[s], 0, st->phi[s]});
        f.push_back({phon[s], 0, st->phi_old[s]});
    }
    return f;
}

struct File {
    FILE *f = nullptr;
    ~File() { if (f) fclose(f); }
};

}  // namespace

mfx_status state_dump(const char *path, const mfx_grid *grid, const mfx_state *st, int n_scalars,
                      const mfx_parcels *pc, double time, double dt, cudaStream_t s)
{
    MFX_ARG_CHECK(path && grid && st, "NULL path/grid/state");
    MFX_ARG_CHECK(n_scalars >= 0 && n_scalars <= 4, "n_scalars %d", n_scalars);
    MFX_ARG_CHECK(grid->nx > 0 && grid->ny > 0 && grid->nz > 0, "bad grid");
    std::vector<FieldRef> fields = state_fields(st, n_scalars);
    for (auto &fr : fields) MFX_ARG_CHECK(fr.dev, "state field %s is NULL", fr.name);
    const long long np = pc ? pc->n : 0;
    MFX_ARG_CHECK(np >= 0, "negative parcel count");
    if (np > 0) {
        const double *pa[7] = {pc->x, pc->y, pc->z, pc->u, pc->v, pc->w, pc->omega};
        for (int q = 0; q < 7; q++) {
            MFX_ARG_CHECK(pa[q], "parcel array %d is NULL", q);
            fields.push_back({kParcelNames[q], 1, const_cast<double *>(pa[q])});
        }
    }
    const long long N = (long long)grid->nx * grid->ny * grid->nz;
    File F;
    F.f = fopen(path, "wb");
    if (!F.f) { set_error("cannot open %s for writing", path); return MFX_ERR_ARG; }
    Header h;
    memset(&h, 0, sizeof(h));
    memcpy(h.magic, "MPXD", 4);
    h.version = kVersion;
    h.nx = grid->nx; h.ny = grid->ny; h.nz = grid->nz;
    h.n_parcels = np;
    h.time = time; h.dt = dt;
    h.n_fields = (uint32_t)fields.size();
    bool ok = fwrite(&h, sizeof(h), 1, F.f) == 1;
    for (auto &fr : fields) {
        TableEntry e;
        memset(&e, 0, sizeof(e));
        memcpy(e.name, fr.name, strnlen(fr.name, sizeof(e.name)));   // NUL padded by the memset
        e.kind = (uint8_t)fr.kind;
        ok = ok && fwrite(&e, sizeof(e), 1, F.f) == 1;
    }
    std::vector<double> buf;
    for (auto &fr : fields) {
        const size_t n = (size_t)(fr.kind ? np : N);
        buf.resize(n);
        MFX_CUDA_TRY(cudaMemcpyAsync(buf.data(), fr.dev, n * sizeof(double), cudaMemcpyDefault, s));
        MFX_CUDA_TRY(cudaStreamSynchronize(s));
        ok = ok && fwrite(buf.data(), sizeof(double), n, F.f) == n;
    }
    if (!ok) { set_error("write error on %s", path); return MFX_ERR_ARG; }
    return MFX_OK;
}

static mfx_status read_header(FILE *f, const char *path, Header &h, std::vector<TableEntry> &tab)
{
    if (fread(&h, sizeof(h), 1, f) != 1) { set_error("%s: truncated header", path); return MFX_ERR_ARG; }
    if (memcmp(h.magic, "MPXD", 4) != 0) { set_error("%s: bad magic (not an MPXD dump)", path); return MFX_ERR_ARG; }
    if (h.version != kVersion) { set_error("%s: unsupported version %u", path, h.version); return MFX_ERR_ARG; }
    if (h.nx <= 0 || h.ny <= 0 || h.nz <= 0 || h.n_parcels < 0 || h.n_fields > 64) {
        set_error("%s: corrupt header", path);
        return MFX_ERR_ARG;
    }
    tab.resize(h.n_fields);
    if (h.n_fields && fread(tab.data(), sizeof(TableEntry), h.n_fields, f) != h.n_fields) {
        set_error("%s: truncated field table", path);
        return MFX_ERR_ARG;
    }
    return MFX_OK;
}

mfx_status dump_info(const char *path, int dims[3], long long *n_parcels, int *n_scalars, double *time, double *dt)
{
    MFX_ARG_CHECK(path, "NULL path");
    File F;
    F.f = fopen(path, "rb");
    if (!F.f) { set_error("cannot open %s", path); return MFX_ERR_ARG; }
    Header h;
    std::vector<TableEntry> tab;
    mfx_status st = read_header(F.f, path, h, tab);
    if (st != MFX_OK) return st;
    if (dims) { dims[0] = h.nx; dims[1] = h.ny; dims[2] = h.nz; }
    if (n_parcels) *n_parcels = h.n_parcels;
    int ns = 0;
    for (auto &e : tab)
        if (!strncmp(e.name, "phi", 3) && e.name[3] >= '0' && e.name[3] <= '3' && e.name[4] == 0) ns++;
    if (n_scalars) *n_scalars = ns;
    if (time) *time = h.time;
    if (dt) *dt = h.dt;
    return MFX_OK;
}

mfx_status state_load(const char *path, const mfx_grid *grid, mfx_state *st, int n_scalars,
                      double *const parcel_out[7], long long parcel_capacity, long long *n_parcels, double *time,
                      double *dt, cudaStream_t s)
{
    MFX_ARG_CHECK(path && grid && st, "NULL path/grid/state");
    MFX_ARG_CHECK(n_scalars >= 0 && n_scalars <= 4, "n_scalars %d", n_scalars);
    File F;
    F.f = fopen(path, "rb");
    if (!F.f) { set_error("cannot open %s", path); return MFX_ERR_ARG; }
    Header h;
    std::vector<TableEntry> tab;
    mfx_status rc = read_header(F.f, path, h, tab);
    if (rc != MFX_OK) return rc;
    if (h.nx != grid->nx || h.ny != grid->ny || h.nz != grid->nz) {
        set_error("%s: grid %dx%dx%d does not match %dx%dx%d", path, h.nx, h.ny, h.nz, grid->nx, grid->ny, grid->nz);
        return MFX_ERR_ARG;
    }
    if (h.n_parcels > 0 && parcel_out) {
        MFX_ARG_CHECK(h.n_parcels <= parcel_capacity, "%s holds %lld parcels, capacity %lld", path,
                      (long long)h.n_parcels, parcel_capacity);
    }
    std::vector<FieldRef> want = state_fields(st, n_scalars);
    const long long N = (long long)grid->nx * grid->ny * grid->nz;
    // validate everything before the first device copy, so a bad file leaves
    // the caller's state untouched: the payload length must equal what the
    // header and table imply, and every wanted field exist
    {
        const long pos = ftell(F.f);
        unsigned long long payload = 0;
        for (auto &e : tab) payload += 8ull * (unsigned long long)(e.kind ? h.n_parcels : N);
        if (pos < 0 || fseek(F.f, 0, SEEK_END) != 0) { set_error("%s: cannot seek", path); return MFX_ERR_ARG; }
        const long end = ftell(F.f);
        if (end < 0 || (unsigned long long)(end - pos) != payload) {
            set_error("%s: payload is %ld bytes, header and table imply %llu", path, end - pos, payload);
            return MFX_ERR_ARG;
        }
        if (fseek(F.f, pos, SEEK_SET) != 0) { set_error("%s: cannot seek", path); return MFX_ERR_ARG; }
        for (auto &fr : want) {
            bool present = false;
            for (auto &e : tab) {
                char name[9];
                memcpy(name, e.name, 8);
                name[8] = 0;
                if (e.kind == 0 && !strcmp(fr.name, name)) present = true;
            }
            if (!present) {
                set_error("%s: requested state field %s is missing", path, fr.name);
                return MFX_ERR_ARG;
            }
        }
    }
    std::vector<double> buf;
    int found = 0;
    for (auto &e : tab) {
        char name[9];
        memcpy(name, e.name, 8);
        name[8] = 0;
        const size_t n = (size_t)(e.kind ? h.n_parcels : N);
        buf.resize(n);
        if (n && fread(buf.data(), sizeof(double), n, F.f) != n) {
            set_error("%s: truncated payload (field %s)", path, name);
            return MFX_ERR_ARG;
        }
        double *dst = nullptr;
        if (e.kind == 0) {
            for (auto &fr : want)
                if (!strcmp(fr.name, name)) { dst = fr.dev; found++; }
        } else if (parcel_out) {
            for (int q = 0; q < 7; q++)
                if (!strcmp(kParcelNames[q], name)) dst = parcel_out[q];
        }
        if (dst && n) {
            MFX_CUDA_TRY(cudaMemcpyAsync(dst, buf.data(), n * sizeof(double), cudaMemcpyDefault, s));
            MFX_CUDA_TRY(cudaStreamSynchronize(s));
        }
    }
    if (found != (int)want.size()) {
        set_error("%s: %d of the %d requested state fields present", path, found, (int)want.size());
        return MFX_ERR_ARG;
    }
    if (n_parcels) *n_parcels = h.n_parcels;
    if (time) *time = h.time;
    if (dt) *dt = h.dt;
    return MFX_OK;
}

}  // namespace mfx

extern "C" {
mfx_status mfx_state_dump(const char *path, const mfx_grid *grid, const mfx_state *state, int n_scalars,
                          const mfx_parcels *parcels, double time, double dt, void *stream)
{
    return mfx::state_dump(path, grid, state, n_scalars, parcels, time, dt, (cudaStream_t)stream);
}
mfx_status mfx_dump_info(const char *path, int dims[3], long long *n_parcels, int *n_scalars, double *time,
                         double *dt)
{
    return mfx::dump_info(path, dims, n_parcels, n_scalars, time, dt);
}
mfx_status mfx_state_load(const char *path, const mfx_grid *grid, mfx_state *state, int n_scalars,
                          double *const parcel_out[7], long long parcel_capacity, long long *n_parcels,
                          double *time, double *dt, void *stream)
{
    return mfx::state_load(path, grid, state, n_scalars, parcel_out, parcel_capacity, n_parcels, time, dt,
                           (cudaStream_t)stream);
}
}
