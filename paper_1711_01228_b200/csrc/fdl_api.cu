// fdl_api.cu -- host runtime behind the C ABI of include/fdl.h.
//
// One context = one GPU (rank) holding the hop rows it owns, the fp64 state of
// those rows and full-length fp32 staging vectors.  fdl_step enqueues one
// Algorithm-2 iteration on the context stream:
//   PCG solve of L^W X^{k+1} = L^{X^k} X^k (x_0 = 0)      -> P2 passes + fp64 vector kernels
//   Eq. 10 combine, P1 fused pass over {X^{k+1}, Xt}      -> f, R of both candidates
//   guard (line 6) and the stop test (DESIGN R4)          -> device select + one D->H copy
// The host only sequences launches; every arithmetic step of the path runs in
// fdl_kernels.cu.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "fdl.h"
#include "fdl_internal.h"

using namespace fdl;

namespace {

// ------------------------------------------------------------- NCCL (dlopen)
// NCCL is loaded at run time (the copy torch already loaded, if any), so the
// single-GPU library has no link-time NCCL dependency.
typedef struct ncclComm* ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { ncclInt8 = 0, ncclUint8 = 1, ncclFloat32 = 7, ncclFloat64 = 8 };

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool load(std::string& err)
    {
        if (h) return true;
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* nm : names) {
            h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (h) break;
        }
        if (!h) {
            err = "cannot dlopen libnccl.so.2";
            return false;
        }
        GetUniqueId = (decltype(GetUniqueId))dlsym(h, "ncclGetUniqueId");
        CommInitRank = (decltype(CommInitRank))dlsym(h, "ncclCommInitRank");
        CommDestroy = (decltype(CommDestroy))dlsym(h, "ncclCommDestroy");
        AllGather = (decltype(AllGather))dlsym(h, "ncclAllGather");
        GetErrorString = (decltype(GetErrorString))dlsym(h, "ncclGetErrorString");
        if (!GetUniqueId || !CommInitRank || !CommDestroy || !AllGather) {
            err = "libnccl.so.2 lacks required symbols";
            return false;
        }
        return true;
    }
};
NcclApi g_nccl;

// SplitMix64 (Steele, Lea, Flood 2014): the roulette stream of the
// probabilistic strategy and the library's own seeded initial placement.
inline uint64_t splitmix64(uint64_t& s)
{
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
inline double u01(uint64_t& s) { return (double)(splitmix64(s) >> 11) * (1.0 / 9007199254740992.0); }

constexpr int kTargetItems = 8 * 148 * 2;  // work items per all-pairs pass (fixed: results independent of GPU count)

}  // namespace

struct fdl_ctx {
    fdl_params p{};
    int n = 0, dim = 0, rank = 0, world = 1, row0 = 0, row1 = 0, nloc = 0;
    double k = 1.0, cap = INFINITY;
    int hb = 1;
    int64_t Np = 0;
    int Mrows = 0, CK = 0, NC = 0, nrb = 0, nblk = 0, nblk_loc = 0;
    int diameter = 0;
    int device = 0;
    int sm_count = 148;
    int p1_grid[3] = {0, 0, 0};
    int p2_grid = 0;
    cudaStream_t stream = nullptr, own_stream = nullptr;
    // device memory
    uint8_t* D = nullptr;
    double *diag = nullptr, *Xk = nullptr, *Xn = nullptr, *Xt = nullptr, *Rk = nullptr, *R1 = nullptr,
           *R2 = nullptr;
    double *cr = nullptr, *cz = nullptr, *cp = nullptr, *cy = nullptr;
    float *posf = nullptr, *pvec = nullptr, *lut = nullptr;
    double *part = nullptr, *blk_f = nullptr, *blk_max = nullptr, *blk_cg = nullptr;
    double* pin_slots = nullptr;  // world x 4: x_0 of the CG solution
    DevScalars* sc = nullptr;
    HostScalars* hs = nullptr;      // host-mapped (host pointer)
    HostScalars* hs_dev = nullptr;  // same memory, device pointer
    DevScalars* sc_host = nullptr;  // pinned copy target
    size_t device_bytes = 0;
    std::vector<void*> allocs;
    // run state
    int iterations = 0;
    bool stopped = false;
    int stop_reason = 0;
    double f = 0.0;
    uint64_t rng = 0;
    // accounting
    fdl_stats stats{};
    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    struct Mark { size_t start; int kind; size_t end; };
    std::vector<Mark> ev_marks;
    double setup_ms = 0.0;
    // errors
    std::string err;
    bool broken = false;
    // NCCL
    ncclComm_t comm = nullptr;
};

namespace {

fdl_status set_err(fdl_ctx* c, fdl_status s, const std::string& msg)
{
    if (c) c->err = msg;
    return s;
}

fdl_status cuda_fail(fdl_ctx* c, cudaError_t e, const char* what)
{
    char buf[512];
    snprintf(buf, sizeof buf, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
    if (c) {
        c->err = buf;
        c->broken = true;
    }
    return (e == cudaErrorMemoryAllocation) ? FDL_E_OOM : FDL_E_CUDA;
}

#define FDL_CUDA(call)                                              \
    do {                                                            \
        cudaError_t e_ = (call);                                    \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call);    \
    } while (0)

#define FDL_LAUNCH(call)                                            \
    do {                                                            \
        cudaError_t e_ = (call);                                    \
        ctx->stats.launches++;                                      \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call);    \
    } while (0)

template <typename T>
fdl_status dalloc(fdl_ctx* ctx, T** ptr, size_t count)
{
    void* q = nullptr;
    const size_t bytes = std::max<size_t>(count * sizeof(T), 256);
    cudaError_t e = cudaMalloc(&q, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        char buf[256];
        snprintf(buf, sizeof buf, "cudaMalloc(%zu bytes) failed: %s", bytes, cudaGetErrorString(e));
        ctx->err = buf;
        return FDL_E_OOM;
    }
    ctx->allocs.push_back(q);
    ctx->device_bytes += bytes;
    *ptr = static_cast<T*>(q);
    return FDL_OK;
}

#define FDL_ALLOC(ptr, count)                              \
    do {                                                   \
        fdl_status s_ = dalloc(ctx, &(ptr), (count));      \
        if (s_ != FDL_OK) return s_;                       \
    } while (0)

// --------------------------------------------------------------- validation
// S:27-31 / S:40-48: undirected (both directions), no self-loops, no
// duplicates, connected.  Also returns the eccentricity of vertex 0 (bounds
// the diameter: ecc0 <= diam <= 2 ecc0).
fdl_status validate_graph(int32_t n, const int64_t* rp, const int32_t* col, std::string& msg, int& ecc0)
{
    if (n < 1) {
        msg = "n must be >= 1";
        return FDL_E_INVALID_ARG;
    }
    if (!rp || (rp[n] > 0 && !col)) {
        msg = "row_ptr/col_idx is NULL";
        return FDL_E_INVALID_ARG;
    }
    if (rp[0] != 0) {
        msg = "row_ptr[0] != 0";
        return FDL_E_INVALID_ARG;
    }
    for (int32_t v = 0; v < n; ++v)
        if (rp[v + 1] < rp[v]) {
            msg = "row_ptr not monotone";
            return FDL_E_INVALID_ARG;
        }
    if (rp[n] > INT32_MAX) {
        msg = "too many edges";
        return FDL_E_INVALID_ARG;
    }
    std::vector<int32_t> sorted(col, col + rp[n]);
    for (int32_t v = 0; v < n; ++v) {
        for (int64_t e = rp[v]; e < rp[v + 1]; ++e) {
            if (col[e] < 0 || col[e] >= n) {
                msg = "neighbour id out of range at vertex " + std::to_string(v);
                return FDL_E_INVALID_ARG;
            }
            if (col[e] == v) {
                msg = "self-loop at vertex " + std::to_string(v);
                return FDL_E_SELF_LOOP;
            }
        }
        std::sort(sorted.begin() + rp[v], sorted.begin() + rp[v + 1]);
        for (int64_t e = rp[v] + 1; e < rp[v + 1]; ++e)
            if (sorted[e] == sorted[e - 1]) {
                msg = "duplicate neighbour at vertex " + std::to_string(v);
                return FDL_E_DUPLICATE_EDGE;
            }
    }
    for (int32_t v = 0; v < n; ++v)
        for (int64_t e = rp[v]; e < rp[v + 1]; ++e) {
            const int32_t u = col[e];
            if (!std::binary_search(sorted.begin() + rp[u], sorted.begin() + rp[u + 1], v)) {
                msg = "edge (" + std::to_string(v) + "," + std::to_string(u) + ") has no reverse";
                return FDL_E_ASYMMETRIC;
            }
        }
    std::vector<int32_t> dist(n, -1), q(n);
    int64_t head = 0, tail = 0;
    dist[0] = 0;
    q[tail++] = 0;
    ecc0 = 0;
    while (head < tail) {
        const int32_t u = q[head++];
        ecc0 = std::max(ecc0, dist[u]);
        for (int64_t e = rp[u]; e < rp[u + 1]; ++e)
            if (dist[col[e]] < 0) {
                dist[col[e]] = dist[u] + 1;
                q[tail++] = col[e];
            }
    }
    if (tail != n) {
        msg = "graph is disconnected (" + std::to_string(n - tail) + " vertices unreachable from 0)";
        return FDL_E_DISCONNECTED;
    }
    return FDL_OK;
}

int ps_p1(int dim, int nsets) { return dim == 2 ? (nsets == 1 ? 2 : 4) : (nsets == 1 ? 4 : 8); }
int ps_p2(int dim) { return dim == 2 ? 2 : 4; }

PairArgs pair_args(fdl_ctx* ctx, const float* pos, int ps)
{
    PairArgs a;
    a.D = ctx->D;
    a.pos = pos;
    a.part = ctx->part;
    a.lut = ctx->lut;
    a.Np = ctx->Np;
    a.n = ctx->n;
    a.row0 = ctx->row0;
    a.nloc = ctx->nloc;
    a.Mrows = ctx->Mrows;
    a.CK = ctx->CK;
    a.NC = ctx->NC;
    a.nrb = ctx->nrb;
    a.ps = ps;
    return a;
}

// ------------------------------------------------------------ event timing
// Intervals are (start event, end event, kind): kind 1 = P1 launch, 2 = P2
// launch, 0 = a whole fdl_step.  Events are recorded on the context stream.
cudaEvent_t next_event(fdl_ctx* ctx)
{
    if (ctx->ev_used == ctx->ev_pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        ctx->ev_pool.push_back(e);
    }
    return ctx->ev_pool[ctx->ev_used++];
}

int mark_begin(fdl_ctx* ctx, int kind)
{
    if (!ctx->timing) return -1;
    ctx->ev_marks.push_back({ctx->ev_used, kind, (size_t)-1});
    cudaEventRecord(next_event(ctx), ctx->stream);
    return (int)ctx->ev_marks.size() - 1;
}

void mark_end(fdl_ctx* ctx, int mark)
{
    if (!ctx->timing || mark < 0) return;
    ctx->ev_marks[mark].end = ctx->ev_used;
    cudaEventRecord(next_event(ctx), ctx->stream);
}

// after a stream sync: fold recorded intervals into the stats
void collect_events(fdl_ctx* ctx)
{
    double p1 = 0, p2 = 0, step = 0;
    for (auto& m : ctx->ev_marks) {
        if (m.end == (size_t)-1) continue;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev_pool[m.start], ctx->ev_pool[m.end]);
        if (m.kind == 1) p1 += ms;
        else if (m.kind == 2) p2 += ms;
        else step += ms;
    }
    ctx->stats.p1_ms += p1;
    ctx->stats.p2_ms += p2;
    if (step > 0) ctx->stats.other_ms += std::max(0.0, step - p1 - p2);
    ctx->ev_used = 0;
    ctx->ev_marks.clear();
}

// ------------------------------------------------------------ pair passes
fdl_status run_p1(fdl_ctx* ctx, int nsets)
{
    if (ctx->nloc == 0) return FDL_OK;
    PairArgs a = pair_args(ctx, ctx->posf, ps_p1(ctx->dim, nsets));
    const int mk = mark_begin(ctx, 1);
    FDL_LAUNCH(launch_p1(a, ctx->dim, nsets, ctx->hb, ctx->p1_grid[nsets], ctx->stream));
    mark_end(ctx, mk);
    ctx->stats.p1_launches++;
    const uint64_t pairs = (uint64_t)ctx->nloc * (uint64_t)(ctx->n - 1) * (uint64_t)nsets;
    ctx->stats.p1_pairs += pairs;
    if (nsets == 2) ctx->stats.p1_pairs_x2 += pairs;
    return FDL_OK;
}

fdl_status run_p2(fdl_ctx* ctx)
{
    if (ctx->nloc == 0) return FDL_OK;
    PairArgs a = pair_args(ctx, ctx->pvec, ps_p2(ctx->dim));
    const int mk = mark_begin(ctx, 2);
    FDL_LAUNCH(launch_p2(a, ctx->dim, ctx->hb, ctx->p2_grid, ctx->stream));
    mark_end(ctx, mk);
    ctx->stats.p2_launches++;
    ctx->stats.p2_pairs += (uint64_t)ctx->nloc * (uint64_t)(ctx->n - 1);
    return FDL_OK;
}

// Multi-GPU exchange: all-gather a per-rank slice of `slice_elems` elements
// (the rank's slice starts at rank*slice_elems) in place.
fdl_status allgather_inplace(fdl_ctx* ctx, void* buf, size_t slice_elems, int nccl_type, size_t esize)
{
    if (ctx->world == 1) return FDL_OK;
    char* base = static_cast<char*>(buf);
    ncclResult_t r = g_nccl.AllGather(base + (size_t)ctx->rank * slice_elems * esize, base, slice_elems, nccl_type,
                                      ctx->comm, ctx->stream);
    if (r != 0) {
        ctx->broken = true;
        return set_err(ctx, FDL_E_NCCL,
                       std::string("ncclAllGather: ") + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?"));
    }
    return FDL_OK;
}

#define FDL_TRY(x)                         \
    do {                                   \
        fdl_status s__ = (x);              \
        if (s__ != FDL_OK) return s__;     \
    } while (0)

// block partials live at global block index; with several ranks each rank
// fills its own blocks, then an all-gather gives every rank all of them.
fdl_status gather_blocks(fdl_ctx* ctx, double* blk, int nquant)
{
    if (ctx->world == 1) return FDL_OK;
    const size_t per_rank = (size_t)ctx->Mrows / kRB;
    for (int q = 0; q < nquant; ++q)
        FDL_TRY(allgather_inplace(ctx, blk + (size_t)q * ctx->nblk, per_rank, ncclFloat64, 8));
    return FDL_OK;
}

// Stress + R at the current placement Xk (one position set): used at create
// and by set_positions.
fdl_status eval_current(fdl_ctx* ctx)
{
    const int ps = ps_p1(ctx->dim, 1);
    if (ctx->nloc > 0) FDL_LAUNCH(launch_stage_pos1(ctx->Xk, ctx->posf, ctx->nloc, ctx->row0, ctx->dim, ps, ctx->stream));
    FDL_TRY(allgather_inplace(ctx, ctx->posf, (size_t)ctx->Mrows * ps, ncclFloat32, 4));
    FDL_TRY(run_p1(ctx, 1));
    if (ctx->nloc > 0)
        FDL_LAUNCH(launch_p1_reduce(ctx->part, ctx->NC, ctx->Mrows, ctx->nloc, ctx->row0, ctx->dim, 1, ctx->Rk,
                                    nullptr, ctx->blk_f, ctx->nblk, ctx->stream));
    FDL_TRY(gather_blocks(ctx, ctx->blk_f, 1));
    FDL_LAUNCH(launch_stress_finalize(ctx->blk_f, ctx->nblk, 1, ctx->sc, 1, ctx->stream));
    FDL_CUDA(cudaMemcpyAsync(ctx->sc_host, ctx->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, ctx->stream));
    FDL_CUDA(cudaStreamSynchronize(ctx->stream));
    collect_events(ctx);
    ctx->f = ctx->sc_host->f_cur;
    if (!std::isfinite(ctx->f)) return set_err(ctx, FDL_E_NONFINITE, "stress is not finite");
    return FDL_OK;
}

// Upload a full n*dim placement (original units): pin x_0 = 0, scale
// by 1/k, keep the owned rows.
fdl_status upload_positions(fdl_ctx* ctx, const double* X)
{
    std::vector<double> loc((size_t)std::max(ctx->nloc, 1) * ctx->dim);
    for (int lr = 0; lr < ctx->nloc; ++lr)
        for (int q = 0; q < ctx->dim; ++q) {
            const size_t g = (size_t)(ctx->row0 + lr) * ctx->dim + q;
            loc[(size_t)lr * ctx->dim + q] = (X[g] - X[q]) / ctx->k;
        }
    if (ctx->nloc > 0)
        FDL_CUDA(cudaMemcpyAsync(ctx->Xk, loc.data(), loc.size() * sizeof(double), cudaMemcpyHostToDevice,
                                 ctx->stream));
    return eval_current(ctx);
}

// ------------------------------------------------------------------ MS-BFS
fdl_status build_hops(fdl_ctx* ctx, const int64_t* rp, const int32_t* col, int ecc0)
{
    const int n = ctx->n;
    int64_t* d_rp = nullptr;
    int32_t* d_col = nullptr;
    uint32_t *fa = nullptr, *fb = nullptr, *vis = nullptr;
    const size_t masks = (size_t)n * kBFSWords;
    // BFS scratch is freed at the end; allocate outside the context list
    FDL_CUDA(cudaMalloc(&d_rp, sizeof(int64_t) * (n + 1)));
    FDL_CUDA(cudaMalloc(&d_col, sizeof(int32_t) * std::max<int64_t>(rp[n], 1)));
    FDL_CUDA(cudaMalloc(&fa, masks * 4));
    FDL_CUDA(cudaMalloc(&fb, masks * 4));
    FDL_CUDA(cudaMalloc(&vis, masks * 4));
    FDL_CUDA(cudaMemcpyAsync(d_rp, rp, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, ctx->stream));
    if (rp[n] > 0)
        FDL_CUDA(cudaMemcpyAsync(d_col, col, sizeof(int32_t) * rp[n], cudaMemcpyHostToDevice, ctx->stream));

    // u8 when the diameter provably fits (diam <= 2 ecc0 <= 255); u16 when it
    // provably does not (ecc0 > 255); otherwise try u8 and redo on overflow.
    int hb = (2 * ecc0 <= 255) ? 1 : (ecc0 > 255 ? 2 : 1);
    fdl_status st = FDL_OK;
    for (int attempt = 0; attempt < 2; ++attempt) {
        ctx->hb = hb;
        const int64_t V = kVecBytes / hb;
        const size_t dbytes = (size_t)ctx->Mrows * (size_t)ctx->Np * hb;
        (void)V;
        if (ctx->D) {
            cudaFree(ctx->D);
            ctx->allocs.erase(std::find(ctx->allocs.begin(), ctx->allocs.end(), (void*)ctx->D));
            ctx->D = nullptr;
        }
        void* q = nullptr;
        cudaError_t e = cudaMalloc(&q, dbytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            st = set_err(ctx, FDL_E_OOM, "hop matrix allocation of " + std::to_string(dbytes) + " bytes failed");
            break;
        }
        ctx->D = static_cast<uint8_t*>(q);
        ctx->allocs.push_back(q);
        ctx->device_bytes += dbytes;
        FDL_CUDA(cudaMemsetAsync(ctx->D, 0, dbytes, ctx->stream));
        const int maxhop = hb == 1 ? 255 : 65535;
        bool overflow = false;
        int diam = 0;
        for (int s0 = 0; s0 < n && !overflow; s0 += 32 * kBFSWords) {
            const int nsrc = std::min(32 * kBFSWords, n - s0);
            FDL_LAUNCH(launch_bfs_init(fa, vis, n, s0, ctx->stream));
            uint32_t *fin = fa, *fout = fb;
            for (int level = 1;; ++level) {
                FDL_CUDA(cudaMemsetAsync(&ctx->sc->anynew, 0, sizeof(unsigned int), ctx->stream));
                FDL_LAUNCH(launch_bfs_level(d_rp, d_col, fin, fout, vis, ctx->D, n, s0, nsrc, level, ctx->row0,
                                            ctx->row1, ctx->Np, hb, &ctx->sc->anynew, ctx->stream));
                FDL_CUDA(cudaMemcpyAsync(ctx->sc_host, ctx->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost,
                                         ctx->stream));
                FDL_CUDA(cudaStreamSynchronize(ctx->stream));
                if (!ctx->sc_host->anynew) break;
                if (level > maxhop) {
                    overflow = true;
                    break;
                }
                diam = std::max(diam, level);
                std::swap(fin, fout);
            }
        }
        if (!overflow) {
            ctx->diameter = diam;
            break;
        }
        if (hb == 2) {
            st = set_err(ctx, FDL_E_DIAMETER, "hop count exceeds 65535");
            break;
        }
        hb = 2;
    }
    cudaFree(d_rp);
    cudaFree(d_col);
    cudaFree(fa);
    cudaFree(fb);
    cudaFree(vis);
    if (st != FDL_OK) return st;
    FDL_CUDA(cudaMemsetAsync(ctx->blk_f, 0, (size_t)ctx->nblk * sizeof(double), ctx->stream));
    if (ctx->nloc > 0)
        FDL_LAUNCH(launch_diag(ctx->D, ctx->Np, ctx->hb, n, ctx->nloc, ctx->row0, ctx->diag, ctx->blk_f, ctx->stream));
    FDL_TRY(gather_blocks(ctx, ctx->blk_f, 1));
    FDL_LAUNCH(launch_set_sigma(ctx->blk_f, ctx->nblk, n, ctx->sc, ctx->stream));
    // w'_h = fp32(1/h^2) (P2 u8 table)
    float lut[256];
    lut[0] = 0.0f;
    for (int h = 1; h < 256; ++h) lut[h] = 1.0f / (float)(h * h);
    FDL_CUDA(cudaMemcpyAsync(ctx->lut, lut, sizeof lut, cudaMemcpyHostToDevice, ctx->stream));
    FDL_CUDA(cudaStreamSynchronize(ctx->stream));
    return FDL_OK;
}

fdl_status check_params(const fdl_params* p, std::string& msg)
{
    if (p->struct_size != sizeof(fdl_params)) {
        msg = "fdl_params.struct_size mismatch (call fdl_params_default)";
        return FDL_E_INVALID_ARG;
    }
    if (p->dim != 2 && p->dim != 3) {
        msg = "dim must be 2 or 3 (kernels are instantiated for these)";
        return p->dim >= 1 ? FDL_E_UNSUPPORTED : FDL_E_INVALID_ARG;
    }
    if (!(p->omega >= 0.0) || !std::isfinite(p->omega)) {
        msg = "omega must be finite and >= 0 (Eq. 10)";
        return FDL_E_INVALID_ARG;
    }
    if (!(p->tol > 0.0)) {
        msg = "tol must be > 0";
        return FDL_E_INVALID_ARG;
    }
    if (p->max_iter < 1) {
        msg = "max_iter must be >= 1";
        return FDL_E_INVALID_ARG;
    }
    if (!(p->step > 0.0)) {
        msg = "step must be > 0 (use INFINITY for no cap)";
        return FDL_E_INVALID_ARG;
    }
    if (p->weight_exp != -2.0) {
        msg = "only weight_exp = -2 (w = d^-2, P:250) is implemented";
        return FDL_E_UNSUPPORTED;
    }
    if (p->strategy != FDL_STRAT_FIXED && p->strategy != FDL_STRAT_PROB) {
        msg = "unknown strategy";
        return FDL_E_INVALID_ARG;
    }
    return FDL_OK;
}

fdl_status create_impl(int32_t n, const int64_t* rp, const int32_t* col, const double* edge_len,
                       const fdl_params* pin, const double* init_pos, const uint8_t* nccl_id, int32_t rank,
                       int32_t world, fdl_ctx* ctx)
{
    auto t0 = std::chrono::steady_clock::now();
    fdl_params p;
    fdl_params_default(&p);
    if (pin) p = *pin;
    std::string msg;
    fdl_status st = check_params(&p, msg);
    if (st != FDL_OK) return set_err(ctx, st, msg);
    if (edge_len) return set_err(ctx, FDL_E_BAD_LENGTH, "weighted edge lengths are not supported yet (unit lengths only)");
    if (world < 1 || rank < 0 || rank >= world) return set_err(ctx, FDL_E_INVALID_ARG, "bad rank/world");
    int ecc0 = 0;
    st = validate_graph(n, rp, col, msg, ecc0);
    if (st != FDL_OK) return set_err(ctx, st, msg);

    ctx->p = p;
    ctx->n = n;
    ctx->dim = p.dim;
    ctx->rank = rank;
    ctx->world = world;
    ctx->device = p.device;
    ctx->k = p.k > 0 ? p.k : std::pow((double)n, -1.0 / p.dim);
    ctx->cap = std::isfinite(p.step) ? p.step / ctx->k : INFINITY;
    if (!(p.cg_rtol > 0)) ctx->p.cg_rtol = std::max(1e-2 * p.tol, 1e-9);
    if (p.cg_max_iter <= 0) ctx->p.cg_max_iter = std::min(10 * n, 10000);
    ctx->rng = p.seed;

    FDL_CUDA(cudaSetDevice(ctx->device));
    FDL_CUDA(cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, ctx->device));
    FDL_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
    ctx->stream = ctx->own_stream;

    if (world > 1) {
        if (!g_nccl.load(msg)) return set_err(ctx, FDL_E_NCCL, msg);
        if (!nccl_id) return set_err(ctx, FDL_E_INVALID_ARG, "nccl_unique_id is NULL");
        ncclUniqueId id;
        memcpy(id.internal, nccl_id, 128);
        ncclResult_t r = g_nccl.CommInitRank(&ctx->comm, world, id, rank);
        if (r != 0)
            return set_err(ctx, FDL_E_NCCL,
                           std::string("ncclCommInitRank: ") + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?"));
    }

    // ---- sizes (all from n and world; CK from n only, so per-row sums do
    // not depend on the number of GPUs)
    const int nblk_total = (n + kRB - 1) / kRB;
    const int blocks_per_rank = (nblk_total + world - 1) / world;
    ctx->Mrows = blocks_per_rank * kRB;
    ctx->nblk = blocks_per_rank * world;
    ctx->Np = (int64_t)ctx->nblk * kRB;
    ctx->row0 = rank * ctx->Mrows;
    ctx->row1 = std::min(n, ctx->row0 + ctx->Mrows);
    ctx->nloc = std::max(0, ctx->row1 - ctx->row0);
    if (ctx->nloc == 0) ctx->row0 = ctx->row1 = std::min(n, ctx->row0);
    ctx->nblk_loc = (ctx->nloc + kRB - 1) / kRB;
    ctx->nrb = ctx->Mrows / kBM;
    {
        const int nt = (n + kColPad - 1) / kColPad;
        const int nc0 = std::min(std::max((kTargetItems + nblk_total - 1) / nblk_total, 1), nt);
        ctx->CK = ((nt + nc0 - 1) / nc0) * kColPad;
        ctx->NC = (n + ctx->CK - 1) / ctx->CK;
    }
    const int dim = ctx->dim;
    const size_t vloc = (size_t)std::max(ctx->nloc, 1) * dim;
    FDL_ALLOC(ctx->sc, 1);
    FDL_CUDA(cudaMemsetAsync(ctx->sc, 0, sizeof(DevScalars), ctx->stream));
    FDL_CUDA(cudaHostAlloc(&ctx->hs, sizeof(HostScalars), cudaHostAllocMapped));
    FDL_CUDA(cudaHostGetDevicePointer((void**)&ctx->hs_dev, ctx->hs, 0));
    FDL_CUDA(cudaHostAlloc(&ctx->sc_host, sizeof(DevScalars), cudaHostAllocDefault));
    memset(ctx->sc_host, 0, sizeof(DevScalars));
    FDL_ALLOC(ctx->diag, std::max(ctx->nloc, 1));
    FDL_ALLOC(ctx->Xk, vloc);
    FDL_ALLOC(ctx->Xn, vloc);
    FDL_ALLOC(ctx->Xt, vloc);
    FDL_ALLOC(ctx->Rk, vloc);
    FDL_ALLOC(ctx->R1, vloc);
    FDL_ALLOC(ctx->R2, vloc);
    FDL_ALLOC(ctx->cr, vloc);
    FDL_ALLOC(ctx->cz, vloc);
    FDL_ALLOC(ctx->cp, vloc);
    FDL_ALLOC(ctx->cy, vloc);
    FDL_ALLOC(ctx->posf, (size_t)ctx->Np * 8);
    FDL_ALLOC(ctx->pvec, (size_t)ctx->Np * 4);
    FDL_ALLOC(ctx->lut, 256);
    FDL_ALLOC(ctx->part, (size_t)ctx->NC * 2 * (dim + 1) * ctx->Mrows);
    FDL_ALLOC(ctx->blk_f, (size_t)2 * ctx->nblk);
    FDL_ALLOC(ctx->blk_max, (size_t)ctx->nblk);
    FDL_ALLOC(ctx->blk_cg, (size_t)16 * ctx->nblk);
    FDL_ALLOC(ctx->pin_slots, (size_t)4 * world);
    FDL_CUDA(cudaMemsetAsync(ctx->posf, 0, (size_t)ctx->Np * 8 * sizeof(float), ctx->stream));
    FDL_CUDA(cudaMemsetAsync(ctx->pvec, 0, (size_t)ctx->Np * 4 * sizeof(float), ctx->stream));
    FDL_CUDA(cudaMemsetAsync(ctx->blk_f, 0, (size_t)2 * ctx->nblk * sizeof(double), ctx->stream));
    FDL_CUDA(cudaMemsetAsync(ctx->blk_cg, 0, (size_t)16 * ctx->nblk * sizeof(double), ctx->stream));

    const int items = ctx->nrb * ctx->NC;
    for (int s = 1; s <= 2; ++s)
        ctx->p1_grid[s] = std::max(1, std::min(items, ctx->sm_count * p1_max_ctas(dim, s, 1, ctx->device)));
    ctx->p2_grid = std::max(1, std::min(items, ctx->sm_count * p2_max_ctas(dim, 1, ctx->device)));

    FDL_TRY(build_hops(ctx, rp, col, ecc0));
    if (ctx->hb == 2) {
        for (int s = 1; s <= 2; ++s)
            ctx->p1_grid[s] = std::max(1, std::min(items, ctx->sm_count * p1_max_ctas(dim, s, 2, ctx->device)));
        ctx->p2_grid = std::max(1, std::min(items, ctx->sm_count * p2_max_ctas(dim, 2, ctx->device)));
    }

    // initial placement: caller's, else seeded uniform on the unit cube
    std::vector<double> X0;
    const double* X = init_pos;
    if (!X) {
        X0.resize((size_t)n * dim);
        uint64_t s = p.seed ^ 0x5DEECE66Dull;
        for (auto& v : X0) v = (double)(float)u01(s);
        X = X0.data();
    }
    for (size_t i = 0; i < (size_t)n * dim; ++i)
        if (!std::isfinite(X[i])) return set_err(ctx, FDL_E_INVALID_ARG, "init_pos has a non-finite value");
    FDL_TRY(upload_positions(ctx, X));
    ctx->setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return FDL_OK;
}

double pick_omega(fdl_ctx* ctx)
{
    if (ctx->p.strategy == FDL_STRAT_PROB) {
        // roulette: P(0.5)=P(1.0)=0.3, P(1.5)=P(2.0)=0.2, one draw per iteration
        const double u = u01(ctx->rng);
        return u < 0.3 ? 0.5 : (u < 0.6 ? 1.0 : (u < 0.8 ? 1.5 : 2.0));
    }
    return ctx->p.omega;
}

// One Algorithm-2 iteration.
fdl_status step_impl(fdl_ctx* ctx, fdl_iter_info* info)
{
    if (ctx->broken) return set_err(ctx, FDL_E_STATE, ctx->err.empty() ? "context is broken" : ctx->err);
    if (ctx->stopped) return set_err(ctx, FDL_E_STATE, "the run has stopped; call fdl_set_positions to restart");
    const double omega = pick_omega(ctx);
    const int nsets = omega > 0.0 ? 2 : 1;
    const int dim = ctx->dim, nloc = ctx->nloc, row0 = ctx->row0;
    const int pq = ps_p2(dim), ps = ps_p1(dim, nsets);
    cudaStream_t s = ctx->stream;
    const int mstep = mark_begin(ctx, 0);
    // ---- line 4: X^{k+1} = H(X^k): PCG on Eq. 5 (zero-mean gauge), warm start X^k
    if (nloc > 0) FDL_LAUNCH(launch_cg_begin(ctx->Xk, ctx->Xn, ctx->pvec, nloc, row0, dim, pq, s));
    FDL_TRY(allgather_inplace(ctx, ctx->pvec, (size_t)ctx->Mrows * pq, ncclFloat32, 4));
    FDL_TRY(run_p2(ctx));
    if (nloc > 0)
        FDL_LAUNCH(launch_cg_init(ctx->part, ctx->NC, ctx->Mrows, ctx->Rk, ctx->Xn, ctx->diag, ctx->cr, ctx->cz,
                                  ctx->cp, ctx->pvec, ctx->blk_cg, ctx->nblk, nloc, row0, dim, pq, s));
    FDL_TRY(gather_blocks(ctx, ctx->blk_cg, 16));
    FDL_TRY(allgather_inplace(ctx, ctx->pvec, (size_t)ctx->Mrows * pq, ncclFloat32, 4));
    FDL_LAUNCH(launch_cg_finalize(ctx->blk_cg, ctx->nblk, dim, 0, ctx->p.cg_rtol, ctx->sc, ctx->hs_dev, s));
    FDL_CUDA(cudaStreamSynchronize(s));
    int cg = 0;
    while (!ctx->hs->done) {
        if (cg >= ctx->p.cg_max_iter) {
            collect_events(ctx);
            return set_err(ctx, FDL_E_SOLVER, "PCG reached cg_max_iter before cg_rtol (S:223)");
        }
        FDL_TRY(run_p2(ctx));
        if (nloc > 0)
            FDL_LAUNCH(launch_cg_ap(ctx->part, ctx->NC, ctx->Mrows, ctx->cp, ctx->cy, ctx->blk_cg, ctx->nblk, nloc,
                                    row0, dim, ctx->sc, s));
        FDL_TRY(gather_blocks(ctx, ctx->blk_cg, 4));
        FDL_LAUNCH(launch_cg_finalize(ctx->blk_cg, ctx->nblk, dim, 1, ctx->p.cg_rtol, ctx->sc, ctx->hs_dev, s));
        if (nloc > 0)
            FDL_LAUNCH(launch_cg_update(ctx->Xn, ctx->cr, ctx->cz, ctx->cp, ctx->cy, ctx->diag, ctx->blk_cg,
                                        ctx->nblk, ctx->sc, nloc, row0, dim, s));
        FDL_TRY(gather_blocks(ctx, ctx->blk_cg, 16));
        FDL_LAUNCH(launch_cg_finalize(ctx->blk_cg, ctx->nblk, dim, 2, ctx->p.cg_rtol, ctx->sc, ctx->hs_dev, s));
        if (nloc > 0) FDL_LAUNCH(launch_cg_p(ctx->cp, ctx->cz, ctx->pvec, ctx->sc, nloc, row0, dim, pq, s));
        FDL_TRY(allgather_inplace(ctx, ctx->pvec, (size_t)ctx->Mrows * pq, ncclFloat32, 4));
        FDL_CUDA(cudaStreamSynchronize(s));
        ++cg;
    }
    // ---- pin x_0 = 0, then line 5: Xt = (1+w) X^{k+1} - w X^k (Eq. 10)
    FDL_LAUNCH(launch_get_pin(ctx->Xn, ctx->pin_slots, ctx->rank, dim, ctx->row0 == 0 && nloc > 0, s));
    FDL_TRY(allgather_inplace(ctx, ctx->pin_slots, 4, ncclFloat64, 8));
    if (nloc > 0)
        FDL_LAUNCH(launch_combine(ctx->Xk, ctx->Xn, ctx->Xt, ctx->posf, ctx->blk_max, ctx->pin_slots, nloc, row0,
                                  dim, omega, ctx->cap, nsets, ps, s));
    FDL_TRY(allgather_inplace(ctx, ctx->posf, (size_t)ctx->Mrows * ps, ncclFloat32, 4));
    // ---- line 6: f(Xt), f(X^{k+1}) and the next right-hand side, one fused pass
    FDL_TRY(run_p1(ctx, nsets));
    if (nloc > 0)
        FDL_LAUNCH(launch_p1_reduce(ctx->part, ctx->NC, ctx->Mrows, nloc, row0, dim, nsets, ctx->R1, ctx->R2,
                                    ctx->blk_f, ctx->nblk, s));
    FDL_TRY(gather_blocks(ctx, ctx->blk_f, nsets));
    FDL_LAUNCH(launch_stress_finalize(ctx->blk_f, ctx->nblk, nsets, ctx->sc, 0, s));
    // ---- lines 6-8: guard
    if (nloc > 0)
        FDL_LAUNCH(launch_select(ctx->Xk, ctx->Rk, ctx->Xn, ctx->Xt, ctx->R1, ctx->R2, ctx->blk_f, ctx->blk_max,
                                 ctx->nblk, nloc, dim, nsets, ctx->sc, s));
    mark_end(ctx, mstep);
    FDL_CUDA(cudaMemcpyAsync(ctx->sc_host, ctx->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, s));
    FDL_CUDA(cudaStreamSynchronize(s));
    collect_events(ctx);
    ctx->stats.steps++;
    ctx->stats.cg_iters += cg;

    const DevScalars& h = *ctx->sc_host;
    const double f_before = ctx->f;
    // With several ranks only rank 0's block partials... all ranks computed the same f.
    double f_next = h.f_set[0];
    double f_rel = nsets == 2 ? h.f_set[1] : NAN;
    const bool accepted = nsets == 2 && (f_rel <= f_next);
    const double f_after = accepted ? f_rel : f_next;
    ctx->iterations++;
    ctx->f = f_after;
    fdl_iter_info inf{};
    inf.it = ctx->iterations;
    inf.accepted = accepted ? 1 : 0;
    inf.cg_iters = cg;
    inf.omega = omega;
    inf.f_before = f_before;
    inf.f_next = f_next;
    inf.f_relaxed = f_rel;
    inf.f_after = f_after;
    inf.rel_decrease = f_before > 0 ? (f_before - f_after) / f_before : 0.0;
    inf.cg_relres = h.relres;
    inf.maxdisp = h.maxdisp * ctx->k;
    int stop = FDL_STOP_NONE;
    if (!std::isfinite(f_after)) {
        ctx->stopped = true;
        if (info) *info = inf;
        return set_err(ctx, FDL_E_NONFINITE, "stress became non-finite (S:316)");
    }
    if (f_after == 0.0)
        stop = FDL_STOP_ZERO_STRESS;
    else if (inf.rel_decrease < ctx->p.tol)
        stop = FDL_STOP_REL_TOL;
    else if (ctx->iterations >= ctx->p.max_iter)
        stop = FDL_STOP_MAX_ITER;
    inf.stop = stop;
    if (stop) {
        ctx->stopped = true;
        ctx->stop_reason = stop;
    }
    if (info) *info = inf;
    return FDL_OK;
}

}  // namespace

// ======================================================================= ABI
extern "C" {

int32_t fdl_abi_version(void) { return FDL_ABI_VERSION; }

void fdl_params_default(fdl_params* p)
{
    if (!p) return;
    memset(p, 0, sizeof *p);
    p->struct_size = sizeof(fdl_params);
    p->dim = 2;
    p->k = 0.0;
    p->omega = 1.5;
    p->step = INFINITY;
    p->tol = 1e-4;
    p->max_iter = 500;
    p->weight_exp = -2.0;
    p->cg_rtol = 0.0;
    p->cg_max_iter = 0;
    p->strategy = FDL_STRAT_FIXED;
    p->seed = 1;
    p->device = 0;
}

const char* fdl_status_str(fdl_status s)
{
    switch (s) {
        case FDL_OK: return "FDL_OK";
        case FDL_E_INVALID_ARG: return "FDL_E_INVALID_ARG";
        case FDL_E_SELF_LOOP: return "FDL_E_SELF_LOOP";
        case FDL_E_DUPLICATE_EDGE: return "FDL_E_DUPLICATE_EDGE";
        case FDL_E_ASYMMETRIC: return "FDL_E_ASYMMETRIC";
        case FDL_E_DISCONNECTED: return "FDL_E_DISCONNECTED";
        case FDL_E_BAD_LENGTH: return "FDL_E_BAD_LENGTH";
        case FDL_E_DIAMETER: return "FDL_E_DIAMETER";
        case FDL_E_OOM: return "FDL_E_OOM";
        case FDL_E_CUDA: return "FDL_E_CUDA";
        case FDL_E_NCCL: return "FDL_E_NCCL";
        case FDL_E_SOLVER: return "FDL_E_SOLVER";
        case FDL_E_NONFINITE: return "FDL_E_NONFINITE";
        case FDL_E_UNSUPPORTED: return "FDL_E_UNSUPPORTED";
        case FDL_E_STATE: return "FDL_E_STATE";
    }
    return "FDL_E_UNKNOWN";
}

const char* fdl_last_error(const fdl_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

void fdl_destroy(fdl_ctx* ctx)
{
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->own_stream) cudaStreamSynchronize(ctx->own_stream);
    for (void* q : ctx->allocs) cudaFree(q);
    if (ctx->hs) cudaFreeHost(ctx->hs);
    if (ctx->sc_host) cudaFreeHost(ctx->sc_host);
    for (auto e : ctx->ev_pool) cudaEventDestroy(e);
    if (ctx->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(ctx->comm);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
}

static fdl_status create_common(int32_t n, const int64_t* row_ptr, const int32_t* col_idx, const double* edge_len,
                                const fdl_params* p, const double* init_pos, const uint8_t* id, int32_t rank,
                                int32_t world, fdl_ctx** out)
{
    if (!out) return FDL_E_INVALID_ARG;
    *out = nullptr;
    fdl_ctx* ctx = new fdl_ctx();
    fdl_status s = create_impl(n, row_ptr, col_idx, edge_len, p, init_pos, id, rank, world, ctx);
    if (s != FDL_OK) {
        fprintf(stderr, "fdl_create: %s: %s\n", fdl_status_str(s), ctx->err.c_str());
        fdl_destroy(ctx);
        return s;
    }
    *out = ctx;
    return FDL_OK;
}

fdl_status fdl_create(int32_t n, const int64_t* row_ptr, const int32_t* col_idx, const double* edge_len,
                      const fdl_params* p, const double* init_pos, fdl_ctx** out)
{
    return create_common(n, row_ptr, col_idx, edge_len, p, init_pos, nullptr, 0, 1, out);
}

fdl_status fdl_create_sharded(int32_t n, const int64_t* row_ptr, const int32_t* col_idx, const double* edge_len,
                              const fdl_params* p, const double* init_pos, const uint8_t* nccl_unique_id,
                              int32_t rank, int32_t world, fdl_ctx** out)
{
    return create_common(n, row_ptr, col_idx, edge_len, p, init_pos, nccl_unique_id, rank, world, out);
}

fdl_status fdl_shard_rows(int32_t n, int32_t world, int32_t rank, int32_t* row0, int32_t* row1)
{
    if (n < 1 || world < 1 || rank < 0 || rank >= world || !row0 || !row1) return FDL_E_INVALID_ARG;
    const int nblk_total = (n + kRB - 1) / kRB;
    const int bpr = (nblk_total + world - 1) / world;
    const int r0 = std::min(n, rank * bpr * kRB);
    *row0 = r0;
    *row1 = std::min(n, r0 + bpr * kRB);
    return FDL_OK;
}

fdl_status fdl_nccl_unique_id(uint8_t* out128)
{
    if (!out128) return FDL_E_INVALID_ARG;
    std::string err;
    if (!g_nccl.load(err)) return FDL_E_NCCL;
    ncclUniqueId id;
    if (g_nccl.GetUniqueId(&id) != 0) return FDL_E_NCCL;
    memcpy(out128, id.internal, 128);
    return FDL_OK;
}

fdl_status fdl_set_stream(fdl_ctx* ctx, void* cuda_stream)
{
    if (!ctx) return FDL_E_INVALID_ARG;
    cudaStreamSynchronize(ctx->stream);
    ctx->stream = cuda_stream ? static_cast<cudaStream_t>(cuda_stream) : ctx->own_stream;
    return FDL_OK;
}

fdl_status fdl_step(fdl_ctx* ctx, fdl_iter_info* info)
{
    if (!ctx) return FDL_E_INVALID_ARG;
    cudaSetDevice(ctx->device);
    return step_impl(ctx, info);
}

fdl_status fdl_run_until_converged(fdl_ctx* ctx, fdl_run_info* info)
{
    if (!ctx) return FDL_E_INVALID_ARG;
    cudaSetDevice(ctx->device);
    fdl_run_info r{};
    r.f_initial = ctx->f;
    fdl_status s = FDL_OK;
    while (!ctx->stopped) {
        fdl_iter_info it;
        s = step_impl(ctx, &it);
        if (s != FDL_OK) break;
        r.iterations++;
        r.accepted += it.accepted;
        r.cg_iters += it.cg_iters;
    }
    r.stop = ctx->stop_reason;
    r.f_final = ctx->f;
    if (info) *info = r;
    return s;
}

fdl_status fdl_get_positions(fdl_ctx* ctx, double* out, size_t count)
{
    if (!ctx || !out) return FDL_E_INVALID_ARG;
    if (count != (size_t)ctx->n * ctx->dim) return set_err(ctx, FDL_E_INVALID_ARG, "count must be n*dim");
    if (ctx->broken) return FDL_E_STATE;
    cudaSetDevice(ctx->device);
    const size_t slice = (size_t)ctx->Mrows * ctx->dim;
    if (ctx->world == 1) {
        FDL_CUDA(cudaMemcpyAsync(out, ctx->Xk, count * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        FDL_CUDA(cudaStreamSynchronize(ctx->stream));
    } else {
        double* g = nullptr;
        FDL_CUDA(cudaMalloc(&g, slice * ctx->world * sizeof(double)));
        cudaMemcpyAsync(g + ctx->rank * slice, ctx->Xk, (size_t)ctx->nloc * ctx->dim * sizeof(double),
                        cudaMemcpyDeviceToDevice, ctx->stream);
        fdl_status st = allgather_inplace(ctx, g, slice, ncclFloat64, 8);
        if (st == FDL_OK) {
            cudaMemcpyAsync(out, g, count * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream);
            cudaStreamSynchronize(ctx->stream);
        }
        cudaFree(g);
        FDL_TRY(st);
    }
    for (size_t i = 0; i < count; ++i) out[i] *= ctx->k;
    return FDL_OK;
}

fdl_status fdl_set_positions(fdl_ctx* ctx, const double* in, size_t count)
{
    if (!ctx || !in) return FDL_E_INVALID_ARG;
    if (count != (size_t)ctx->n * ctx->dim) return set_err(ctx, FDL_E_INVALID_ARG, "count must be n*dim");
    if (ctx->broken) return FDL_E_STATE;
    for (size_t i = 0; i < count; ++i)
        if (!std::isfinite(in[i])) return set_err(ctx, FDL_E_INVALID_ARG, "non-finite position");
    cudaSetDevice(ctx->device);
    ctx->stopped = false;
    ctx->stop_reason = 0;
    return upload_positions(ctx, in);
}

fdl_status fdl_eval_forces(fdl_ctx* ctx, double* R, double* A, double* stress)
{
    if (!ctx) return FDL_E_INVALID_ARG;
    if (ctx->broken) return FDL_E_STATE;
    cudaSetDevice(ctx->device);
    const int dim = ctx->dim;
    const size_t count = (size_t)ctx->n * dim, slice = (size_t)ctx->Mrows * dim;
    std::vector<double> tmp;
    auto fetch = [&](const double* dev, double* out) -> fdl_status {
        if (ctx->world == 1) {
            FDL_CUDA(cudaMemcpyAsync(out, dev, count * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        } else {
            double* g = nullptr;
            FDL_CUDA(cudaMalloc(&g, slice * ctx->world * sizeof(double)));
            cudaMemcpyAsync(g + ctx->rank * slice, dev, (size_t)ctx->nloc * dim * sizeof(double),
                            cudaMemcpyDeviceToDevice, ctx->stream);
            fdl_status st = allgather_inplace(ctx, g, slice, ncclFloat64, 8);
            cudaMemcpyAsync(out, g, count * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream);
            cudaStreamSynchronize(ctx->stream);
            cudaFree(g);
            FDL_TRY(st);
        }
        FDL_CUDA(cudaStreamSynchronize(ctx->stream));
        for (size_t i = 0; i < count; ++i) out[i] /= ctx->k;  // R = (1/k) R', A = (1/k) A'
        return FDL_OK;
    };
    if (R) FDL_TRY(fetch(ctx->Rk, R));
    if (A) {
        const int pq = ps_p2(dim);
        if (ctx->nloc > 0)
            FDL_LAUNCH(launch_cg_begin(ctx->Xk, ctx->cy, ctx->pvec, ctx->nloc, ctx->row0, dim, pq, ctx->stream));
        FDL_TRY(allgather_inplace(ctx, ctx->pvec, (size_t)ctx->Mrows * pq, ncclFloat32, 4));
        FDL_TRY(run_p2(ctx));
        if (ctx->nloc > 0)
            FDL_LAUNCH(launch_reduce_rows(ctx->part, ctx->NC, ctx->Mrows, ctx->nloc, dim, ctx->cy, ctx->stream));
        FDL_TRY(fetch(ctx->cy, A));
        collect_events(ctx);
    }
    if (stress) *stress = ctx->f;
    return FDL_OK;
}

fdl_status fdl_get_hop_rows(fdl_ctx* ctx, int32_t r0, int32_t nrows, uint16_t* out)
{
    if (!ctx || !out || nrows < 0) return FDL_E_INVALID_ARG;
    if (r0 < ctx->row0 || r0 + nrows > ctx->row1) return set_err(ctx, FDL_E_INVALID_ARG, "rows not owned");
    cudaSetDevice(ctx->device);
    if (nrows == 0) return FDL_OK;
    const int lr0 = r0 - ctx->row0;
    const int g0 = lr0 / kRowGroup, g1 = (lr0 + nrows - 1) / kRowGroup;
    const size_t group_bytes = (size_t)kRowGroup * ctx->Np * ctx->hb;
    std::vector<uint8_t> buf((size_t)(g1 - g0 + 1) * group_bytes);
    FDL_CUDA(cudaMemcpyAsync(buf.data(), ctx->D + (size_t)g0 * group_bytes, buf.size(), cudaMemcpyDeviceToHost,
                             ctx->stream));
    FDL_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int r = 0; r < nrows; ++r) {
        const int64_t lr = lr0 + r;
        for (int64_t j = 0; j < ctx->n; ++j) {
            const size_t off = d_offset(lr, j, ctx->Np, ctx->hb) - (size_t)g0 * group_bytes;
            out[(size_t)r * ctx->n + j] = ctx->hb == 1 ? buf[off] : *reinterpret_cast<const uint16_t*>(&buf[off]);
        }
    }
    return FDL_OK;
}

fdl_status fdl_get_diag(fdl_ctx* ctx, double* out, size_t count)
{
    if (!ctx || !out) return FDL_E_INVALID_ARG;
    if (count != (size_t)ctx->nloc) return set_err(ctx, FDL_E_INVALID_ARG, "count must be the owned row count");
    cudaSetDevice(ctx->device);
    if (count == 0) return FDL_OK;
    FDL_CUDA(cudaMemcpyAsync(out, ctx->diag, count * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    FDL_CUDA(cudaStreamSynchronize(ctx->stream));
    const double k2 = ctx->k * ctx->k;
    for (size_t i = 0; i < count; ++i) out[i] /= k2;  // w = w'/k^2
    return FDL_OK;
}

fdl_status fdl_get_info(fdl_ctx* ctx, fdl_ctx_info* info)
{
    if (!ctx || !info) return FDL_E_INVALID_ARG;
    fdl_ctx_info r{};
    r.n = ctx->n;
    r.dim = ctx->dim;
    r.diameter = ctx->diameter;
    r.hop_bytes = ctx->hb;
    r.row0 = ctx->row0;
    r.row1 = ctx->row1;
    r.rank = ctx->rank;
    r.world = ctx->world;
    r.iterations = ctx->iterations;
    r.k = ctx->k;
    r.f = ctx->f;
    r.hop_matrix_bytes = (uint64_t)ctx->Mrows * (uint64_t)ctx->Np * ctx->hb;
    r.device_bytes = ctx->device_bytes;
    r.setup_ms = ctx->setup_ms;
    *info = r;
    return FDL_OK;
}

fdl_status fdl_set_timing(fdl_ctx* ctx, int32_t enable)
{
    if (!ctx) return FDL_E_INVALID_ARG;
    ctx->timing = enable != 0;
    return FDL_OK;
}

fdl_status fdl_get_stats(fdl_ctx* ctx, fdl_stats* out)
{
    if (!ctx || !out) return FDL_E_INVALID_ARG;
    *out = ctx->stats;
    return FDL_OK;
}

fdl_status fdl_reset_stats(fdl_ctx* ctx)
{
    if (!ctx) return FDL_E_INVALID_ARG;
    memset(&ctx->stats, 0, sizeof ctx->stats);
    return FDL_OK;
}

fdl_status fdl_bench_ffma(int32_t device, double* tflops, double* ms)
{
    if (!tflops || !ms) return FDL_E_INVALID_ARG;
    if (cudaSetDevice(device) != cudaSuccess) return FDL_E_CUDA;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    float* out = nullptr;
    if (cudaMalloc(&out, 1024 * sizeof(float)) != cudaSuccess) return FDL_E_OOM;
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    launch_ffma_bench(out, 64, blocks, threads, s);  // warm-up
    cudaEventRecord(a, s);
    launch_ffma_bench(out, iters, blocks, threads, s);
    cudaEventRecord(b, s);
    cudaError_t e = cudaEventSynchronize(b);
    float t = 0.f;
    cudaEventElapsedTime(&t, a, b);
    const double flops = (double)blocks * threads * iters * 16.0 * 8.0 * 2.0;
    *ms = t;
    *tflops = flops / (t * 1e-3) / 1e12;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaStreamDestroy(s);
    cudaFree(out);
    return e == cudaSuccess ? FDL_OK : FDL_E_CUDA;
}

}  // extern "C"
