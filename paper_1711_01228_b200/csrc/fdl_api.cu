// fdl_api.cu -- host runtime behind the C ABI of include/fdl.h.
//
// A context holds, on one GPU, the upper-triangle hop tiles of its tile range
// and replicated O(n) state (fp64 positions, R, PCG vectors; fp32 staging).
// fdl_step enqueues one Algorithm-2 iteration:
//   PCG solve of L^W X^{k+1} = L^{X^k} X^k          -> symmetric P2 passes + fp64 vector kernels
//   pin x_0 = 0, Eq. 10 combine              -> k_combine
//   fused symmetric P1 pass over {X^{k+1}, Xt}       -> f and R of both candidates
//   guard (lines 6-8) on device, stop test on host   -> one D->H scalar copy
// With several GPUs each rank evaluates the pairs of its tiles; after every
// pair pass the dense per-rank partials are all-gathered and summed in rank
// order, so every rank holds identical state and takes identical decisions.
// The host only sequences launches; all arithmetic of the path is in the
// kernels (fdl_sym.cu, fdl_kernels.cu).
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <map>
#include <tuple>
#include <mutex>
#include <condition_variable>

#include "fdl.h"
#include "fdl_internal.h"

using namespace fdl;

namespace {

#ifndef FDL_CG_HISTORY_DEFAULT
#define FDL_CG_HISTORY_DEFAULT 8  // step differences kept for the recycled PCG start (R27)
#endif

// ------------------------------------------------------------- NCCL (dlopen)
// NCCL is loaded at run time (the copy torch already loaded, if any), so the
// single-GPU library has no link-time NCCL dependency.
typedef struct ncclComm* ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { ncclInt8 = 0, ncclUint8 = 1, ncclInt32 = 2, ncclFloat32 = 7, ncclFloat64 = 8 };

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
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
        Send = (decltype(Send))dlsym(h, "ncclSend");
        Recv = (decltype(Recv))dlsym(h, "ncclRecv");
        GroupStart = (decltype(GroupStart))dlsym(h, "ncclGroupStart");
        GroupEnd = (decltype(GroupEnd))dlsym(h, "ncclGroupEnd");
        GetErrorString = (decltype(GetErrorString))dlsym(h, "ncclGetErrorString");
        if (!GetUniqueId || !CommInitRank || !CommDestroy || !AllGather || !Send || !Recv || !GroupStart ||
            !GroupEnd) {
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

// work-item length in tiles (strip segments)
// tiles per work item: 32 for large triangles (C5's 1.2e6 tiles: half the i-side partials
// and reduction work, P2 5.22 -> 5.07 ms, other -0.24 ms per step), kSeg = 16 below (C4's
// 7e4 tiles and C3 got slower with 32: fewer items per CTA).  A function of n only, so the
// items -- and every fp32 segment sum -- are the same for any number of GPUs
int seg_len(int64_t nb) { return nb * (nb + 1) / 2 >= ((int64_t)1 << 18) ? 2 * kSeg : kSeg; }

// (I, J) of triangle index t (row-major upper triangle over nb blocks)
void tri_coords(int64_t t, int64_t nb, int64_t& I, int64_t& J)
{
    int64_t lo = 0, hi = nb - 1;  // largest I with tri_index(I, I) <= t
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) / 2;
        if (tri_index(mid, mid, nb) <= t)
            lo = mid;
        else
            hi = mid - 1;
    }
    I = lo;
    J = I + (t - tri_index(I, I, nb));
}

}  // namespace

extern "C" fdl_status fdl_shard_tiles(int32_t n, int32_t world, int32_t rank, int64_t* t0, int64_t* t1);

// In-process loopback transport (test hook): the ranks of one group are contexts
// in one process, driven from separate host threads.  An all-gather syncs the
// rank's stream, copies its slice to a shared host buffer, waits on a host
// barrier for every rank, and copies the gathered buffer back; no kernel ever
// waits for another rank (the exchange is host-side), so all ranks may share
// one GPU.  Same data movement as the NCCL all-gather, hence the same results.
struct fdl_group {
    int world = 0;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    std::vector<char> buf;
    void barrier()
    {
        std::unique_lock<std::mutex> lk(m);
        const uint64_t g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};

struct StepGraphCounts {
    uint64_t launches, p1_launches, p2_launches, p1_pairs, p2_pairs, p1_pairs_x2, p1_pairs_nor;
};
struct StepGraph {
    cudaGraphExec_t exec = nullptr;
    StepGraphCounts once{}, body{};
};

struct fdl_ctx {
    fdl_params p{};
    int n = 0, dim = 0, rank = 0, world = 1;
    double k = 1.0, cap = INFINITY;
    double alpha = -2.0;                          // weight exponent (NEXT-3 any)
    double fscale = 1.0, rscale = 1.0, dscale = 1.0;  // k^(alpha+2), k^(alpha+1), k^alpha
    bool general = false;                         // fp32 distance tiles (weighted or alpha != -2)
    int hb = 1;
    int nb = 0;              // vertex blocks of kT
    int64_t npad = 0;        // nb * kT
    int64_t t0 = 0, t1 = 0;  // local tile range [t0, t1) in triangle order
    int Ilo = 0, Ihi = -1;   // row blocks of the local tiles
    int nitems = 0;
    uint64_t local_pairs = 0;  // unordered pairs in the local tiles
    int diameter = 0;
    int device = 0;
    int sm_count = 148;
    int nblk = 0;  // 256-row reduction blocks of the vector kernels
    int grid_p1[3] = {0, 0, 0}, grid_p2 = 0, grid_diag = 0, grid_enum = 0, grid_p1s = 0, grid_p1a = 0, grid_p1r = 0;
    bool p1_split = false;  // P1 over {X^{k+1}, Xt} computes R of Xt only (R(X^{k+1}) on rejection)
    bool p1_predict = false;     // p1_split = 2: a step whose guard is predicted to reject runs the two-set pass
    bool p1_fused_next = true;   // ... the prediction for the next step (the first step of a run: reject)
    bool p1_fused_now = false;   // ... the current step runs the two-set pass
    cudaStream_t stream = nullptr, own_stream = nullptr;
    // device memory
    uint8_t* D = nullptr;
    int4* items = nullptr;
    // per grid size: slot -> item schedule of the pair passes (item_order)
    std::vector<std::pair<int, int*>> item_orders;
    int *it_lo = nullptr, *it_hi = nullptr;
    float* jpart = nullptr;
    float* ipart = nullptr;
    double* spart = nullptr;
    double* stress_scratch = nullptr;  // chunk sums of the two-stage stress reduction
    double *rparts = nullptr, *sparts = nullptr;  // this rank's dense partial [world * rslice rows][C]; stress partials
    // row-slice exchange of the pair passes (several ranks): rank g owns rows
    // [g * rslice, (g + 1) * rslice) of the reduction
    int64_t rslice = 0;
    double* xrecv = nullptr;  // [world][rslice * C]: the other ranks' partials of this rank's rows
    double* xgath = nullptr;  // [world][rslice * C + 2]: reduced row slices + stress partials, all ranks
    double *diag = nullptr, *Xk = nullptr, *Xn = nullptr, *Xt = nullptr, *Rk = nullptr, *R1 = nullptr,
           *R2 = nullptr;
    double *cr = nullptr, *cz = nullptr, *cp = nullptr, *cy = nullptr;
    double *Ak = nullptr, *An = nullptr, *At = nullptr;  // carried L^W X^k, L^W X^{k+1}, L^W Xt
    double *Xprev = nullptr, *Aprev = nullptr;           // X^{k-1}, L^W X^{k-1} (PCG start extrapolation)
    double *Vh = nullptr, *AVh = nullptr;               // recycled start (R27): kGalMax step differences, L^W of them
    double* blk_gal = nullptr;                          // ... block partials of its Gram systems
    double* spart_enum = nullptr;  // [item][kEnumNC] enumerating-strategy stress partials
    double* enum_f = nullptr;      // [kEnumMax] candidate stresses
    double* omega_v = nullptr;   // per-vertex relax factors (fdl_set_omega_vertex), device
    double omega_v_max = 0.0;
    bool a_valid = false;
    bool ext_ok = false;  // Xprev/Aprev hold the previous accepted iterate
    int a_age = 0;  // steps since Ak was last computed by a full pass
    float *posf = nullptr, *pvec = nullptr;
    double *blk_max = nullptr, *blk_cg = nullptr;
    double* pin_slots = nullptr;
    DevScalars* sc = nullptr;
    HostScalars* hs = nullptr;      // host-mapped (host pointer)
    HostScalars* hs_dev = nullptr;  // same memory, device pointer
    DevScalars* sc_host = nullptr;  // pinned copy target
    size_t device_bytes = 0;
    uint64_t hop_bytes_total = 0;
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
    struct Mark {
        size_t start;
        int kind;
        size_t end;
    };
    std::vector<Mark> ev_marks;
    double setup_ms = 0.0;
    double setup_dist_ms = 0.0;       // MS-BFS (or Bellman-Ford) part of the setup
    unsigned long long bfs_bytes = 0;  // MS-BFS level-kernel gather bytes
    // errors
    std::string err;
    bool broken = false;
    // NCCL
    ncclComm_t comm = nullptr;
    fdl_group* group = nullptr;  // loopback transport instead of NCCL (test hook)
    // CUDA-graph steps (fdl_params.use_graphs): one captured graph per step shape
    bool use_graphs = false;
    bool capturing = false;
    uint64_t steps_eager = 0;  // the first step runs eagerly (kernel attributes set, lazy allocations done)
    cudaStream_t aux_stream = nullptr;
    std::map<std::tuple<int, int, int, double>, StepGraph> graphs;
    bool emulated = false;  // world > 1 without communicator (fdl_eval_partial only)
    bool distributed = false;  // partials exchanged through comm or group (any world, incl. 1)
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

#define FDL_CUDA(call)                                           \
    do {                                                         \
        cudaError_t e_ = (call);                                 \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
    } while (0)

#define FDL_LAUNCH(call)                                         \
    do {                                                         \
        cudaError_t e_ = (call);                                 \
        ctx->stats.launches++;                                   \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
    } while (0)

// launchers that enqueue two kernels (count both in the launch statistics)
#define FDL_LAUNCH2(call)      \
    do {                       \
        FDL_LAUNCH(call);      \
        ctx->stats.launches++; \
    } while (0)
#define FDL_LAUNCH3(call)          \
    do {                           \
        FDL_LAUNCH(call);          \
        ctx->stats.launches += 2;  \
    } while (0)

#define FDL_TRY(x)                     \
    do {                               \
        fdl_status s__ = (x);          \
        if (s__ != FDL_OK) return s__; \
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

#define FDL_ALLOC(ptr, count)                         \
    do {                                              \
        fdl_status s_ = dalloc(ctx, &(ptr), (count)); \
        if (s_ != FDL_OK) return s_;                  \
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

// ------------------------------------------------------------ event timing
// Intervals are (start event, end event, kind): kind 1 = P1 pass, 2 = P2
// pass, 3 = DIAG pass, 4 = split line-6 pass (P1S, also a P1 pass), 0 = a whole
// fdl_step.  Recorded on the context stream.
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
    if (!ctx->timing || ctx->capturing) return -1;
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
        if (m.kind == 4) {  // the split line-6 pass (also counted as P1)
            ctx->stats.p1s_ms += ms;
            p1 += ms;
        } else if (m.kind == 1) p1 += ms;
        else if (m.kind == 2) p2 += ms;
        else if (m.kind == 0) step += ms;
    }
    ctx->stats.p1_ms += p1;
    ctx->stats.p2_ms += p2;
    if (step > 0) ctx->stats.other_ms += std::max(0.0, step - p1 - p2);
    ctx->ev_used = 0;
    ctx->ev_marks.clear();
}

// Schedule of the pair passes' work items over `grid` CTAs (CTA b takes slots b, b + grid,
// ...): items sorted by tile count, longest first, dealt to the CTAs in snake order (round r
// left to right when r is even, right to left when odd).  Work items are strip segments of
// up to kSeg tiles and each row ends in a shorter one, so plain round-robin over triangle
// order leaves per-CTA work uneven (C5: the busiest CTA has 2.3% more tiles than the mean,
// the pass waits for it); the snake deal is within 0.05%.  Outputs are indexed by item and
// tile, so the schedule does not change any sum.  FDL_ITEM_ORDER=rr: plain round-robin.
static std::vector<int> snake_order(const std::vector<int4>& items, int grid)
{
    const int m = (int)items.size();
    std::vector<int> order(std::max(m, 1), 0);
    static const bool rr = [] {
        const char* e = getenv("FDL_ITEM_ORDER");
        return e && std::string(e) == "rr";
    }();
    if (rr || grid <= 1) {
        for (int i = 0; i < m; ++i) order[i] = i;
        return order;
    }
    std::vector<int> srt(m);
    for (int i = 0; i < m; ++i) srt[i] = i;
    std::stable_sort(srt.begin(), srt.end(), [&](int a, int b) { return items[a].z > items[b].z; });
    for (int s = 0; s < m; ++s) {
        const int r = s / grid, c = s % grid;
        const int cnt = std::min(grid, m - r * grid);  // items in this round
        const int b = (r & 1) ? cnt - 1 - c : c;
        order[r * grid + b] = srt[s];
    }
    return order;
}

static fdl_status build_item_orders(fdl_ctx* ctx, const std::vector<int4>& items)
{
    const int grids[] = {ctx->grid_p1[1], ctx->grid_p1[2], ctx->grid_p2, ctx->grid_diag,
                         ctx->grid_enum,  ctx->grid_p1s,   ctx->grid_p1a, ctx->grid_p1r};
    for (int g : grids) {
        if (g <= 0) continue;
        bool have = false;
        for (auto& e : ctx->item_orders) have = have || e.first == g;
        if (have) continue;
        const std::vector<int> o = snake_order(items, g);
        int* d = nullptr;
        FDL_ALLOC(d, o.size());
        FDL_CUDA(cudaMemcpyAsync(d, o.data(), sizeof(int) * o.size(), cudaMemcpyHostToDevice, ctx->stream));
        FDL_CUDA(cudaStreamSynchronize(ctx->stream));  // `o` is a host temporary
        ctx->item_orders.emplace_back(g, d);
    }
    return FDL_OK;
}

static const int* item_order(const fdl_ctx* ctx, int grid)
{
    for (auto& e : ctx->item_orders)
        if (e.first == grid) return e.second;
    return nullptr;
}

// Multi-GPU: all-gather the rank slices (slice_elems each, rank slice at
// rank * slice_elems) of `buf` in place.
fdl_status allgather_inplace(fdl_ctx* ctx, void* buf, size_t slice_elems, int nccl_type, size_t esize)
{
    if (!ctx->distributed) return FDL_OK;
    char* base = static_cast<char*>(buf);
    if (ctx->group) {
        fdl_group& G = *ctx->group;
        const size_t sb = slice_elems * esize;
        FDL_CUDA(cudaStreamSynchronize(ctx->stream));
        {
            std::lock_guard<std::mutex> lk(G.m);
            if (G.buf.size() < sb * G.world) G.buf.resize(sb * G.world);
        }
        G.barrier();  // every rank sized the buffer
        // copies on the context's (non-blocking) stream: a plain cudaMemcpy from pageable
        // memory may return before the data lands and is not ordered with that stream
        FDL_CUDA(cudaMemcpyAsync(G.buf.data() + (size_t)ctx->rank * sb, base + (size_t)ctx->rank * sb, sb,
                                 cudaMemcpyDeviceToHost, ctx->stream));
        FDL_CUDA(cudaStreamSynchronize(ctx->stream));
        G.barrier();  // every slice is in
        FDL_CUDA(cudaMemcpyAsync(base, G.buf.data(), sb * G.world, cudaMemcpyHostToDevice, ctx->stream));
        FDL_CUDA(cudaStreamSynchronize(ctx->stream));
        G.barrier();  // every rank read the buffer before it is reused
        return FDL_OK;
    }
    ncclResult_t r = g_nccl.AllGather(base + (size_t)ctx->rank * slice_elems * esize, base, slice_elems, nccl_type,
                                      ctx->comm, ctx->stream);
    if (r != 0) {
        ctx->broken = true;
        return set_err(ctx, FDL_E_NCCL,
                       std::string("ncclAllGather: ") + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?"));
    }
    return FDL_OK;
}

// Multi-GPU: all-to-all of row slices.  `src` holds world slices of `slice_elems`
// doubles (slice h for rank h); rank h's slice of every rank lands in
// dst[g * slice_elems] for source rank g (the reduce-scatter's data movement; the
// sum is done by a kernel in rank order, so it is deterministic).
fdl_status alltoall_slices(fdl_ctx* ctx, const double* src, double* dst, size_t slice_elems)
{
    const int G = ctx->world;
    const size_t sb = slice_elems * sizeof(double);
    if (ctx->group) {
        fdl_group& Gr = *ctx->group;
        FDL_CUDA(cudaStreamSynchronize(ctx->stream));
        {
            std::lock_guard<std::mutex> lk(Gr.m);
            if (Gr.buf.size() < sb * G * G) Gr.buf.resize(sb * G * G);
        }
        Gr.barrier();
        // rank g's whole partial at host row g (G slices)
        FDL_CUDA(cudaMemcpyAsync(Gr.buf.data() + (size_t)ctx->rank * G * sb, src, sb * G, cudaMemcpyDeviceToHost,
                                 ctx->stream));
        FDL_CUDA(cudaStreamSynchronize(ctx->stream));
        Gr.barrier();
        // slice `rank` of every rank's partial: G rows of sb bytes, pitch G * sb
        FDL_CUDA(cudaMemcpy2DAsync(dst, sb, Gr.buf.data() + (size_t)ctx->rank * sb, (size_t)G * sb, sb, G,
                                   cudaMemcpyHostToDevice, ctx->stream));
        FDL_CUDA(cudaStreamSynchronize(ctx->stream));
        Gr.barrier();
        return FDL_OK;
    }
    ncclResult_t r = g_nccl.GroupStart();
    for (int h = 0; h < G && r == 0; ++h) {
        r = g_nccl.Send(src + (size_t)h * slice_elems, slice_elems, ncclFloat64, h, ctx->comm, ctx->stream);
        if (r == 0) r = g_nccl.Recv(dst + (size_t)h * slice_elems, slice_elems, ncclFloat64, h, ctx->comm, ctx->stream);
    }
    const ncclResult_t r2 = g_nccl.GroupEnd();
    if (r == 0) r = r2;
    if (r != 0) {
        ctx->broken = true;
        return set_err(ctx, FDL_E_NCCL,
                       std::string("ncclSend/ncclRecv: ") + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?"));
    }
    return FDL_OK;
}

// ------------------------------------------------------------ pair passes
// One symmetric pass over the local tiles + the per-row fixed-order
// reduction; with several ranks the dense rank partials are all-gathered and
// summed in rank order.  out0 gets components [0, D0), out1 the rest.
fdl_status run_sym(fdl_ctx* ctx, int mode, int nsets, const float* pos, double* out0, double* out1, int set_cur,
                   bool p2_finish = true)
{
    const int dim = ctx->dim;
    const bool p1 = mode == kSymP1 || mode == kSymP1S || mode == kSymP1A;
    const int C = mode == kSymP1 ? nsets * dim
                                 : (mode == kSymP1A ? 2 * dim
                                                    : ((mode == kSymP2 || mode == kSymP1S || mode == kSymP1R) ? dim : 1));
    const int D0 = (mode == kSymP1 || mode == kSymP1A) ? dim : C;  // P1A: R into out0, L^W X into out1
    const int inter = (mode == kSymP1 && nsets == 2) ? 1 : 0;  // P1 two sets: components interleaved by set
    SymArgs a;
    a.D = ctx->D;
    a.pos = pos;
    a.jpart = ctx->jpart;
    a.ipart = ctx->ipart;
    a.spart = ctx->spart;
    a.items = ctx->items;
    a.nitems = ctx->nitems;
    a.n = ctx->n;
    a.ntiles = ctx->t1 - ctx->t0;
    a.nstage = ctx->npad;
    a.magic = 0x4B000000u;
    a.alpha = (float)ctx->alpha;
    const int grid = mode == kSymP1S   ? ctx->grid_p1s
                     : mode == kSymP1A ? ctx->grid_p1a
                     : mode == kSymP1R ? ctx->grid_p1r
                     : (mode == kSymP1 ? ctx->grid_p1[nsets] : (mode == kSymP2 ? ctx->grid_p2 : ctx->grid_diag));
    a.order = item_order(ctx, grid);
    if (ctx->nitems > 0 && !a.order) return set_err(ctx, FDL_E_STATE, "no work-item schedule for the grid");
    const int mk = mark_begin(ctx, mode == kSymP1S ? 4 : ((p1 || mode == kSymP1R) ? 1 : (mode == kSymP2 ? 2 : 3)));
    if (ctx->nitems > 0) FDL_LAUNCH(launch_sym(a, mode, dim, nsets, ctx->hb, grid, ctx->stream));
    mark_end(ctx, mk);
    if (mode == kSymP1R) {  // R-only rejection pass: a P1 launch (its time is P1 time)
        ctx->stats.p1_launches++;
        ctx->stats.p1_pairs += ctx->local_pairs;
    }
    if (p1) {
        ctx->stats.p1_launches++;
        ctx->stats.p1_pairs += ctx->local_pairs * (uint64_t)nsets;
        if (mode == kSymP1S) {
            ctx->stats.p1_pairs_nor += ctx->local_pairs;
            ctx->stats.p1s_launches++;
        }
        if (nsets == 2) ctx->stats.p1_pairs_x2 += ctx->local_pairs * 2;
    } else if (mode == kSymP2) {
        ctx->stats.p2_launches++;
        ctx->stats.p2_pairs += ctx->local_pairs;
    }
    if (!ctx->distributed) {
        FDL_LAUNCH(launch_sym_reduce(ctx->ipart, ctx->jpart, ctx->it_lo, ctx->it_hi, ctx->nb, ctx->t0, ctx->t1,
                                     ctx->Ilo, ctx->Ihi, C, D0,
                                     inter, out0, out1, ctx->stream));
        if (mode == kSymP2 && p2_finish)  // product form: L^W p = diag p - sum_j w p_j (rank-local diag when emulated)
            FDL_LAUNCH(launch_p2_finish(out0, pos, ctx->diag, ctx->n, dim, ps_p2(dim), ctx->stream));
        if (p1) {
            FDL_LAUNCH2(launch_sym_stress(ctx->spart, ctx->nitems * 8, nsets, ctx->sparts, ctx->stress_scratch, ctx->stream));
            FDL_LAUNCH(launch_stress_ranks(ctx->sparts, 2, 1, nsets, ctx->sc, set_cur, ctx->stream));
        }
        return FDL_OK;
    }
    // Several ranks: this rank's dense partial (rows of its tiles) -> all-to-all of row
    // slices -> each rank sums its slice over the ranks in rank order -> all-gather of
    // the reduced slices, with each rank's stress partial appended to its slice (one
    // all-gather per pass).  Every element is the rank-order sum of the rank partials
    // (as a sum of all-gathered partials would be), on 2 (G-1)/G of a dense vector
    // per rank instead of G - 1 dense vectors.
    const size_t rs = (size_t)ctx->rslice * C;  // elements of one row slice
    const size_t gs = rs + 2;                   // ... plus the stress partials
    double* mine = ctx->rparts;
    FDL_LAUNCH(launch_sym_reduce(ctx->ipart, ctx->jpart, ctx->it_lo, ctx->it_hi, ctx->nb, ctx->t0, ctx->t1, ctx->Ilo,
                                 ctx->Ihi, C, C, 0,
                                 mine, nullptr, ctx->stream));
    FDL_TRY(alltoall_slices(ctx, mine, ctx->xrecv, rs));
    double* myg = ctx->xgath + (size_t)ctx->rank * gs;
    FDL_LAUNCH(launch_slice_sum(ctx->xrecv, ctx->world, rs, myg, ctx->stream));
    if (p1)
        FDL_LAUNCH2(launch_sym_stress(ctx->spart, ctx->nitems * 8, nsets, myg + rs, ctx->stress_scratch, ctx->stream));
    FDL_TRY(allgather_inplace(ctx, ctx->xgath, gs, ncclFloat64, 8));
    FDL_LAUNCH(launch_slice_unpack(ctx->xgath, ctx->world, ctx->rslice, ctx->npad, C, D0, inter, out0, out1,
                                   ctx->stream));
    if (mode == kSymP2 && p2_finish)
        FDL_LAUNCH(launch_p2_finish(out0, pos, ctx->diag, ctx->n, dim, ps_p2(dim), ctx->stream));
    if (p1) FDL_LAUNCH(launch_stress_ranks(ctx->xgath + rs, gs, ctx->world, nsets, ctx->sc, set_cur, ctx->stream));
    return FDL_OK;
}

// Stress + R at the current placement Xk (one position set): used at create
// and by set_positions.
fdl_status eval_current(fdl_ctx* ctx)
{
    const int ps = ps_p1(ctx->dim, 1);
    FDL_LAUNCH(launch_stage_pos1(ctx->Xk, ctx->posf, ctx->n, 0, ctx->dim, ps, ctx->stream));
    if (ctx->general) {
        FDL_TRY(run_sym(ctx, kSymP1, 1, ctx->posf, ctx->Rk, nullptr, 1));
    } else {
        // one pass for f, R = L^X X and L^W X (the first step needs no refresh pass)
        FDL_TRY(run_sym(ctx, kSymP1A, 1, ctx->posf, ctx->Rk, ctx->Ak, 1));
        ctx->a_valid = true;
        ctx->a_age = 0;
    }
    FDL_CUDA(cudaMemcpyAsync(ctx->sc_host, ctx->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, ctx->stream));
    FDL_CUDA(cudaStreamSynchronize(ctx->stream));
    collect_events(ctx);
    ctx->p1_fused_next = true;  // a new placement: its first relaxed step is predicted to be rejected (R30)
    ctx->f = ctx->sc_host->f_cur;
    if (!std::isfinite(ctx->f)) return set_err(ctx, FDL_E_NONFINITE, "stress is not finite");
    return FDL_OK;
}

// Upload a full n*dim placement (original units): pin x_0 = 0, scale by 1/k.
fdl_status upload_positions(fdl_ctx* ctx, const double* X)
{
    ctx->a_valid = false;
    ctx->ext_ok = false;
    // (the recycled-start basis is kept: V and L^W V belong to the matrix L^W, which
    // does not depend on the placement, so they remain a valid Galerkin subspace, R27)
    // raw copy (a DMA straight from the caller's buffer when it is page-locked), then the
    // pin x_0 = 0 and the 1/k scaling on the device: (x - x_0) / k in fp64
    const size_t count = (size_t)ctx->n * ctx->dim;
    FDL_CUDA(cudaMemcpyAsync(ctx->Xt, X, count * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    FDL_LAUNCH(launch_pin_scale(ctx->Xt, ctx->Xk, ctx->n, ctx->dim, ctx->k, 0, ctx->stream));
    return eval_current(ctx);
}

// Temporary device buffers of one call, freed on every return path.
struct Scratch {
    std::vector<void*> bufs;
    ~Scratch()
    {
        for (void* q : bufs) cudaFree(q);
    }
    template <typename T>
    cudaError_t alloc(T** p, size_t bytes)
    {
        void* q = nullptr;
        const cudaError_t e = cudaMalloc(&q, bytes);
        if (e == cudaSuccess) bufs.push_back(q);
        *p = static_cast<T*>(q);
        return e;
    }
    void release(void* q)
    {
        for (auto& b : bufs)
            if (b == q) {
                cudaFree(b);
                b = nullptr;
            }
    }
};

// Source batches as compact graph neighbourhoods: clusters of up to S sources of
// [lo, hi), each grown by BFS (over vertices not yet taken) from the first untaken
// vertex.  Sources close to each other have nearly concentric wavefronts, so a batch's
// searches touch a band of the graph at a time instead of all of it (geometric graphs:
// MS-BFS on C4, the weighted sweeps on W4).  Inside a batch, each 32-source word
// is itself a compact ball (compact_words): the BFS order of the batch puts a
// shell of the seed's neighbourhood into a word, whose sources then reach a
// distant vertex over many sweeps with one or two bits each.
static void compact_words(const int64_t* rp, const int32_t* col, int* seg, int cnt, std::vector<char>& inb,
                          std::vector<int>& seen, int& stamp)
{
    if (cnt <= 32) return;
    for (int i = 0; i < cnt; ++i) inb[seg[i]] = 1;  // 1: in the batch, untaken; 2: taken
    std::vector<int> out, q;
    out.reserve((size_t)cnt);
    for (int i = 0; i < cnt; ++i) {
        const int s0 = seg[i];
        if (inb[s0] != 1) continue;
        // a ball around s0 over the batch's vertices (taken or not) until the current
        // word is full; an exhausted ball leaves the word to the next seed
        ++stamp;
        q.clear();
        q.push_back(s0);
        seen[s0] = stamp;
        for (size_t h = 0; h < q.size(); ++h) {
            const int u = q[h];
            if (inb[u] == 1) {
                inb[u] = 2;
                out.push_back(u);
                if (out.size() % 32 == 0) break;
            }
            for (int64_t e = rp[u]; e < rp[u + 1]; ++e) {
                const int w = col[e];
                if (inb[w] && seen[w] != stamp) {
                    seen[w] = stamp;
                    q.push_back(w);
                }
            }
        }
    }
    for (int i = 0; i < cnt; ++i) inb[seg[i]] = 0;
    std::copy(out.begin(), out.end(), seg);
}

std::vector<int> cluster_sources(int32_t n, const int64_t* rp, const int32_t* col, int lo, int hi, int S,
                                 bool words)
{
    std::vector<char> inb(words ? (size_t)n : 0, 0);
    std::vector<int> seen(words ? (size_t)n : 0, 0);
    int stamp = 0;
    std::vector<int> order;
    order.reserve((size_t)std::max(0, hi - lo));
    std::vector<char> taken((size_t)n, 0);
    std::vector<int> q;
    q.reserve((size_t)n);
    std::vector<int> mark((size_t)n, -1);
    int cluster = 0;
    for (int seed = lo; seed < hi; ++seed) {
        if (taken[seed]) continue;
        q.clear();
        q.push_back(seed);
        mark[seed] = cluster;
        int got = 0;
        for (size_t h = 0; h < q.size() && got < S; ++h) {
            const int u = q[h];
            if (u >= lo && u < hi && !taken[u]) {
                taken[u] = 1;
                order.push_back(u);
                ++got;
            }
            for (int64_t e = rp[u]; e < rp[u + 1]; ++e) {
                const int w = col[e];
                if (mark[w] != cluster) {
                    mark[w] = cluster;
                    q.push_back(w);
                }
            }
        }
        if (words) compact_words(rp, col, order.data() + (order.size() - got), got, inb, seen, stamp);
        ++cluster;
    }
    return order;
}

// FDL_SETUP_TRACE=1: host timestamps of the setup phases on stderr (each after a
// stream sync, so only for diagnosis)
void setup_trace(fdl_ctx* ctx, const char* what)
{
    static const bool on = getenv("FDL_SETUP_TRACE") != nullptr;
    if (!on) return;
    static auto t_last = std::chrono::steady_clock::now();
    cudaStreamSynchronize(ctx->stream);
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "fdl setup: %-28s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t_last).count());
    t_last = t;
}

// ------------------------------------------------------------------ MS-BFS
// Sources: the rows of the blocks I of the local tiles.  Writes the upper
// triangle tiles of the local range; the Jacobi diagonal follows from one
// symmetric DIAG pass.
fdl_status build_hops(fdl_ctx* ctx, const int64_t* rp, const int32_t* col, int ecc0)
{
    const int n = ctx->n;
    int64_t* d_rp = nullptr;
    int32_t* d_col = nullptr;
    uint32_t *fa = nullptr, *fb = nullptr, *vis = nullptr;
    const size_t masks = (size_t)n * kBFSWords;
    Scratch tmp;
    FDL_CUDA(tmp.alloc(&d_rp, sizeof(int64_t) * (n + 1)));
    FDL_CUDA(tmp.alloc(&d_col, sizeof(int32_t) * std::max<int64_t>(rp[n], 1)));
    FDL_CUDA(tmp.alloc(&fa, masks * 4));
    FDL_CUDA(tmp.alloc(&fb, masks * 4));
    FDL_CUDA(tmp.alloc(&vis, masks * 4));
    FDL_CUDA(cudaMemcpyAsync(d_rp, rp, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, ctx->stream));
    if (rp[n] > 0)
        FDL_CUDA(cudaMemcpyAsync(d_col, col, sizeof(int32_t) * rp[n], cudaMemcpyHostToDevice, ctx->stream));

    int64_t Ilo = 0, Jlo = 0, Ihi = -1, Jhi = 0;
    if (ctx->t1 > ctx->t0) {
        tri_coords(ctx->t0, ctx->nb, Ilo, Jlo);
        tri_coords(ctx->t1 - 1, ctx->nb, Ihi, Jhi);
    }
    const int src_lo = (int)std::min<int64_t>(n, Ilo * kT);
    const int src_hi = (int)std::min<int64_t>(n, (Ihi + 1) * kT);
    const int64_t ntiles = ctx->t1 - ctx->t0;

    // Narrowest width whose range can hold the diameter (ecc0 <= diam <= 2 ecc0):
    // the first width with max >= ecc0 is tried (a later attempt widens on
    // overflow); hop_bits forces a minimum width.
    int hb = 0;
    const int min_hb = ctx->p.hop_bits >= 16 ? 2 : (ctx->p.hop_bits >= 8 ? 1 : 0);
    while (hb < 2 && (hb < min_hb || ecc0 > hb_max_hop(hb))) ++hb;
    fdl_status st = FDL_OK;
    for (int attempt = 0; attempt < 3; ++attempt) {
        ctx->hb = hb;
        const size_t dbytes = (size_t)std::max<int64_t>(ntiles, 1) * (size_t)tile_bytes(hb);
        if (ctx->D) {
            cudaFree(ctx->D);
            ctx->allocs.erase(std::find(ctx->allocs.begin(), ctx->allocs.end(), (void*)ctx->D));
            ctx->device_bytes -= ctx->hop_bytes_total;
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
        ctx->hop_bytes_total = dbytes;
        setup_trace(ctx, "hop tiles allocated");
        FDL_CUDA(cudaMemsetAsync(ctx->D, 0, dbytes, ctx->stream));
        setup_trace(ctx, "hop tiles zeroed");
        const int maxhop = hb_max_hop(hb);
        // levels per batch: every BFS ends within diam <= 2 ecc(0) levels; one level past the
        // width's maximum detects an overflow.  The loop runs on the device (level flags),
        // with one host sync after all batches (MS-BFS)
        const int nlev = std::max(1, std::min(2 * ecc0, maxhop + 1));
        // high-diameter graphs: clustered batches of 4096 sources (compact graph
        // neighbourhoods), per-vertex frontier flags and a scattered store into the tiles
        // (id-contiguous batches spread their wavefronts over the whole graph: every vertex
        // gathers at every level; a quarter of the batches is a quarter of the levels).
        // Low-diameter graphs keep id-contiguous 1024-source batches and the tiled store (the
        // whole graph is within a few levels of any batch anyway)
        static const int cl_min_ecc = getenv("FDL_BFS_CLUSTER_ECC") ? atoi(getenv("FDL_BFS_CLUSTER_ECC")) : 24;
        const bool clustered = ecc0 >= cl_min_ecc && src_hi - src_lo > 32 * kBFSWords;
        const int bsrc = clustered ? 32 * kBfsWideWords : 32 * kBFSWords;  // sources per batch
        const int64_t rb = (int64_t)bfs_row_bytes_host(hb) * (bsrc / (32 * kBFSWords));  // batch bytes / vertex
        uint8_t* bbuf = nullptr;
        unsigned int* flags = nullptr;
        const size_t bbytes = (size_t)n * (size_t)rb;
        FDL_CUDA(tmp.alloc(&bbuf, bbytes));
        FDL_CUDA(tmp.alloc(&flags, sizeof(unsigned int) * (size_t)(nlev + 2)));
        FDL_CUDA(cudaMemsetAsync(&ctx->sc->bfs_diam, 0, sizeof(int), ctx->stream));
        FDL_CUDA(cudaMemsetAsync(&ctx->sc->bfs_overflow, 0, sizeof(int), ctx->stream));
        FDL_CUDA(cudaMemsetAsync(&ctx->sc->bfs_bytes, 0, sizeof(unsigned long long), ctx->stream));
        static const int grid_mult = getenv("FDL_BFS_GRID") ? atoi(getenv("FDL_BFS_GRID")) : 8;  // A/B knob
        const int grid = ctx->sm_count * std::max(1, grid_mult);
        // hubs (degree > kBfsHubDeg): a block each per level
        std::vector<int> hub_list;
        static const bool no_hubs = getenv("FDL_BFS_NO_HUBS") != nullptr;  // A/B of the hub blocks
        for (int v = 0; v < n && !no_hubs; ++v)
            if (rp[v + 1] - rp[v] > kBfsHubDeg) hub_list.push_back(v);
        int* d_hubs = nullptr;
        if (!hub_list.empty()) {
            FDL_CUDA(tmp.alloc(&d_hubs, sizeof(int) * hub_list.size()));
            FDL_CUDA(cudaMemcpyAsync(d_hubs, hub_list.data(), sizeof(int) * hub_list.size(), cudaMemcpyHostToDevice,
                                     ctx->stream));
        }
        const int nhub = (int)hub_list.size();
        std::vector<int> order;
        int* d_srcs = nullptr;
        uint8_t *fl_a = nullptr, *fl_b = nullptr;
        uint32_t *wa = nullptr, *wb = nullptr, *wv = nullptr;  // 128-word frontier / visited sets
        const size_t wmasks = (size_t)n * kBfsWideWords;
        if (clustered) {
            // compact words: C4 ideal distances 0.40 -> 0.365 s
            static const bool no_words = getenv("FDL_BFS_NO_WORDS") != nullptr;  // A/B knob
            order = cluster_sources(n, rp, col, src_lo, src_hi, bsrc, !no_words);
            FDL_CUDA(tmp.alloc(&d_srcs, sizeof(int) * order.size()));
            FDL_CUDA(cudaMemcpyAsync(d_srcs, order.data(), sizeof(int) * order.size(), cudaMemcpyHostToDevice,
                                     ctx->stream));
            FDL_CUDA(tmp.alloc(&fl_a, (size_t)n));
            FDL_CUDA(tmp.alloc(&fl_b, (size_t)n));
            FDL_CUDA(tmp.alloc(&wa, wmasks * 4));
            FDL_CUDA(tmp.alloc(&wb, wmasks * 4));
            FDL_CUDA(tmp.alloc(&wv, wmasks * 4));
        }
        for (int s0 = src_lo; s0 < src_hi; s0 += bsrc) {
            const int nsrc = std::min(bsrc, src_hi - s0);
            const int* srcs = clustered ? d_srcs + (s0 - src_lo) : nullptr;
            FDL_CUDA(cudaMemsetAsync(bbuf, 0, bbytes, ctx->stream));
            FDL_CUDA(cudaMemsetAsync(flags, 0, sizeof(unsigned int) * (size_t)(nlev + 2), ctx->stream));
            if (clustered) {
                FDL_CUDA(cudaMemsetAsync(wa, 0, wmasks * 4, ctx->stream));
                FDL_CUDA(cudaMemsetAsync(wv, 0, wmasks * 4, ctx->stream));
                FDL_CUDA(cudaMemsetAsync(fl_a, 0, (size_t)n, ctx->stream));
                FDL_LAUNCH(launch_bfs_init_list(wa, wv, fl_a, srcs, nsrc, kBfsWideWords, ctx->stream));
                uint32_t *fin = wa, *fout = wb;
                uint8_t *flin = fl_a, *flout = fl_b;
                for (int level = 1; level <= nlev; ++level) {
                    FDL_LAUNCH(launch_bfs_level_wide(d_rp, d_col, fin, fout, wv, bbuf, n, nsrc, level, hb, flags,
                                                     &ctx->sc->bfs_bytes, grid, flin, flout, ctx->stream));
                    std::swap(fin, fout);
                    std::swap(flin, flout);
                }
            } else {
                FDL_LAUNCH(launch_bfs_init(fa, vis, n, s0, ctx->stream));
                uint32_t *fin = fa, *fout = fb;
                for (int level = 1; level <= nlev; ++level) {
                    FDL_LAUNCH(launch_bfs_level_sym(d_rp, d_col, fin, fout, vis, bbuf, n, nsrc, level, hb, flags,
                                                    &ctx->sc->bfs_bytes, d_hubs, nhub, grid, ctx->stream));
                    std::swap(fin, fout);
                }
            }
            FDL_LAUNCH(launch_bfs_batch_end(flags, nlev, maxhop, &ctx->sc->bfs_diam, &ctx->sc->bfs_overflow,
                                            ctx->stream));
            if (clustered)
                FDL_LAUNCH(launch_bfs_scatter(bbuf, ctx->D, srcs, nsrc, n, ctx->nb, ctx->t0, ctx->t1, hb, rb,
                                              ctx->stream));
            else
                FDL_LAUNCH(launch_bfs_retile(bbuf, ctx->D, n, s0, nsrc, ctx->nb, ctx->t0, ctx->t1, hb, ctx->stream));
        }
        setup_trace(ctx, "MS-BFS batches");
        FDL_CUDA(cudaMemcpyAsync(ctx->sc_host, ctx->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, ctx->stream));
        FDL_CUDA(cudaStreamSynchronize(ctx->stream));
        tmp.release(bbuf);
        tmp.release(flags);
        if (d_hubs) tmp.release(d_hubs);
        if (d_srcs) tmp.release(d_srcs);
        if (fl_a) tmp.release(fl_a);
        if (fl_b) tmp.release(fl_b);
        if (wa) tmp.release(wa);
        if (wb) tmp.release(wb);
        if (wv) tmp.release(wv);
        setup_trace(ctx, "batch buffers freed");
        const bool overflow = ctx->sc_host->bfs_overflow != 0;
        const int diam = ctx->sc_host->bfs_diam;
        ctx->bfs_bytes += ctx->sc_host->bfs_bytes;
        if (!overflow) {
            ctx->diameter = diam;
            if (hb == 0) FDL_LAUNCH(launch_nib_encode(ctx->D, dbytes, ctx->stream));
            setup_trace(ctx, "nibble encode");
            break;
        }
        if (hb == 2) {
            st = set_err(ctx, FDL_E_DIAMETER, "hop count exceeds 65535");
            break;
        }
        ++hb;
    }
    if (st != FDL_OK) return st;
    if (ctx->distributed) {
        // every rank BFSed only its sources: agree on the diameter and hop width (max over ranks)
        int* dd = nullptr;
        FDL_CUDA(tmp.alloc(&dd, sizeof(int) * 2 * ctx->world));
        int mine[2] = {ctx->diameter, ctx->hb};
        FDL_CUDA(cudaMemcpyAsync(dd + 2 * ctx->rank, mine, sizeof mine, cudaMemcpyHostToDevice, ctx->stream));
        fdl_status s2 = allgather_inplace(ctx, dd, 2, ncclInt32, 4);
        std::vector<int> all(2 * ctx->world);
        cudaMemcpyAsync(all.data(), dd, sizeof(int) * 2 * ctx->world, cudaMemcpyDeviceToHost, ctx->stream);
        cudaStreamSynchronize(ctx->stream);
        FDL_TRY(s2);
        for (int g = 0; g < ctx->world; ++g) ctx->diameter = std::max(ctx->diameter, all[2 * g]);
    }
    return FDL_OK;
}

// Weighted graphs / general alpha (NEXT-3): fp64 multi-source Bellman-Ford over
// the CSR with edge lengths (unit lengths when edge_len is NULL), stored as fp32
// path lengths in the local upper-triangle tiles.
fdl_status build_dists(fdl_ctx* ctx, const int64_t* rp, const int32_t* col, const double* edge_len)
{
    const int n = ctx->n;
    const int64_t m = std::max<int64_t>(rp[n], 1);
    int64_t Ilo = 0, Jlo = 0, Ihi = -1, Jhi = 0;
    if (ctx->t1 > ctx->t0) {
        tri_coords(ctx->t0, ctx->nb, Ilo, Jlo);
        tri_coords(ctx->t1 - 1, ctx->nb, Ihi, Jhi);
    }
    const int src_lo = (int)std::min<int64_t>(n, Ilo * kT);
    const int src_hi = (int)std::min<int64_t>(n, (Ihi + 1) * kT);
    // sources per batch: up to kBfMaxChunks chunks of 4096, the fp64 distances within
    // min(24 GB, a third of the free memory); fewer, larger batches mean fewer sweeps in
    // all (a batch takes ~ max distance / delta sweeps however many sources it has)
    static const double budget_gb = getenv("FDL_BF_BUDGET_GB") ? atof(getenv("FDL_BF_BUDGET_GB")) : 24.0;
    size_t free_b = 0, total_b = 0;
    FDL_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const int64_t nsrc_all = std::max(1, src_hi - src_lo);
    const int64_t by_mem = std::min<int64_t>((int64_t)(budget_gb * 1e9), (int64_t)(free_b / 3)) / (8 * (int64_t)n);
    int S;
    if (nsrc_all <= kBfChunk || by_mem < 2 * kBfChunk)
        S = (int)std::max<int64_t>(32, std::min<int64_t>({(nsrc_all + 31) / 32 * 32, (int64_t)kBfChunk, by_mem / 32 * 32}));
    else
        S = kBfChunk * (int)std::min<int64_t>({(int64_t)kBfMaxChunks, (nsrc_all + kBfChunk - 1) / kBfChunk,
                                                by_mem / kBfChunk});
    Scratch tmp;
    int64_t* d_rp = nullptr;
    int32_t* d_col = nullptr;
    double *d_len = nullptr, *da = nullptr, *dmax = nullptr;
    FDL_CUDA(tmp.alloc(&d_rp, sizeof(int64_t) * (n + 1)));
    FDL_CUDA(tmp.alloc(&d_col, sizeof(int32_t) * m));
    FDL_CUDA(tmp.alloc(&d_len, sizeof(double) * m));
    FDL_CUDA(tmp.alloc(&da, sizeof(double) * (size_t)n * S));
    // per (vertex, source) change bits of the last sweep, double-buffered
    const int W = S / 32;
    uint32_t *chg_a = nullptr, *chg_b = nullptr;
    uint16_t *pend_a = nullptr, *pend_b = nullptr;
    unsigned int* flags = nullptr;
    constexpr int kChunk = 16;  // sweeps enqueued between host checks
    // Delta-stepping threshold: sweep t propagates only distances <= (t + 1) delta, so a
    // value is rarely passed on before it is final; delta = 2 x the mean edge length
    double sum_len = 0.0;
    for (int64_t e = 0; e < rp[n]; ++e) sum_len += edge_len ? edge_len[e] : 1.0;
    // A/B knob; W4: 2 -> 3.08 s, 1 -> 3.46 s, plain Bellman-Ford (1e30) -> 3.40 s
    static const double dmult = getenv("FDL_BF_DELTA") ? atof(getenv("FDL_BF_DELTA")) : 2.0;
    const double delta = rp[n] > 0 ? dmult * sum_len / (double)rp[n] : 1.0;
    const int max_sweeps = (int)std::min<int64_t>(INT32_MAX - kChunk, 4 * (int64_t)n + rp[n] + 8);
    FDL_CUDA(tmp.alloc(&chg_a, sizeof(uint32_t) * (size_t)n * W));
    FDL_CUDA(tmp.alloc(&chg_b, sizeof(uint32_t) * (size_t)n * W));
    FDL_CUDA(tmp.alloc(&pend_a, sizeof(uint16_t) * (size_t)n));
    FDL_CUDA(tmp.alloc(&pend_b, sizeof(uint16_t) * (size_t)n));
    FDL_CUDA(tmp.alloc(&flags, sizeof(unsigned int) * (size_t)(max_sweeps + kChunk)));
    FDL_CUDA(tmp.alloc(&dmax, sizeof(double)));
    FDL_CUDA(cudaMemsetAsync(dmax, 0, sizeof(double), ctx->stream));
    std::vector<double> ones;
    const double* lens = edge_len;
    if (!lens) {
        ones.assign((size_t)m, 1.0);
        lens = ones.data();
    }
    FDL_CUDA(cudaMemcpyAsync(d_rp, rp, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, ctx->stream));
    if (rp[n] > 0) {
        FDL_CUDA(cudaMemcpyAsync(d_col, col, sizeof(int32_t) * rp[n], cudaMemcpyHostToDevice, ctx->stream));
        FDL_CUDA(cudaMemcpyAsync(d_len, lens, sizeof(double) * rp[n], cudaMemcpyHostToDevice, ctx->stream));
    }
    ctx->hb = kHbDist;
    const size_t dbytes = (size_t)std::max<int64_t>(ctx->t1 - ctx->t0, 1) * (size_t)tile_bytes(kHbDist);
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, dbytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_err(ctx, FDL_E_OOM, "distance tile allocation of " + std::to_string(dbytes) + " bytes failed");
    }
    ctx->D = static_cast<uint8_t*>(q);
    ctx->allocs.push_back(q);
    ctx->device_bytes += dbytes;
    ctx->hop_bytes_total = dbytes;
    FDL_CUDA(cudaMemsetAsync(ctx->D, 0, dbytes, ctx->stream));
    // Source batches as compact graph neighbourhoods: clusters of up to S sources of
    // this rank's range, each grown by BFS (over vertices not yet taken) from the first
    // untaken vertex.  Sources close to each other have nearly concentric wavefronts,
    // so each sweep's change words are dense (many sources per vertex at once) instead
    // of one bit per 32-lane word (measured: W4 setup 6.2 s with id-contiguous batches).
    // compact words: W4 distances 2.2 -> 1.4-1.6 s
    static const bool no_words = getenv("FDL_BF_NO_WORDS") != nullptr;  // A/B knob
    const std::vector<int> order = cluster_sources(n, rp, col, src_lo, src_hi, S, !no_words);
    int* d_srcs = nullptr;
    FDL_CUDA(tmp.alloc(&d_srcs, sizeof(int) * std::max<size_t>(order.size(), 1)));
    if (!order.empty())
        FDL_CUDA(cudaMemcpyAsync(d_srcs, order.data(), sizeof(int) * order.size(), cudaMemcpyHostToDevice,
                                 ctx->stream));
    for (int b0 = 0; b0 < (int)order.size(); b0 += S) {
        const int nsrc = std::min(S, (int)order.size() - b0);
        const int* srcs = d_srcs + b0;
        FDL_LAUNCH(launch_bf_init(da, n, srcs, nsrc, S, ctx->stream));
        FDL_CUDA(cudaMemsetAsync(chg_a, 0, sizeof(uint32_t) * (size_t)n * W, ctx->stream));
        FDL_CUDA(cudaMemsetAsync(pend_a, 0, sizeof(uint16_t) * (size_t)n, ctx->stream));
        FDL_CUDA(cudaMemsetAsync(flags, 0, sizeof(unsigned int) * (size_t)(max_sweeps + kChunk), ctx->stream));
        FDL_LAUNCH(launch_bf_seed(chg_a, pend_a, srcs, nsrc, S, ctx->stream));
        uint32_t *cin = chg_a, *cout = chg_b;
        uint16_t *pin = pend_a, *pout = pend_b;
        // sweeps on the device, kChunk between host checks of the last sweep's flag
        // (a sweep after one without changes returns at once)
        bool done = false;
        for (int it = 0; it < max_sweeps && !done; it += kChunk) {
            for (int k = 0; k < kChunk; ++k) {
                FDL_LAUNCH(launch_bf_sweep(d_rp, d_col, d_len, da, cin, cout, pin, pout, n, S, nsrc, it + k, delta,
                                           flags, ctx->sm_count * 8, ctx->stream));
                std::swap(cin, cout);
                std::swap(pin, pout);
            }
            unsigned int last = 1;
            FDL_CUDA(cudaMemcpyAsync(&last, flags + it + kChunk - 1, sizeof(unsigned int), cudaMemcpyDeviceToHost,
                                     ctx->stream));
            FDL_CUDA(cudaStreamSynchronize(ctx->stream));
            done = last == 0u;
        }
        FDL_LAUNCH(launch_bf_store(da, n, srcs, nsrc, S, ctx->nb, ctx->t0, ctx->t1, ctx->D, dmax, ctx->stream));
    }
    double mx = 0.0;
    FDL_CUDA(cudaMemcpyAsync(&mx, dmax, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    FDL_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->diameter = (int)std::ceil(mx);
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
    if (!std::isfinite(p->weight_exp)) {
        msg = "weight_exp must be finite (w = d^alpha)";
        return FDL_E_INVALID_ARG;
    }
    if (p->strategy == FDL_STRAT_ENUM) {
        if (p->enum_count < 1 || p->enum_count > kEnumMax || !(p->enum_step > 0.0) || !std::isfinite(p->enum_step)) {
            msg = "enum_count must be in 1..32 and enum_step > 0";
            return FDL_E_INVALID_ARG;
        }
        if (std::isfinite(p->step)) {
            msg = "the enumerating strategy does not take a step cap";
            return FDL_E_UNSUPPORTED;
        }
    }
    if (p->cg_extrap < 0 || p->cg_extrap > 2) {
        msg = "cg_extrap must be 0, 1 or 2";
        return FDL_E_INVALID_ARG;
    }
    if (p->cg_history < 0 || p->cg_history > kGalMax) {
        msg = "cg_history must be in 0..8";
        return FDL_E_INVALID_ARG;
    }
    if (p->strategy != FDL_STRAT_FIXED && p->strategy != FDL_STRAT_PROB && p->strategy != FDL_STRAT_ENUM) {
        msg = "unknown strategy";
        return FDL_E_INVALID_ARG;
    }
    return FDL_OK;
}

// Work items of the local tile range: strip segments of <= seg_len(nb) tiles.
void build_items(fdl_ctx* ctx, std::vector<int4>& items, std::vector<int>& lo, std::vector<int>& hi)
{
    const int64_t nb = ctx->nb;
    lo.assign(nb, 0);
    hi.assign(nb, 0);
    std::vector<char> seen(nb, 0);
    int64_t t = ctx->t0;
    ctx->local_pairs = 0;
    while (t < ctx->t1) {
        int64_t I, J;
        tri_coords(t, nb, I, J);
        const int64_t strip_end = tri_index(I, nb - 1, nb) + 1;
        const int64_t nt = std::min<int64_t>({(int64_t)seg_len(nb), strip_end - t, ctx->t1 - t});
        if (!seen[I]) {
            seen[I] = 1;
            lo[I] = (int)items.size();
        }
        items.push_back(make_int4((int)I, (int)J, (int)nt, (int)(t - ctx->t0)));
        hi[I] = (int)items.size();
        const int64_t mi = std::min<int64_t>(kT, ctx->n - I * kT);
        for (int64_t j = J; j < J + nt; ++j) {
            const int64_t mj = std::min<int64_t>(kT, ctx->n - j * kT);
            ctx->local_pairs += (j == I) ? (uint64_t)(mi * (mi - 1) / 2) : (uint64_t)(mi * mj);
        }
        t += nt;
    }
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
    if (edge_len) {  // lengths positive and finite, equal in both directions
        for (int32_t v = 0; v < n; ++v)
            for (int64_t e = rp[v]; e < rp[v + 1]; ++e) {
                if (!(edge_len[e] > 0.0) || !std::isfinite(edge_len[e]))
                    return set_err(ctx, FDL_E_BAD_LENGTH, "edge lengths must be finite and > 0");
            }
    }
    if (world < 1 || rank < 0 || rank >= world) return set_err(ctx, FDL_E_INVALID_ARG, "bad rank/world");
    int ecc0 = 0;
    st = validate_graph(n, rp, col, msg, ecc0);
    if (st != FDL_OK) return set_err(ctx, st, msg);
    if (edge_len) {  // the two stored directions of an edge carry the same length
        for (int32_t v = 0; v < n; ++v)
            for (int64_t e = rp[v]; e < rp[v + 1]; ++e) {
                const int32_t u = col[e];
                if (u < v) continue;  // each undirected edge once, from its smaller endpoint
                int64_t r = -1;
                for (int64_t f = rp[u]; f < rp[u + 1]; ++f)
                    if (col[f] == v) {
                        r = f;
                        break;
                    }
                if (r < 0 || edge_len[r] != edge_len[e])
                    return set_err(ctx, FDL_E_BAD_LENGTH,
                                   "edge (" + std::to_string(v) + "," + std::to_string(u) +
                                       ") has different lengths in its two directions (S:52)");
            }
    }

    ctx->p = p;
    ctx->n = n;
    ctx->dim = p.dim;
    ctx->rank = rank;
    ctx->world = world;
    ctx->device = p.device;
    ctx->k = p.k > 0 ? p.k : std::pow((double)n, -1.0 / p.dim);
    ctx->alpha = p.weight_exp;
    ctx->general = edge_len != nullptr || p.weight_exp != -2.0;
    ctx->fscale = std::pow(ctx->k, ctx->alpha + 2.0);
    ctx->rscale = std::pow(ctx->k, ctx->alpha + 1.0);
    ctx->dscale = std::pow(ctx->k, ctx->alpha);
    if (ctx->general && p.strategy == FDL_STRAT_ENUM)
        return set_err(ctx, FDL_E_UNSUPPORTED, "the enumerating strategy needs unit lengths and alpha = -2");
    ctx->cap = std::isfinite(p.step) ? p.step / ctx->k : INFINITY;
    // X^{k+1} is the minimiser of Eq. 4 (DESIGN R8): solved to 1e-9 relative residual by
    // default (tighter only for tol < 1e-7).  S:246's 1e-2 tol gives a different, equally
    // valid trajectory on slowly converging inputs (C4 seeds 2-3: 169 / 179 iterations
    // against 160 / 189 for every solve at <= 1e-9)
    if (!(p.cg_rtol > 0)) ctx->p.cg_rtol = std::min(1e-2 * p.tol, 1e-9);
    if (p.cg_history == 0) ctx->p.cg_history = FDL_CG_HISTORY_DEFAULT;
    if (p.cg_max_iter <= 0) ctx->p.cg_max_iter = std::min(10 * n, 10000);
    if (p.a_refresh <= 0) ctx->p.a_refresh = 10;
    if (std::isfinite(p.step)) ctx->p.a_refresh = 1;  // the cap makes Xt non-linear in X^{k+1}
    ctx->rng = p.seed;

    FDL_CUDA(cudaSetDevice(ctx->device));
    FDL_CUDA(cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, ctx->device));
    FDL_CUDA(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
    ctx->stream = ctx->own_stream;

    ctx->emulated = world > 1 && nccl_id == nullptr && ctx->group == nullptr;
    // A communicator is made whenever an id is given, also for world = 1 (a one-rank NCCL
    // run of the distributed path: exercises the NCCL calls on a single GPU).
    if (nccl_id != nullptr && !ctx->group) {
        if (!g_nccl.load(msg)) return set_err(ctx, FDL_E_NCCL, msg);
        ncclUniqueId id;
        memcpy(id.internal, nccl_id, 128);
        ncclResult_t r = g_nccl.CommInitRank(&ctx->comm, world, id, rank);
        if (r != 0)
            return set_err(ctx, FDL_E_NCCL, std::string("ncclCommInitRank: ") +
                                                 (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?"));
    }
    ctx->distributed = ctx->comm != nullptr || ctx->group != nullptr;

    // ---- geometry: tiles of kT x kT, this rank's share of the triangle
    ctx->nb = (n + kT - 1) / kT;
    ctx->npad = (int64_t)ctx->nb * kT;
    fdl_shard_tiles(n, world, rank, &ctx->t0, &ctx->t1);
    if (ctx->t1 > ctx->t0) {
        int64_t a, b;
        tri_coords(ctx->t0, ctx->nb, a, b);
        ctx->Ilo = (int)a;
        tri_coords(ctx->t1 - 1, ctx->nb, a, b);
        ctx->Ihi = (int)a;
    }
    std::vector<int4> items;
    std::vector<int> lo, hi;
    build_items(ctx, items, lo, hi);
    ctx->nitems = (int)items.size();
    ctx->nblk = (int)((ctx->npad + kRB - 1) / kRB);
    const int dim = ctx->dim;
    const size_t vn = (size_t)ctx->npad * dim;
    const int64_t ntiles = ctx->t1 - ctx->t0;
    const int Cmax = 2 * dim;

    FDL_ALLOC(ctx->sc, 1);
    FDL_CUDA(cudaMemsetAsync(ctx->sc, 0, sizeof(DevScalars), ctx->stream));
    FDL_CUDA(cudaHostAlloc(&ctx->hs, sizeof(HostScalars), cudaHostAllocMapped));
    FDL_CUDA(cudaHostGetDevicePointer((void**)&ctx->hs_dev, ctx->hs, 0));
    FDL_CUDA(cudaHostAlloc(&ctx->sc_host, sizeof(DevScalars), cudaHostAllocDefault));
    memset(ctx->sc_host, 0, sizeof(DevScalars));
    FDL_ALLOC(ctx->items, std::max(ctx->nitems, 1));
    FDL_ALLOC(ctx->it_lo, ctx->nb);
    FDL_ALLOC(ctx->it_hi, ctx->nb);
    FDL_ALLOC(ctx->jpart, (size_t)std::max<int64_t>(ntiles, 1) * kT * Cmax);
    FDL_ALLOC(ctx->ipart, (size_t)std::max(ctx->nitems, 1) * 8 * kT * Cmax);
    FDL_ALLOC(ctx->spart, (size_t)std::max(ctx->nitems, 1) * 8 * 2);
    FDL_ALLOC(ctx->sparts, (size_t)2 * world);
    FDL_ALLOC(ctx->stress_scratch, (size_t)sym_stress_chunks(std::max(ctx->nitems, 1) * 8) * kEnumNC);
    if (p.strategy == FDL_STRAT_ENUM) {
        if (world > 1 || ctx->distributed)
            return set_err(ctx, FDL_E_UNSUPPORTED, "the enumerating strategy runs on one GPU");
        FDL_ALLOC(ctx->spart_enum, (size_t)std::max(ctx->nitems, 1) * kEnumNC);
        // candidate passes write kEnumNC stresses each at enum_f + c0 (c0 a multiple of
        // kEnumNC), so the buffer holds kEnumMax rounded up to whole passes
        FDL_ALLOC(ctx->enum_f, (size_t)((kEnumMax + kEnumNC - 1) / kEnumNC) * kEnumNC);
    }
    if (ctx->distributed) {
        ctx->rslice = (ctx->npad + world - 1) / world;
        FDL_ALLOC(ctx->rparts, (size_t)world * ctx->rslice * Cmax);
        FDL_ALLOC(ctx->xrecv, (size_t)world * ctx->rslice * Cmax);
        FDL_ALLOC(ctx->xgath, (size_t)world * (ctx->rslice * Cmax + 2));
        FDL_CUDA(cudaMemsetAsync(ctx->rparts, 0, sizeof(double) * (size_t)world * ctx->rslice * Cmax, ctx->stream));
    }
    FDL_ALLOC(ctx->diag, (size_t)ctx->npad);
    FDL_ALLOC(ctx->Xk, vn);
    FDL_ALLOC(ctx->Xn, vn);
    FDL_ALLOC(ctx->Xt, vn);
    FDL_ALLOC(ctx->Rk, vn);
    FDL_ALLOC(ctx->R1, vn);
    FDL_ALLOC(ctx->R2, vn);
    FDL_ALLOC(ctx->cr, vn);
    FDL_ALLOC(ctx->cz, vn);
    FDL_ALLOC(ctx->cp, vn);
    FDL_ALLOC(ctx->cy, vn);
    FDL_ALLOC(ctx->Ak, vn);
    FDL_ALLOC(ctx->An, vn);
    FDL_ALLOC(ctx->At, vn);
    FDL_ALLOC(ctx->Xprev, vn);
    FDL_ALLOC(ctx->Aprev, vn);
    if (ctx->p.cg_extrap == 2) {
        const int m = ctx->p.cg_history;
        FDL_ALLOC(ctx->Vh, (size_t)m * vn);
        FDL_ALLOC(ctx->AVh, (size_t)m * vn);
        FDL_ALLOC(ctx->blk_gal, (size_t)3 * kGalNV * ctx->nblk);
        FDL_CUDA(cudaMemsetAsync(ctx->Vh, 0, (size_t)m * vn * sizeof(double), ctx->stream));
        FDL_CUDA(cudaMemsetAsync(ctx->AVh, 0, (size_t)m * vn * sizeof(double), ctx->stream));
        FDL_CUDA(cudaMemcpyAsync(&ctx->sc->gal_m, &m, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
        FDL_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    FDL_ALLOC(ctx->posf, (size_t)ctx->npad * 8);
    FDL_ALLOC(ctx->pvec, (size_t)ctx->npad * 4);
    FDL_ALLOC(ctx->blk_max, (size_t)ctx->nblk);
    FDL_ALLOC(ctx->blk_cg, (size_t)16 * ctx->nblk);
    FDL_ALLOC(ctx->pin_slots, 4);
    FDL_CUDA(cudaMemsetAsync(ctx->posf, 0, (size_t)ctx->npad * 8 * sizeof(float), ctx->stream));
    FDL_CUDA(cudaMemsetAsync(ctx->pvec, 0, (size_t)ctx->npad * 4 * sizeof(float), ctx->stream));
    FDL_CUDA(cudaMemsetAsync(ctx->Xk, 0, vn * sizeof(double), ctx->stream));
    FDL_CUDA(cudaMemsetAsync(ctx->Xprev, 0, vn * sizeof(double), ctx->stream));
    FDL_CUDA(cudaMemsetAsync(ctx->Aprev, 0, vn * sizeof(double), ctx->stream));
    FDL_CUDA(cudaMemsetAsync(ctx->blk_cg, 0, (size_t)16 * ctx->nblk * sizeof(double), ctx->stream));
    if (ctx->nitems > 0)
        FDL_CUDA(cudaMemcpyAsync(ctx->items, items.data(), sizeof(int4) * items.size(), cudaMemcpyHostToDevice,
                                 ctx->stream));
    FDL_CUDA(cudaMemcpyAsync(ctx->it_lo, lo.data(), sizeof(int) * ctx->nb, cudaMemcpyHostToDevice, ctx->stream));
    FDL_CUDA(cudaMemcpyAsync(ctx->it_hi, hi.data(), sizeof(int) * ctx->nb, cudaMemcpyHostToDevice, ctx->stream));

    // hop matrix first (fixes the hop width), then grids, then the Jacobi diagonal
    setup_trace(ctx, "create: buffers");
    const auto td0 = std::chrono::steady_clock::now();
    if (ctx->general)
        FDL_TRY(build_dists(ctx, rp, col, edge_len));
    else
        FDL_TRY(build_hops(ctx, rp, col, ecc0));
    ctx->setup_dist_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - td0).count();
    setup_trace(ctx, "ideal distances");
    const int cap_items = std::max(ctx->nitems, 1);
    for (int s = 1; s <= 2; ++s)
        ctx->grid_p1[s] = std::max(1, std::min(cap_items, ctx->sm_count * sym_max_ctas(kSymP1, dim, s, ctx->hb)));
    ctx->grid_p2 = std::max(1, std::min(cap_items, ctx->sm_count * sym_max_ctas(kSymP2, dim, 1, ctx->hb)));
    ctx->grid_diag = std::max(1, std::min(cap_items, ctx->sm_count * sym_max_ctas(kSymDiag, dim, 1, ctx->hb)));
    ctx->grid_enum = std::max(1, std::min(cap_items, ctx->sm_count * 2));
    ctx->grid_p1s = std::max(1, std::min(cap_items, ctx->sm_count * sym_max_ctas(kSymP1S, dim, 2, ctx->hb)));
    if (!ctx->general) {
        ctx->grid_p1a = std::max(1, std::min(cap_items, ctx->sm_count * sym_max_ctas(kSymP1A, dim, 1, ctx->hb)));
        ctx->grid_p1r = std::max(1, std::min(cap_items, ctx->sm_count * sym_max_ctas(kSymP1R, dim, 1, ctx->hb)));
    }
    FDL_TRY(build_item_orders(ctx, items));
    // large problems: the extra host sync of the split P1 is negligible against the pass
    ctx->use_graphs = ctx->p.use_graphs == 1 || (ctx->p.use_graphs < 0 && !ctx->distributed && (int64_t)n * n < (int64_t)1 << 30);
    ctx->p1_split = !ctx->general && (ctx->p.p1_split == 1 || ctx->p.p1_split == 2 ||
                                      (ctx->p.p1_split < 0 && (int64_t)n * n >= (int64_t)1 << 30));
    ctx->p1_predict = ctx->p1_split && ctx->p.p1_split != 1;
    // Jacobi diagonal sum_{j != i} w'_ij (one symmetric DIAG pass) and sigma = mean(diag)/n
    FDL_TRY(run_sym(ctx, kSymDiag, 1, ctx->posf, ctx->diag, nullptr, 0));
    FDL_LAUNCH(launch_set_sigma_rows(ctx->diag, ctx->n, ctx->sc, ctx->stream));
    setup_trace(ctx, "Jacobi diagonal");

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
    setup_trace(ctx, "positions + first evaluation");
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
constexpr int kTailBlocks = 8;  // fused PCG tail for n <= 8 * 256 rows (one block is slower beyond)

// ---- the three phases of one Algorithm-2 iteration (enqueue only; the eager
// step syncs between them, the graph step captures them once).
struct StepShape {
    bool refresh;
    bool enumerate;
    int nsets;
    double omega;
};

// every step refreshes L^W X^k: Xt is then not a scalar combination of carried products
bool always_refresh(const fdl_ctx* ctx) { return ctx->p.a_refresh <= 1 || ctx->omega_v != nullptr; }

// line 4, start: L^W X^k (carried or a refresh pass), PCG start and first residual
fdl_status enqueue_prologue(fdl_ctx* ctx, const StepShape& sh, unsigned long long cond)
{
    const int dim = ctx->dim, n = ctx->n, pq = ps_p2(dim);
    const bool refresh = sh.refresh;
    cudaStream_t s = ctx->stream;
    FDL_LAUNCH3(launch_cg_begin(ctx->Xk, ctx->Xn, ctx->pvec, n, 0, dim, pq, ctx->sc, ctx->blk_cg, s));
    if (refresh) FDL_TRY(run_sym(ctx, kSymP2, 1, ctx->pvec, ctx->Ak, nullptr, 0));
    const double* y0 = ctx->Ak;
    if (ctx->p.cg_extrap == 2) {  // recycled start (R27): x0 into Xn, L^W x0 into cy
        // history when every step refreshes A^k (per-vertex omega, step cap, a_refresh = 1):
        // the last step's X^k - X^{k-1} with the difference of the two fresh products
        // (Xprev/Aprev were set by k_rho at the end of the last step)
        if (ctx->ext_ok && always_refresh(ctx))
            FDL_LAUNCH(launch_gal_push(ctx->Xk, ctx->Xprev, ctx->Ak, ctx->Aprev, ctx->Vh, ctx->AVh, n, dim,
                                       ctx->p.cg_history, s));
        FDL_LAUNCH(launch_gal_start(ctx->Vh, ctx->AVh, ctx->Rk, ctx->Xk, ctx->Ak, ctx->Xn, ctx->cy, ctx->blk_gal,
                                    ctx->nblk, ctx->sc, n, dim, s));
        ctx->stats.launches += 2;
        y0 = ctx->cy;
    } else if (ctx->p.cg_extrap) {  // extrapolated start (R23): x0 into Xn, L^W x0 into cy
        // not right after a refresh of carried products: A^k - A^{k-1} would then hold the
        // whole accumulated drift of A^{k-1}, and the start would feed it back (x0 = X^k there)
        const bool ok = ctx->ext_ok && (!refresh || always_refresh(ctx));
        FDL_LAUNCH(launch_extrap(ctx->Xk, ctx->Xprev, ctx->Ak, ctx->Aprev, ctx->Xn, ctx->cy, ctx->sc, n, dim,
                                 ok ? 1 : 0, s));
        y0 = ctx->cy;
    }
    FDL_LAUNCH(launch_cg_init(y0, ctx->Rk, ctx->diag, ctx->cr, ctx->cz, ctx->cp, ctx->pvec, ctx->blk_cg, ctx->nblk,
                              n, dim, pq, s));
    FDL_LAUNCH(launch_cg_finalize(ctx->blk_cg, ctx->nblk, dim, 0, ctx->p.cg_rtol, ctx->sc, ctx->hs_dev, s, cond,
                                  cond != 0, ctx->p.cg_max_iter));
    FDL_LAUNCH(launch_stage_p(ctx->cp, ctx->pvec, ctx->sc, n, dim, pq, s));
    return FDL_OK;
}

// one PCG iteration: a P2 pass (L^W p) and the fp64 vector updates
fdl_status enqueue_cg_body(fdl_ctx* ctx, unsigned long long cond)
{
    const int dim = ctx->dim, n = ctx->n, pq = ps_p2(dim);
    cudaStream_t s = ctx->stream;
    if (ctx->nblk <= kTailBlocks) {
        // small n: the vector part of the iteration in one block (bitwise the same sequence)
        FDL_TRY(run_sym(ctx, kSymP2, 1, ctx->pvec, ctx->cy, nullptr, 0, false));
        FDL_LAUNCH(launch_cg_tail(ctx->cy, ctx->pvec, ctx->diag, ctx->Xn, ctx->cr, ctx->cz, ctx->cp, ctx->pvec,
                                  ctx->blk_cg, n, dim, (n + kRB - 1) / kRB, pq, ctx->p.cg_rtol, ctx->sc, ctx->hs_dev,
                                  s, cond, cond != 0, ctx->p.cg_max_iter));
        return FDL_OK;
    }
    FDL_TRY(run_sym(ctx, kSymP2, 1, ctx->pvec, ctx->cy, nullptr, 0));
    FDL_LAUNCH(launch_cg_ap(ctx->cp, ctx->cy, ctx->blk_cg, ctx->nblk, n, dim, ctx->sc, s));
    FDL_LAUNCH(launch_cg_finalize(ctx->blk_cg, ctx->nblk, dim, 1, ctx->p.cg_rtol, ctx->sc, ctx->hs_dev, s));
    FDL_LAUNCH(launch_cg_update(ctx->Xn, ctx->cr, ctx->cz, ctx->cp, ctx->cy, ctx->diag, ctx->blk_cg, ctx->nblk,
                                ctx->sc, n, 0, dim, s));
    FDL_LAUNCH(launch_cg_finalize(ctx->blk_cg, ctx->nblk, dim, 2, ctx->p.cg_rtol, ctx->sc, ctx->hs_dev, s, cond,
                                  cond != 0, ctx->p.cg_max_iter));
    FDL_LAUNCH(launch_cg_p(ctx->cp, ctx->cz, ctx->pvec, ctx->sc, n, 0, dim, pq, s));
    return FDL_OK;
}

// lines 5-8: pin, combine (Eq. 10), the line-6 pass and the guard
fdl_status enqueue_epilogue(fdl_ctx* ctx, const StepShape& sh)
{
    const int dim = ctx->dim, n = ctx->n, pq = ps_p2(dim);
    const bool enumerate = sh.enumerate;
    const int nsets = sh.nsets;
    const double omega = sh.omega;
    const int ps = ps_p1(dim, nsets);
    cudaStream_t s = ctx->stream;
    // carried L^W X^{k+1} and L^W Xt (before Rk is replaced by the select)
    FDL_LAUNCH(launch_carry_a(ctx->Rk, ctx->cr, ctx->Ak, ctx->An, ctx->At, ctx->sc, n, dim, enumerate ? 0.0 : omega,
                              s));
    // ---- pin x_0 = 0, then line 5: Xt = (1+w) X^{k+1} - w X^k (Eq. 10)
    FDL_LAUNCH(launch_get_pin(ctx->Xn, ctx->pin_slots, 0, dim, 1, s));
    if (enumerate) {
        // lines 286-288: stress of every candidate w_c in multi-candidate passes over
        // the hop tiles, omega* = first argmin, then stress + R of X~(omega*)
        FDL_LAUNCH(launch_enum_stage(ctx->Xk, ctx->Xn, ctx->posf, ctx->blk_max, ctx->pin_slots, n, dim, 2 * pq, s));
        if (ctx->p.cg_extrap)
            FDL_LAUNCH2(launch_rho(ctx->Xn, ctx->Xk, ctx->Xprev, ctx->Ak, ctx->Aprev, ctx->blk_cg, n, dim,
                                  ctx->ext_ok ? 1 : 0, ctx->sc, s));
        const int m = ctx->p.enum_count;
        for (int c0 = 0; c0 < m; c0 += kEnumNC) {
            EnumOmegas w;
            for (int k = 0; k < kEnumNC; ++k) w.w[k] = (float)(ctx->p.enum_step * std::min(c0 + k, m - 1));
            SymArgs a;
            a.D = ctx->D;
            a.pos = ctx->posf;
            a.jpart = nullptr;
            a.ipart = nullptr;
            a.spart = ctx->spart_enum;
            a.items = ctx->items;
            a.order = item_order(ctx, ctx->grid_enum);
            a.nitems = ctx->nitems;
            a.n = ctx->n;
            a.ntiles = ctx->t1 - ctx->t0;
            a.nstage = ctx->npad;
            a.magic = 0x4B000000u;
            if (ctx->nitems > 0 && !a.order) return set_err(ctx, FDL_E_STATE, "no work-item schedule for the grid");
            if (ctx->nitems > 0) FDL_LAUNCH(launch_enum(a, w, dim, ctx->hb, ctx->grid_enum, s));
            FDL_LAUNCH2(launch_sym_stress(ctx->spart_enum, ctx->nitems, kEnumNC, ctx->enum_f + c0, ctx->stress_scratch, s));
        }
        FDL_LAUNCH(launch_enum_pick(ctx->enum_f, m, ctx->p.enum_step, ctx->sc, s));
        FDL_LAUNCH(launch_enum_apply(ctx->Xn, ctx->Xk, ctx->An, ctx->Ak, ctx->Xt, ctx->At, ctx->posf, ctx->sc, n, dim,
                                     ps_p1(dim, 1), s));
        FDL_TRY(run_sym(ctx, kSymP1, 1, ctx->posf, ctx->R1, nullptr, 0));
        // X^{k+1} <- X~(omega*) (omega* = 0 is X^{k+1} itself)
        FDL_LAUNCH(launch_select(ctx->Xk, ctx->Rk, ctx->Xt, ctx->Xt, ctx->R1, ctx->R1, ctx->blk_max, n, dim, 1, ctx->sc,
                                 ctx->Ak, ctx->At, ctx->At, s));
    } else {
        FDL_LAUNCH(launch_combine(ctx->Xk, ctx->Xn, ctx->Xt, ctx->posf, ctx->blk_max, ctx->pin_slots, n, 0, dim, omega,
                                  ctx->omega_v, ctx->cap, nsets, ps, s));
        if (ctx->p.cg_extrap)  // ratio of successive corrections for the next start; X^{k-1} <- X^k
            FDL_LAUNCH2(launch_rho(ctx->Xn, ctx->Xk, ctx->Xprev, ctx->Ak, ctx->Aprev, ctx->blk_cg, n, dim,
                                  ctx->ext_ok ? 1 : 0, ctx->sc, s));
        // ---- line 6: f(Xt), f(X^{k+1}) and the next right-hand side, one fused pass
        if (nsets == 2 && ctx->p1_split && !ctx->p1_fused_now) {
            // stress of both candidates + R(Xt); R(X^{k+1}) only if the guard rejects Xt
            FDL_TRY(run_sym(ctx, kSymP1S, 2, ctx->posf, ctx->R2, nullptr, 0));
            FDL_CUDA(cudaMemcpyAsync(ctx->sc_host, ctx->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, s));
            FDL_CUDA(cudaStreamSynchronize(s));
            if (!(ctx->sc_host->f_set[1] <= ctx->sc_host->f_set[0])) {
                FDL_LAUNCH(launch_stage_pos1(ctx->Xn, ctx->posf, n, 0, dim, ps_p1(dim, 1), s));
                FDL_TRY(run_sym(ctx, kSymP1R, 1, ctx->posf, ctx->R1, nullptr, 0));  // R only: f(X^{k+1}) is known
                ctx->stats.p1_rejected++;
            }
        } else {
            FDL_TRY(run_sym(ctx, kSymP1, nsets, ctx->posf, ctx->R1, ctx->R2, 0));
        }
        // ---- lines 6-8: guard
        FDL_LAUNCH(launch_select(ctx->Xk, ctx->Rk, ctx->Xn, ctx->Xt, ctx->R1, ctx->R2, ctx->blk_max, n, dim, nsets,
                                 ctx->sc, ctx->Ak, ctx->An, ctx->At, s));
    }
    // history with carried products: X^{k+1} - X^k and A^{k+1} - A^k, both from this step
    // (A^{k+1} - A^k = L^W (x0 - X^k) + sum alpha L^W p algebraically, (1 + w) times that
    // for Xt: no carried drift enters the history; a difference against a refreshed A^k
    // would bring the whole accumulated drift in and feed it back through the start)
    if (ctx->p.cg_extrap == 2 && !always_refresh(ctx))
        FDL_LAUNCH(launch_gal_push(ctx->Xk, ctx->Xprev, ctx->Ak, ctx->Aprev, ctx->Vh, ctx->AVh, n, dim,
                                       ctx->p.cg_history, s));
    return FDL_OK;
}

// Stats increments of the captured phases: once per launch, and per PCG iteration.
using StatDelta = StepGraphCounts;
StatDelta stat_snapshot(const fdl_ctx* ctx)
{
    const fdl_stats& t = ctx->stats;
    return {t.launches, t.p1_launches, t.p2_launches, t.p1_pairs, t.p2_pairs, t.p1_pairs_x2, t.p1_pairs_nor};
}
StatDelta stat_diff(const StatDelta& a, const StatDelta& b)
{
    return {b.launches - a.launches, b.p1_launches - a.p1_launches, b.p2_launches - a.p2_launches,
            b.p1_pairs - a.p1_pairs, b.p2_pairs - a.p2_pairs, b.p1_pairs_x2 - a.p1_pairs_x2,
            b.p1_pairs_nor - a.p1_pairs_nor};
}
void stat_add(fdl_ctx* ctx, const StatDelta& d, uint64_t times)
{
    fdl_stats& t = ctx->stats;
    t.launches += d.launches * times;
    t.p1_launches += d.p1_launches * times;
    t.p2_launches += d.p2_launches * times;
    t.p1_pairs += d.p1_pairs * times;
    t.p2_pairs += d.p2_pairs * times;
    t.p1_pairs_x2 += d.p1_pairs_x2 * times;
    t.p1_pairs_nor += d.p1_pairs_nor * times;
}

// Capture one iteration as a CUDA graph: prologue -> WHILE(PCG not converged and
// cg_iters < cg_max) { PCG iteration } -> epilogue -> D2H of the device scalars.
// The WHILE condition is set on the device by k_cg_finalize, so a whole step is
// one graph launch and one host sync (instead of one sync per PCG iteration).
fdl_status build_step_graph(fdl_ctx* ctx, const StepShape& sh, StepGraph& out)
{
    cudaStream_t s = ctx->stream;
    if (!ctx->aux_stream) FDL_CUDA(cudaStreamCreateWithFlags(&ctx->aux_stream, cudaStreamNonBlocking));
    ctx->capturing = true;
    const StatDelta s0 = stat_snapshot(ctx);
    cudaGraph_t g = nullptr;
    auto fail = [&](fdl_status st) {
        ctx->capturing = false;
        ctx->stream = s;
        cudaGraph_t tmp = nullptr;
        cudaStreamEndCapture(s, &tmp);
        if (tmp) cudaGraphDestroy(tmp);
        cudaGetLastError();
        return st;
    };
    FDL_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    cudaStreamCaptureStatus cst;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    if (cudaStreamGetCaptureInfo(s, &cst, nullptr, &g, &deps, &ndeps) != cudaSuccess) return fail(FDL_E_CUDA);
    cudaGraphConditionalHandle h;
    if (cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault) != cudaSuccess) return fail(FDL_E_CUDA);
    fdl_status st = enqueue_prologue(ctx, sh, (unsigned long long)h);
    if (st != FDL_OK) return fail(st);
    const StatDelta s1 = stat_snapshot(ctx);
    if (cudaStreamGetCaptureInfo(s, &cst, nullptr, &g, &deps, &ndeps) != cudaSuccess) return fail(FDL_E_CUDA);
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    if (cudaGraphAddNode(&cnode, g, deps, ndeps, &cp) != cudaSuccess) return fail(FDL_E_CUDA);
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    // body: captured on the auxiliary stream into the WHILE node's graph
    if (cudaStreamBeginCaptureToGraph(ctx->aux_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) !=
        cudaSuccess)
        return fail(FDL_E_CUDA);
    ctx->stream = ctx->aux_stream;
    st = enqueue_cg_body(ctx, (unsigned long long)h);
    ctx->stream = s;
    cudaGraph_t body_out = nullptr;
    const cudaError_t eb = cudaStreamEndCapture(ctx->aux_stream, &body_out);
    if (st != FDL_OK) return fail(st);
    if (eb != cudaSuccess) return fail(FDL_E_CUDA);
    const StatDelta s2 = stat_snapshot(ctx);
    if (cudaStreamUpdateCaptureDependencies(s, &cnode, 1, cudaStreamSetCaptureDependencies) != cudaSuccess)
        return fail(FDL_E_CUDA);
    // lines 5-8 inside an IF node on sc->done: a solve that hit cg_max_iter leaves the
    // context as the eager step does (X^k, R^k, A^k untouched; FDL_E_SOLVER on the host)
    cudaGraphConditionalHandle hif;
    if (cudaGraphConditionalHandleCreate(&hif, g, 0, cudaGraphCondAssignDefault) != cudaSuccess)
        return fail(FDL_E_CUDA);
    if (launch_cond_done(ctx->sc, s, (unsigned long long)hif) != cudaSuccess) return fail(FDL_E_CUDA);
    if (cudaStreamGetCaptureInfo(s, &cst, nullptr, &g, &deps, &ndeps) != cudaSuccess) return fail(FDL_E_CUDA);
    cudaGraphNodeParams ip = {};
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = hif;
    ip.conditional.type = cudaGraphCondTypeIf;
    ip.conditional.size = 1;
    cudaGraphNode_t inode;
    if (cudaGraphAddNode(&inode, g, deps, ndeps, &ip) != cudaSuccess) return fail(FDL_E_CUDA);
    if (cudaStreamBeginCaptureToGraph(ctx->aux_stream, ip.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                      cudaStreamCaptureModeThreadLocal) != cudaSuccess)
        return fail(FDL_E_CUDA);
    ctx->stream = ctx->aux_stream;
    st = enqueue_epilogue(ctx, sh);
    ctx->stream = s;
    cudaGraph_t epi_out = nullptr;
    const cudaError_t ee = cudaStreamEndCapture(ctx->aux_stream, &epi_out);
    if (st != FDL_OK) return fail(st);
    if (ee != cudaSuccess) return fail(FDL_E_CUDA);
    if (cudaStreamUpdateCaptureDependencies(s, &inode, 1, cudaStreamSetCaptureDependencies) != cudaSuccess)
        return fail(FDL_E_CUDA);
    ctx->stats.launches++;  // k_cond_done
    if (cudaMemcpyAsync(ctx->sc_host, ctx->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, s) != cudaSuccess)
        return fail(FDL_E_CUDA);
    const StatDelta s3 = stat_snapshot(ctx);
    ctx->capturing = false;
    cudaGraph_t gout = nullptr;
    FDL_CUDA(cudaStreamEndCapture(s, &gout));
    const cudaError_t ei = cudaGraphInstantiate(&out.exec, gout, 0);
    cudaGraphDestroy(gout);
    FDL_CUDA(ei);
    // counters: the captured launches ran once at capture time; undo, keep the deltas
    out.once = stat_diff(s0, s1);
    const StatDelta e = stat_diff(s2, s3);
    out.once.launches += e.launches;
    out.once.p1_launches += e.p1_launches;
    out.once.p2_launches += e.p2_launches;
    out.once.p1_pairs += e.p1_pairs;
    out.once.p2_pairs += e.p2_pairs;
    out.once.p1_pairs_x2 += e.p1_pairs_x2;
    out.once.p1_pairs_nor += e.p1_pairs_nor;
    out.body = stat_diff(s1, s2);
    fdl_stats& t = ctx->stats;
    t.launches = s0.launches;
    t.p1_launches = s0.p1_launches;
    t.p2_launches = s0.p2_launches;
    t.p1_pairs = s0.p1_pairs;
    t.p2_pairs = s0.p2_pairs;
    t.p1_pairs_x2 = s0.p1_pairs_x2;
    t.p1_pairs_nor = s0.p1_pairs_nor;
    return FDL_OK;
}

fdl_status step_impl(fdl_ctx* ctx, fdl_iter_info* info)
{
    if (ctx->emulated) return set_err(ctx, FDL_E_UNSUPPORTED, "emulated rank: only fdl_eval_partial is available");
    if (ctx->broken) return set_err(ctx, FDL_E_STATE, ctx->err.empty() ? "context is broken" : ctx->err);
    if (ctx->stopped) return set_err(ctx, FDL_E_STATE, "the run has stopped; call fdl_set_positions to restart");
    const bool enumerate = ctx->p.strategy == FDL_STRAT_ENUM;
    double omega = ctx->omega_v ? ctx->omega_v_max : (enumerate ? 0.0 : pick_omega(ctx));
    const int nsets = omega > 0.0 ? 2 : 1;
    cudaStream_t s = ctx->stream;
    // ---- line 4: X^{k+1} = H(X^k): PCG on Eq. 5 (zero-mean gauge, R7), warm start X^k.
    // The warm-start residual needs L^W X^k: carried from the previous solve, or a full
    // P2 pass every a_refresh steps (bounds the fp32 drift of the carried value).
    // per-vertex omega: Xt is not a scalar combination, At cannot be carried
    const bool refresh = !ctx->a_valid || ctx->a_age + 1 >= ctx->p.a_refresh || ctx->omega_v;
    const StepShape sh{refresh, enumerate, nsets, omega};
    // p1_split = 2 (R30): the two-set line-6 pass when a rejection is predicted (the same
    // results as the split pass plus the rejection pass, bitwise; R25)
    ctx->p1_fused_now = ctx->p1_predict && nsets == 2 && !enumerate && ctx->p1_fused_next;
    int cg = 0;
    // graph mode: one launch per step; not with a host decision inside the step
    // (split line 6, enumeration) or host-side exchanges (several ranks)
    bool graph = ctx->use_graphs && !enumerate && !(nsets == 2 && ctx->p1_split) && !ctx->distributed &&
                 ctx->steps_eager > 0;
    const auto key = std::make_tuple((int)refresh, nsets, (int)ctx->ext_ok, omega);
    auto it = ctx->graphs.find(key);
    if (graph && it == ctx->graphs.end()) {
        StepGraph sg;
        if (build_step_graph(ctx, sh, sg) == FDL_OK) {
            it = ctx->graphs.emplace(key, sg).first;
        } else {
            // capture refused (driver without conditional nodes, ...): eager from now on
            fprintf(stderr, "fdl: step graph capture failed (%s); using eager launches\n", ctx->err.c_str());
            cudaGetLastError();
            ctx->use_graphs = false;
            ctx->broken = false;
            ctx->err.clear();
            graph = false;
        }
    }
    const int mstep = mark_begin(ctx, 0);
    if (graph) {
        FDL_CUDA(cudaGraphLaunch(it->second.exec, s));
        mark_end(ctx, mstep);
        FDL_CUDA(cudaStreamSynchronize(s));
        cg = ctx->sc_host->cg_iters;
        stat_add(ctx, it->second.once, 1);
        stat_add(ctx, it->second.body, (uint64_t)cg);
        if (!ctx->sc_host->done) {
            collect_events(ctx);
            return set_err(ctx, FDL_E_SOLVER, "PCG reached cg_max_iter before cg_rtol (S:223)");
        }
    } else {
        FDL_TRY(enqueue_prologue(ctx, sh, 0));
        FDL_CUDA(cudaStreamSynchronize(s));
        while (!ctx->hs->done) {
            if (cg >= ctx->p.cg_max_iter) {
                collect_events(ctx);
                return set_err(ctx, FDL_E_SOLVER, "PCG reached cg_max_iter before cg_rtol (S:223)");
            }
            FDL_TRY(enqueue_cg_body(ctx, 0));
            FDL_CUDA(cudaStreamSynchronize(s));
            ++cg;
        }
        FDL_TRY(enqueue_epilogue(ctx, sh));
        mark_end(ctx, mstep);
        FDL_CUDA(cudaMemcpyAsync(ctx->sc_host, ctx->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, s));
        FDL_CUDA(cudaStreamSynchronize(s));
        ctx->steps_eager++;
    }
    if (refresh)
        ctx->a_age = 0;
    else
        ctx->a_age++;
    ctx->a_valid = true;
    ctx->ext_ok = ctx->p.cg_extrap != 0;
    collect_events(ctx);
    ctx->stats.steps++;
    ctx->stats.cg_iters += cg;

    const DevScalars& h = *ctx->sc_host;
    const double f_before = ctx->f;
    double f_next = h.f_set[0];
    double f_rel = nsets == 2 ? h.f_set[1] : NAN;
    bool accepted = nsets == 2 && (f_rel <= f_next);
    double f_after = accepted ? f_rel : f_next;
    if (enumerate) {  // candidate stresses from the enumeration pass; f_after from the chosen point's P1 pass
        omega = h.omega_star;
        accepted = h.enum_best > 0;
        f_next = h.enum_f0;
        f_rel = h.enum_fbest;
        f_after = h.f_set[0];
    }
    if (ctx->p1_fused_now) {
        ctx->stats.p1_predicted++;
        if (!accepted) ctx->stats.p1_predicted_rejected++;
    }
    // R30: predict the next guard decision from this one -- after an accepted Xt whose
    // extra decrease f(X^{k+1}) - f(Xt) fell below 0.6 of the solve's own decrease
    // f(X^k) - f(X^{k+1}), the relaxation is running out and the next Xt tends to overshoot
    if (ctx->p1_predict && nsets == 2 && !enumerate)
        ctx->p1_fused_next = accepted && (f_next - f_rel) < 0.6 * (f_before - f_next);
    ctx->iterations++;
    ctx->f = f_after;
    fdl_iter_info inf{};
    inf.it = ctx->iterations;
    inf.accepted = accepted ? 1 : 0;
    inf.cg_iters = cg;
    inf.omega = omega;
    inf.f_before = f_before * ctx->fscale;  // f = k^(alpha+2) f' (units of k)
    inf.f_next = f_next * ctx->fscale;
    inf.f_relaxed = f_rel * ctx->fscale;
    inf.f_after = f_after * ctx->fscale;
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
    p->a_refresh = 10;
    p->hop_bits = 0;
    p->cg_extrap = 2;
    p->enum_count = 19;
    p->enum_step = 0.5;
    p->p1_split = -1;
    p->use_graphs = -1;
    p->cg_history = 0;
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
    if (ctx) {
        for (auto& kv : ctx->graphs)
            if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
        ctx->graphs.clear();
        if (ctx->aux_stream) cudaStreamDestroy(ctx->aux_stream);
        ctx->aux_stream = nullptr;
    }
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
                                int32_t world, fdl_ctx** out, fdl_group* group = nullptr)
{
    if (!out) return FDL_E_INVALID_ARG;
    *out = nullptr;
    fdl_ctx* ctx = new fdl_ctx();
    ctx->group = group;
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

fdl_status fdl_group_create(int32_t world, fdl_group** out)
{
    if (!out || world < 1) return FDL_E_INVALID_ARG;
    *out = new fdl_group();
    (*out)->world = world;
    return FDL_OK;
}

void fdl_group_destroy(fdl_group* g) { delete g; }

fdl_status fdl_create_loopback(int32_t n, const int64_t* row_ptr, const int32_t* col_idx, const double* edge_len,
                               const fdl_params* p, const double* init_pos, fdl_group* group, int32_t rank,
                               fdl_ctx** out)
{
    if (!group) return FDL_E_INVALID_ARG;
    return create_common(n, row_ptr, col_idx, edge_len, p, init_pos, nullptr, rank, group->world, out, group);
}

fdl_status fdl_shard_tiles(int32_t n, int32_t world, int32_t rank, int64_t* t0, int64_t* t1)
{
    if (n < 1 || world < 1 || rank < 0 || rank >= world || !t0 || !t1) return FDL_E_INVALID_ARG;
    // Boundaries fall on global work-item boundaries (strip segments of <= seg_len(nb)
    // tiles), nearest to equal tile shares: every item -- and so every fp32
    // segment sum -- is the same for any number of GPUs.
    const int64_t nb = (n + kT - 1) / kT;
    const int64_t total = nb * (nb + 1) / 2;
    auto boundary = [&](int64_t target) -> int64_t {
        if (target <= 0) return 0;
        if (target >= total) return total;
        int64_t best = 0;
        for (int64_t I = 0; I < nb; ++I) {
            const int64_t s0 = tri_index(I, I, nb), len = nb - I;
            if (s0 + len < target) continue;  // strip entirely before the target
            // segment starts inside strip I: s0, s0 + kSeg, ...
            const int64_t sl = seg_len(nb);
            const int64_t k = (target - s0 + sl / 2) / sl;
            best = std::min(s0 + k * sl, s0 + len);
            break;
        }
        return best;
    };
    *t0 = boundary(total * rank / world);
    *t1 = boundary(total * (rank + 1) / world);
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

fdl_status fdl_set_omega_vertex(fdl_ctx* ctx, const double* omega, size_t count)
{
    if (!ctx) return FDL_E_INVALID_ARG;
    if (ctx->broken) return set_err(ctx, FDL_E_STATE, ctx->err);
    for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second.exec);
    ctx->graphs.clear();
    if (!omega) {
        if (ctx->omega_v) {
            cudaFree(ctx->omega_v);
            ctx->allocs.erase(std::find(ctx->allocs.begin(), ctx->allocs.end(), (void*)ctx->omega_v));
            ctx->omega_v = nullptr;
        }
        return FDL_OK;
    }
    if (count != (size_t)ctx->n) return set_err(ctx, FDL_E_INVALID_ARG, "omega count must be n");
    if (ctx->p.strategy != FDL_STRAT_FIXED)
        return set_err(ctx, FDL_E_UNSUPPORTED, "per-vertex omega requires the fixed strategy");
    double mx = 0.0;
    for (size_t i = 0; i < count; ++i) {
        if (!(omega[i] >= 0.0) || !std::isfinite(omega[i]))
            return set_err(ctx, FDL_E_INVALID_ARG, "omega_i must be finite and >= 0");
        mx = std::max(mx, omega[i]);
    }
    FDL_CUDA(cudaSetDevice(ctx->device));
    if (!ctx->omega_v) FDL_ALLOC(ctx->omega_v, (size_t)ctx->n);
    FDL_CUDA(cudaMemcpyAsync(ctx->omega_v, omega, sizeof(double) * count, cudaMemcpyHostToDevice, ctx->stream));
    FDL_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->omega_v_max = mx;
    for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second.exec);  // they baked the old omega_v
    ctx->graphs.clear();
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
    r.f_initial = ctx->f * ctx->fscale;
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
    r.f_final = ctx->f * ctx->fscale;
    if (info) *info = r;
    return s;
}

fdl_status fdl_get_positions(const fdl_ctx* cctx, double* out, size_t count)
{
    // logically const: the placement is only read; the x k scaling runs
    // in the context's PCG scratch vector and on its stream
    fdl_ctx* ctx = const_cast<fdl_ctx*>(cctx);
    if (!ctx || !out) return FDL_E_INVALID_ARG;
    if (ctx->emulated) return set_err(ctx, FDL_E_UNSUPPORTED, "emulated rank: only fdl_eval_partial");
    if (count != (size_t)ctx->n * ctx->dim) return set_err(ctx, FDL_E_INVALID_ARG, "count must be n*dim");
    if (ctx->broken) return FDL_E_STATE;
    cudaSetDevice(ctx->device);
    // x k on the device (into PCG scratch, free between steps), then one copy to the caller
    FDL_LAUNCH(launch_pin_scale(ctx->Xk, ctx->cy, ctx->n, ctx->dim, ctx->k, 1, ctx->stream));
    FDL_CUDA(cudaMemcpyAsync(out, ctx->cy, count * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    FDL_CUDA(cudaStreamSynchronize(ctx->stream));
    return FDL_OK;
}

fdl_status fdl_set_positions(fdl_ctx* ctx, const double* in, size_t count)
{
    if (!ctx || !in) return FDL_E_INVALID_ARG;
    if (ctx->emulated) return set_err(ctx, FDL_E_UNSUPPORTED, "emulated rank: only fdl_eval_partial");
    if (count != (size_t)ctx->n * ctx->dim) return set_err(ctx, FDL_E_INVALID_ARG, "count must be n*dim");
    if (ctx->broken) return FDL_E_STATE;
    for (size_t i = 0; i < count; ++i)
        if (!std::isfinite(in[i])) return set_err(ctx, FDL_E_INVALID_ARG, "non-finite position");
    cudaSetDevice(ctx->device);
    ctx->stopped = false;
    ctx->stop_reason = 0;
    if (ctx->a_valid && std::isfinite(ctx->f)) {
        // the placement fdl_get_positions returned, passed back unchanged (a caller that
        // round-trips its placement through the host every step): the context's f, R, L^W X
        // and PCG history are already those of this placement, so no evaluation pass
        FDL_CUDA(cudaMemcpyAsync(ctx->Xt, in, count * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        FDL_CUDA(cudaMemsetAsync(&ctx->sc->anynew, 0, sizeof(unsigned int), ctx->stream));
        FDL_LAUNCH(launch_placement_differs(ctx->Xt, ctx->Xk, count, ctx->k, &ctx->sc->anynew, ctx->stream));
        unsigned int differs = 1;
        FDL_CUDA(cudaMemcpyAsync(&differs, &ctx->sc->anynew, sizeof differs, cudaMemcpyDeviceToHost, ctx->stream));
        FDL_CUDA(cudaStreamSynchronize(ctx->stream));
        if (!differs) return FDL_OK;
    }
    return upload_positions(ctx, in);
}

fdl_status fdl_eval_forces(fdl_ctx* ctx, double* R, double* A, double* stress)
{
    if (!ctx) return FDL_E_INVALID_ARG;
    if (ctx->emulated) return set_err(ctx, FDL_E_UNSUPPORTED, "emulated rank: only fdl_eval_partial");
    if (ctx->broken) return FDL_E_STATE;
    cudaSetDevice(ctx->device);
    const int dim = ctx->dim;
    const size_t count = (size_t)ctx->n * dim;
    auto fetch = [&](const double* dev, double* out) -> fdl_status {
        FDL_CUDA(cudaMemcpyAsync(out, dev, count * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        FDL_CUDA(cudaStreamSynchronize(ctx->stream));
        for (size_t i = 0; i < count; ++i) out[i] *= ctx->rscale;  // R = k^(alpha+1) R' (= R'/k at alpha = -2)
        return FDL_OK;
    };
    if (R) FDL_TRY(fetch(ctx->Rk, R));
    if (A) {
        // A = L^W X: one symmetric P2 pass with p = X
        FDL_LAUNCH3(launch_cg_begin(ctx->Xk, ctx->cy, ctx->pvec, ctx->n, 0, dim, ps_p2(dim), ctx->sc, ctx->blk_cg,
                                    ctx->stream));
        FDL_TRY(run_sym(ctx, kSymP2, 1, ctx->pvec, ctx->cy, nullptr, 0));
        FDL_TRY(fetch(ctx->cy, A));
        collect_events(ctx);
    }
    if (stress) *stress = ctx->f * ctx->fscale;
    return FDL_OK;
}

fdl_status fdl_eval_partial(fdl_ctx* ctx, int32_t mode, const double* X, double* out, double* stress)
{
    if (!ctx || !X || !out || (mode != 0 && mode != 1)) return FDL_E_INVALID_ARG;
    if (ctx->broken) return FDL_E_STATE;
    cudaSetDevice(ctx->device);
    const int dim = ctx->dim;
    const size_t count = (size_t)ctx->n * dim;
    std::vector<double> xs(count);
    for (int i = 0; i < ctx->n; ++i)
        for (int q = 0; q < dim; ++q) xs[(size_t)i * dim + q] = (X[(size_t)i * dim + q] - X[q]) / ctx->k;
    FDL_CUDA(cudaMemcpyAsync(ctx->Xt, xs.data(), count * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    if (mode == 0) {
        FDL_LAUNCH(launch_stage_pos1(ctx->Xt, ctx->posf, ctx->n, 0, dim, ps_p1(dim, 1), ctx->stream));
        FDL_TRY(run_sym(ctx, kSymP1, 1, ctx->posf, ctx->R1, nullptr, 0));
    } else {
        FDL_LAUNCH3(launch_cg_begin(ctx->Xt, ctx->R1, ctx->pvec, ctx->n, 0, dim, ps_p2(dim), ctx->sc, ctx->blk_cg,
                                    ctx->stream));
        FDL_TRY(run_sym(ctx, kSymP2, 1, ctx->pvec, ctx->R1, nullptr, 0));
    }
    FDL_CUDA(cudaMemcpyAsync(out, ctx->R1, count * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    FDL_CUDA(cudaMemcpyAsync(ctx->sc_host, ctx->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, ctx->stream));
    FDL_CUDA(cudaStreamSynchronize(ctx->stream));
    collect_events(ctx);
    for (size_t i = 0; i < count; ++i) out[i] *= ctx->rscale;
    if (stress) *stress = mode == 0 ? ctx->sc_host->f_set[0] * ctx->fscale : 0.0;
    return FDL_OK;
}

fdl_status fdl_get_hop_rows(fdl_ctx* ctx, int32_t r0, int32_t nrows, uint16_t* out)
{
    if (!ctx || !out || nrows < 0 || r0 < 0 || r0 + nrows > ctx->n) return FDL_E_INVALID_ARG;
    if (ctx->hb == kHbDist) return set_err(ctx, FDL_E_UNSUPPORTED, "fp32 path-length tiles: use fdl_get_dist_rows");
    cudaSetDevice(ctx->device);
    if (nrows == 0) return FDL_OK;
    std::vector<int> rows(nrows);
    for (int r = 0; r < nrows; ++r) rows[r] = r0 + r;
    int* d_rows = nullptr;
    int* d_missing = nullptr;
    uint16_t* d_out = nullptr;
    Scratch tmp;
    FDL_CUDA(tmp.alloc(&d_rows, sizeof(int) * nrows));
    FDL_CUDA(tmp.alloc(&d_missing, sizeof(int)));
    FDL_CUDA(tmp.alloc(&d_out, sizeof(uint16_t) * (size_t)nrows * ctx->n));
    cudaMemcpyAsync(d_rows, rows.data(), sizeof(int) * nrows, cudaMemcpyHostToDevice, ctx->stream);
    cudaMemsetAsync(d_missing, 0, sizeof(int), ctx->stream);
    cudaError_t e = launch_hop_rows(ctx->D, ctx->hb, ctx->nb, ctx->t0, ctx->t1, d_rows, nrows, ctx->n, d_out,
                                    d_missing, ctx->stream);
    int missing = 0;
    if (e == cudaSuccess) {
        cudaMemcpyAsync(out, d_out, sizeof(uint16_t) * (size_t)nrows * ctx->n, cudaMemcpyDeviceToHost, ctx->stream);
        cudaMemcpyAsync(&missing, d_missing, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream);
        e = cudaStreamSynchronize(ctx->stream);
    }
    FDL_CUDA(e);
    if (missing) return set_err(ctx, FDL_E_INVALID_ARG, "some requested entries live in tiles of other ranks");
    return FDL_OK;
}

fdl_status fdl_get_dist_rows(fdl_ctx* ctx, int32_t r0, int32_t nrows, double* out)
{
    if (!ctx || !out || nrows < 0 || r0 < 0 || r0 + nrows > ctx->n) return FDL_E_INVALID_ARG;
    cudaSetDevice(ctx->device);
    if (nrows == 0) return FDL_OK;
    std::vector<int> rows(nrows);
    for (int r = 0; r < nrows; ++r) rows[r] = r0 + r;
    const size_t cnt = (size_t)nrows * ctx->n;
    int* d_rows = nullptr;
    int* d_missing = nullptr;
    float* d_out = nullptr;
    Scratch tmp;
    FDL_CUDA(tmp.alloc(&d_rows, sizeof(int) * nrows));
    FDL_CUDA(tmp.alloc(&d_missing, sizeof(int)));
    FDL_CUDA(tmp.alloc(&d_out, sizeof(float) * cnt));
    cudaMemcpyAsync(d_rows, rows.data(), sizeof(int) * nrows, cudaMemcpyHostToDevice, ctx->stream);
    cudaMemsetAsync(d_missing, 0, sizeof(int), ctx->stream);
    cudaError_t e = launch_dist_rows(ctx->D, ctx->hb, ctx->nb, ctx->t0, ctx->t1, d_rows, nrows, ctx->n, d_out,
                                     d_missing, ctx->stream);
    int missing = 0;
    std::vector<float> host(cnt);
    if (e == cudaSuccess) {
        cudaMemcpyAsync(host.data(), d_out, sizeof(float) * cnt, cudaMemcpyDeviceToHost, ctx->stream);
        cudaMemcpyAsync(&missing, d_missing, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream);
        e = cudaStreamSynchronize(ctx->stream);
    }
    FDL_CUDA(e);
    if (missing) return set_err(ctx, FDL_E_INVALID_ARG, "some requested entries live in tiles of other ranks");
    for (size_t i = 0; i < cnt; ++i) out[i] = ctx->k * (double)host[i];
    return FDL_OK;
}

fdl_status fdl_get_diag(fdl_ctx* ctx, double* out, size_t count)
{
    if (!ctx || !out) return FDL_E_INVALID_ARG;
    if (count != (size_t)ctx->n) return set_err(ctx, FDL_E_INVALID_ARG, "count must be n");
    cudaSetDevice(ctx->device);
    FDL_CUDA(cudaMemcpyAsync(out, ctx->diag, count * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    FDL_CUDA(cudaStreamSynchronize(ctx->stream));
    for (size_t i = 0; i < count; ++i) out[i] *= ctx->dscale;  // w = k^alpha w'
    return FDL_OK;
}

fdl_status fdl_get_info(fdl_ctx* ctx, fdl_ctx_info* info)
{
    if (!ctx || !info) return FDL_E_INVALID_ARG;
    fdl_ctx_info r{};
    r.n = ctx->n;
    r.dim = ctx->dim;
    r.diameter = ctx->diameter;
    r.hop_bits = ctx->hb ? 8 * ctx->hb : 4;
    r.tile0 = ctx->t0;
    r.tile1 = ctx->t1;
    r.rank = ctx->rank;
    r.world = ctx->world;
    r.iterations = ctx->iterations;
    r.k = ctx->k;
    r.f = ctx->f * ctx->fscale;
    r.hop_matrix_bytes = ctx->hop_bytes_total;
    r.local_pairs = ctx->local_pairs;
    r.device_bytes = ctx->device_bytes;
    r.setup_ms = ctx->setup_ms;
    r.setup_dist_ms = ctx->setup_dist_ms;
    r.bfs_bytes = ctx->bfs_bytes;
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

// pairs/s of sym_tile<mode> on a resident tile (fdl_bench_p1s_mix, fdl_bench_p2_mix)
static fdl_status bench_tile_mix(int32_t device, int mode, double* pairs_per_s, double* ms)
{
    if (!pairs_per_s || !ms) return FDL_E_INVALID_ARG;
    if (cudaSetDevice(device) != cudaSuccess) return FDL_E_CUDA;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int blocks = sms * tile_mix_ctas_per_sm(mode), iters = 2000;
    float *pos = nullptr, *out = nullptr;
    if (cudaMalloc(&pos, kT * 4 * sizeof(float)) != cudaSuccess) return FDL_E_OOM;
    if (cudaMalloc(&out, (size_t)blocks * 256 * sizeof(float)) != cudaSuccess) {
        cudaFree(pos);
        return FDL_E_OOM;
    }
    std::vector<float> h(kT * 4);
    for (int k = 0; k < kT * 4; ++k) h[k] = (float)((k * 37 % 101) * 0.01);
    cudaMemcpy(pos, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch_tile_mix(mode, pos, out, 20, blocks, s);  // warm-up
    cudaEventRecord(a, s);
    launch_tile_mix(mode, pos, out, iters, blocks, s);
    cudaEventRecord(b, s);
    cudaError_t e = cudaEventSynchronize(b);
    float t = 0.f;
    cudaEventElapsedTime(&t, a, b);
    const double pairs = (double)blocks * 256 * iters * 64.0;  // 64 pairs per thread per tile
    *ms = t;
    *pairs_per_s = pairs / (t * 1e-3);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaStreamDestroy(s);
    cudaFree(pos);
    cudaFree(out);
    return e == cudaSuccess ? FDL_OK : FDL_E_CUDA;
}

fdl_status fdl_bench_p1s_mix(int32_t device, double* tflops, double* ms)
{
    double pps = 0.0;
    fdl_status st = bench_tile_mix(device, kSymP1S, &pps, ms);
    if (st == FDL_OK) *tflops = pps * 29.0 / 1e12;  // 29 algorithmic flops per pair
    return st;
}

fdl_status fdl_bench_p2_mix(int32_t device, double* hop_gbs, double* ms)
{
    double pps = 0.0;
    fdl_status st = bench_tile_mix(device, kSymP2, &pps, ms);
    if (st == FDL_OK) *hop_gbs = pps * 0.5 / 1e9;  // 4-bit hops: 0.5 B per unordered pair
    return st;
}

}  // extern "C"
