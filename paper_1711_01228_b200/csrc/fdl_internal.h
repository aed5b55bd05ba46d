// fdl_internal.h -- shared declarations between the host runtime (fdl_api.cu)
// and the kernels (fdl_kernels.cu).  Not part of the ABI (include/fdl.h is).
//
// Units: the device works in units of k (scaled coordinates X' = X / k), where
// the ideal distance is the hop count itself (d' = h) and w' = h^-2.  For
// w = d^-2 this is exact (f is scale-free, H_{kD}(kY) = k H_D(Y)); the
// library converts at the boundary.  DESIGN.md §6 "Units".
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

namespace fdl {

// Slot of vertex v in the staged fp32 vectors (P1 positions, P2 p): inside each
// 128-vertex block, v -> (v % 8) * 16 + (v % 128) / 8, so the 16 thread columns
// of k_sym read 16 consecutive slots for their column c (no bank conflicts).
__host__ __device__ inline int64_t stage_slot(int64_t v)
{
    return (v & ~(int64_t)127) | ((v & 7) << 4) | ((v & 127) >> 3);
}

// ------------------------------------------------------------ debug bounds
// FDL_DEBUG_BOUNDS builds (scripts/debug_build.sh, tests run against them through
// FDL_LIB) check the global-memory indices of the pair, reduction and setup kernels and
// trap on a violation: the pool's compute-sanitizer is closed, so out-of-range accesses
// are caught by the kernels themselves.
#ifdef FDL_DEBUG_BOUNDS
#define FDL_DCHECK(c)                                                                        \
    do {                                                                                     \
        if (!(c)) {                                                                          \
            printf("FDL_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
                   (int)blockIdx.x, (int)threadIdx.x);                                       \
            __trap();                                                                        \
        }                                                                                    \
    } while (0)
#else
#define FDL_DCHECK(c) \
    do {              \
    } while (0)
#endif

// ------------------------------------------------------------ constants
constexpr int kRB = 256;           // row block of all fp64 vector reductions
constexpr int kGalMax = 8;         // history window of the recycled PCG start (R27)
constexpr int kGalNV = kGalMax * (kGalMax + 1) / 2 + kGalMax;  // Gram entries + right-hand sides per column
constexpr int kBFSWords = 32;      // MS-BFS source batch = 32 words x 32 bits = 1024
constexpr int kBfsHubDeg = 256;
constexpr int kBfsWideWords = 128;  // clustered MS-BFS batches: 128 words x 32 = 4096 sources
// weighted APSP: a warp relaxes one chunk of 32 x 4 x 32 = 4096 sources of a vertex at a
// time; a batch holds up to kBfMaxChunks chunks (one 16-bit pending mask per vertex)
constexpr int kBfWordsPerLane = 4;
constexpr int kBfChunk = 32 * 32 * kBfWordsPerLane;
constexpr int kBfMaxChunks = 16;

// Device-resident scalars of the iteration (one struct per context).
struct DevScalars {
    double f_set[2];       // stress of the position sets of the last P1 pass
    double f_cur;          // f(X^k)
    double f_next, f_relaxed;
    int accepted;
    int nonfinite;
    double maxdisp;        // scaled units
    // PCG (per column, up to 3)
    double rz[4], bb[4], rr[4], alpha[4], beta[4], pap[4];
    double S[4];           // sum_i p_i per column (rank-one term of the regularised operator)
    double Sd[4];          // sum_i d_i of the PCG correction d = x - x0 (for the carried L^W X)
    double rho;            // PCG start extrapolation ratio (k_rho)
    double omega_star;     // enumerating strategy: chosen relax factor
    int enum_best;         // ... and its candidate index
    double enum_f0, enum_fbest;  // ... stress of candidate 0 (X^{k+1}) and of the chosen one
    double cmean[4];       // column means of the staged X (centring of the product-form P2 input)
    double inv_n;          // 1 / n
    double sigma;          // regularisation weight: (L + sigma 1 1^T), sigma = mean(diag)/n
    int active[4];
    int done;
    int cg_iters;
    double relres;
    unsigned int anynew;   // fdl_set_positions: the uploaded placement differs from X^k
    // recycled PCG start (R27): y of x0 = X^k + V y per column, basis vectors in use
    double gal_y[3][8];
    int gal_cnt;           // valid history vectors for the next start (<= kGalMax)
    int gal_use;           // vectors used by the current start
    int gal_dropped;       // dependent vectors skipped by the last solve
    int gal_m;             // window (fdl_params.cg_history, <= kGalMax)
    // MS-BFS setup (device-driven level loop)
    int bfs_diam;          // deepest level found so far
    int bfs_overflow;      // a level beyond the stored width's maximum found a vertex
    unsigned long long bfs_bytes;  // gather bytes of the level kernels (roofline)
};

// Host-mapped flag the host reads after a stream sync.
struct HostScalars {
    volatile int done;
    volatile unsigned int anynew;
};

// ------------------------------------------------------------ launchers
// All launchers enqueue on `s` and return the CUDA error of the launch.
cudaError_t launch_bfs_init(uint32_t* frontier, uint32_t* visited, int n, int s0, cudaStream_t s);

// staging / vector kernels (dim columns, rows [0, nloc); row0 = 0 with replicated state)
cudaError_t launch_stage_pos1(const double* X, float* posf, int nloc, int row0, int dim, int ps,
                              cudaStream_t s);
cudaError_t launch_combine(const double* Xk, double* Xn, double* Xt, float* posf, double* blk_max,
                           const double* xpin, int nloc, int row0, int dim, double omega, const double* omega_v,
                           double cap, int nsets, int ps, cudaStream_t s);
// carried A = L^W X: An = Rk - r_cg - sigma Sd 1 (for X^{k+1}), At = (1+w) An - w Ak (for Xt)
cudaError_t launch_carry_a(const double* Rk, const double* rcg, const double* Ak, double* An, double* At,
                           const DevScalars* sc, int n, int dim, double omega, cudaStream_t s);
cudaError_t launch_extrap(const double* Xk, const double* Xprev, const double* Ak, const double* Aprev, double* x,
                          double* y0, const DevScalars* sc, int n, int dim, int valid, cudaStream_t s);
// ABI units: mode 0 y = (x - x_0) / k (upload, pin), mode 1 y = x k (download)
cudaError_t launch_pin_scale(const double* x, double* y, int n, int dim, double k, int mode, cudaStream_t s);
cudaError_t launch_placement_differs(const double* x, const double* Xk, size_t cnt, double k, unsigned int* differs,
                                     cudaStream_t s);
// Recycled PCG start (R27): Galerkin projection of the warm-start error onto the
// last kGalMax step differences V (with AV = L^W V from the carried products).
cudaError_t launch_gal_start(const double* V, const double* AV, const double* b, const double* Xk, const double* Ak,
                             double* x, double* y0, double* blk, int nblk, DevScalars* sc, int n, int dim,
                             cudaStream_t s);
// V <- [X^k - X^{k-1}, V[0..m-2]], AV likewise (m = window)
cudaError_t launch_gal_push(const double* Xk, const double* Xprev, const double* Ak, const double* Aprev, double* V,
                            double* AV, int n, int dim, int m, cudaStream_t s);
cudaError_t launch_rho(const double* Xn, const double* Xk, double* Xprev, const double* Ak, double* Aprev,
                       double* blk, int n, int dim, int valid, DevScalars* sc, cudaStream_t s);
cudaError_t launch_enum_stage(const double* Xk, double* Xn, float* posf, double* blk_max, const double* xpin, int n,
                              int dim, int ps, cudaStream_t s);
cudaError_t launch_enum_pick(const double* fs, int m, double step, DevScalars* sc, cudaStream_t s);
cudaError_t launch_enum_apply(const double* Xn, const double* Xk, const double* An, const double* Ak, double* Xt,
                              double* At, float* posf, const DevScalars* sc, int n, int dim, int ps, cudaStream_t s);
cudaError_t launch_get_pin(const double* x, double* slots, int rank, int dim, int owns_row0, cudaStream_t s);
cudaError_t launch_select(double* Xk, double* Rk, const double* Xn, const double* Xt, const double* R1,
                          const double* R2, const double* blk_max, int nloc, int dim, int nsets,
                          DevScalars* sc, double* Ak, const double* An, const double* At, cudaStream_t s);
cudaError_t launch_cg_begin(const double* Xk, double* x, float* pvec, int nloc, int row0, int dim, int pq,
                            DevScalars* sc, double* blk /* >= 4 x ceil(nloc / kRB) doubles, scratch */,
                            cudaStream_t s);
cudaError_t launch_stage_p(const double* p, float* pvec, const DevScalars* sc, int n, int dim, int pq,
                           cudaStream_t s);
cudaError_t launch_p2_finish(double* out, const float* pvec, const double* diag, int n, int dim, int pq,
                             cudaStream_t s);
cudaError_t launch_cg_init(const double* y, const double* b, const double* diag, double* r, double* z,
                           double* p, float* pvec, double* blk, int nblk, int n, int dim, int pq,
                           cudaStream_t s);
cudaError_t launch_cg_ap(const double* p, double* y, double* blk, int nblk, int n, int dim,
                         const DevScalars* sc, cudaStream_t s);
cudaError_t launch_cg_update(double* x, double* r, double* z, const double* p, const double* y,
                             const double* diag, double* blk, int nblk, const DevScalars* sc, int nloc,
                             int row0, int dim, cudaStream_t s);
cudaError_t launch_cg_p(double* p, const double* z, float* pvec, const DevScalars* sc, int nloc, int row0,
                        int dim, int pq, cudaStream_t s);
// mode 0: after init (rz, rr, bb, sum z); 1: alpha from pAp; 2: beta + convergence
// cond/use_cond: the WHILE-node handle of a captured step graph (continue = PCG not done
// and cg_iters < cg_max); use_cond = 0 outside graphs
cudaError_t launch_cond_done(const DevScalars* sc, cudaStream_t s, unsigned long long cond);
cudaError_t launch_cg_finalize(const double* blk, int nblk, int dim, int mode, double rtol,
                               DevScalars* sc, HostScalars* hs, cudaStream_t s, unsigned long long cond = 0,
                               int use_cond = 0, int cg_max = 0);
// one PCG iteration after the P2 pass in one 1024-thread block (small n), bitwise the
// k_p2_finish / k_cg_ap / finalize / k_cg_update / finalize / k_cg_p sequence
cudaError_t launch_cg_tail(double* y, const float* pvec_in, const double* diag, double* x, double* r, double* z,
                           double* p, float* pvec, double* blk, int n, int dim, int nblk, int pq, double rtol,
                           DevScalars* sc, HostScalars* hs, cudaStream_t s, unsigned long long cond, int use_cond,
                           int cg_max);
cudaError_t launch_ffma_bench(float* out, int iters, int blocks, int threads, cudaStream_t s);
// sym_tile<mode> (kSymP1S or kSymP2, 2-D, 4-bit) on a resident tile: the pass's arithmetic ceiling
cudaError_t launch_tile_mix(int mode, const float* pos, float* out, int iters, int blocks, cudaStream_t s);
int tile_mix_ctas_per_sm(int mode);

// ------------------------------------------------------- symmetric (triangle) passes
constexpr int kT = 128;            // tile edge: tiles (I, J), I <= J, of kT x kT pairs
#ifndef FDL_SEG
#define FDL_SEG 16
#endif
constexpr int kSeg = FDL_SEG;      // tiles per work item (strip segment)
// P1S: 2 stress sets, R of set 1; P1A: 1 set, stress + R + L^W X (difference form, unit lengths);
// P1R: 1 set, R only (the rejection pass: its stress is known from P1S)
enum { kSymP1 = 0, kSymP2 = 1, kSymDiag = 2, kSymP1S = 3, kSymP1A = 4, kSymP1R = 5 };

// triangle index of tile (I, J), I <= J, over nb blocks (row-major upper triangle)
__host__ __device__ inline int64_t tri_index(int64_t I, int64_t J, int64_t nb)
{
    return I * nb - I * (I - 1) / 2 + (J - I);
}

// Hop width code `hb`: 0 = 4-bit (diameter <= 15), 1 = uint8, 2 = uint16;
// 4 = fp32 path lengths (weighted graphs / general alpha, NEXT-3).
__host__ __device__ constexpr int64_t tile_bytes(int hb) { return hb ? (int64_t)kT * kT * hb : (int64_t)kT * kT / 2; }
constexpr int hb_max_hop(int hb) { return hb == 0 ? 15 : (hb == 1 ? 255 : 65535); }
constexpr int kHbDist = 4;

// 4-bit tiles store the hops of rows (2p, 2p+1) of one column in one byte.  The
// byte is a bijective encoding of the pair, chosen so that the shared-memory
// LUT the kernels index with it (8-byte entries) spreads the common hop pairs
// over the banks: low nibble = (lo + 4 hi) mod 16, high nibble = hi.
__host__ __device__ inline uint32_t nib_encode(uint32_t lo, uint32_t hi) { return ((lo + 4u * hi) & 15u) | (hi << 4); }
__host__ __device__ inline uint32_t nib_decode_lo(uint32_t b) { return ((b & 15u) - 4u * (b >> 4)) & 15u; }
__host__ __device__ inline uint32_t nib_decode_hi(uint32_t b) { return b >> 4; }

// byte offset of entry (row rl, col cl) inside local tile lt: thread (ty, tx) =
// (rl/8, cl/8) of a 16 x 16 grid, linear index tx*16 + ty (= k_sym's threadIdx),
// owns an 8 x 8 sub-block stored as 16-byte chunks interleaved across the 256
// threads.  4-bit: chunk = 4 columns x 4 row pairs,
// the entry is nibble (rl & 1) of the returned byte (before nib_encode).
__host__ __device__ inline size_t sym_offset(int64_t lt, int rl, int cl, int hb)
{
    const int tid = (cl >> 3) * 16 + (rl >> 3), r = rl & 7, c = cl & 7;
    const size_t base = (size_t)lt * (size_t)tile_bytes(hb);
    if (hb == 0) return base + ((size_t)(c >> 2) * 256 + tid) * 16 + (c & 3) * 4 + (r >> 1);
    if (hb == 4) return base + ((size_t)(c * 2 + (r >> 2)) * 256 + tid) * 16 + (r & 3) * 4;  // fp32 distances
    if (hb == 1) return base + ((size_t)(c >> 1) * 256 + tid) * 16 + (c & 1) * 8 + r;
    return base + ((size_t)c * 256 + tid) * 16 + r * 2;
}

struct SymArgs {
    const uint8_t* D;      // local tiles, triangle order
    const float* pos;      // staged positions / p vector, stride sym_ps floats, nb*kT vertices
    float* jpart;          // [local tile][kT][C] fp32 j-side partials
    float* ipart;          // [item][warp][kT][C] fp32 i-side partials
    double* spart;         // [item][warp][nsets] fp64 stress partials (P1); k_enum: [item][kEnumNC]
    const int4* items;     // {I, J0, ntiles, first local tile}
    const int* order;      // schedule: CTA b takes items order[b], order[b + grid], ... (item_order)
    int nitems;
    int n;
    uint32_t magic;        // 0x4B000000 (2^23 as fp32 bits) for the hop decode, passed as a
                           // parameter so the PRMT selector can stay an immediate
    float alpha;           // weight exponent w = d^alpha (fp32 distance tiles, hb = 4)
    int64_t ntiles;        // local tiles (bounds checks of the debug build)
    int64_t nstage;        // vertices of the staged position vector (nb * kT)
};

cudaError_t launch_sym(const SymArgs& a, int mode, int dim, int nsets, int hb, int grid, cudaStream_t s);

// enumerating strategy: stress of kEnumNC relaxed candidates per pass
constexpr int kEnumNC = 10;  // 19 paper candidates -> 2 passes
constexpr int kEnumMax = 32;
struct EnumOmegas {
    float w[kEnumNC];
};
cudaError_t launch_enum(const SymArgs& a, const EnumOmegas& w, int dim, int hb, int grid, cudaStream_t s);
int sym_max_ctas(int mode, int dim, int nsets, int hb);
// Ilo..Ihi: row blocks of the local tiles [t0, t1)
cudaError_t launch_sym_reduce(const float* ipart, const float* jpart, const int* it_lo, const int* it_hi, int nb,
                              int64_t t0, int64_t t1, int Ilo, int Ihi, int C, int D, int inter, double* out0,
                              double* out1, cudaStream_t s);
// scratch: sym_stress_chunks(nitems) * nsets doubles
int sym_stress_chunks(int nitems);
cudaError_t launch_sym_stress(const double* spart, int nitems, int nsets, double* out, double* scratch,
                              cudaStream_t s);
cudaError_t launch_bfs_level_sym(const int64_t* row_ptr, const int32_t* col, const uint32_t* fin, uint32_t* fout,
                                 uint32_t* visited, uint8_t* bbuf, int n, int nsrc, int level, int hb,
                                 unsigned int* flags, unsigned long long* bytes, const int* hubs, int nhub, int grid,
                                 cudaStream_t s);
cudaError_t launch_bfs_init_list(uint32_t* frontier, uint32_t* visited, uint8_t* fl, const int* srcs, int nsrc,
                                 int nw, cudaStream_t s);
cudaError_t launch_bfs_level_wide(const int64_t* row_ptr, const int32_t* col, const uint32_t* fin, uint32_t* fout,
                                  uint32_t* visited, uint8_t* bbuf, int n, int nsrc, int level, int hb,
                                  unsigned int* flags, unsigned long long* bytes, int grid, const uint8_t* fl_in,
                                  uint8_t* fl_out, cudaStream_t s);
cudaError_t launch_bfs_scatter(const uint8_t* bbuf, uint8_t* D, const int* srcs, int nsrc, int n, int nb, int64_t t0,
                               int64_t t1, int hb, int64_t rb, cudaStream_t s);
cudaError_t launch_bfs_batch_end(const unsigned int* flags, int nlevels, int maxhop, int* diam, int* overflow,
                                 cudaStream_t s);
cudaError_t launch_bfs_retile(const uint8_t* bbuf, uint8_t* D, int n, int s0, int nsrc, int nb, int64_t t0,
                              int64_t t1, int hb, cudaStream_t s);
int bfs_row_bytes_host(int hb);  // batch-buffer bytes per vertex
// weighted / general-alpha setup: multi-source Bellman-Ford in fp64 over the
// CSR with edge lengths; dist[v * S + s] for the batch's sources s0..s0+S-1
cudaError_t launch_bf_init(double* dist, int n, const int* srcs, int nsrc, int S, cudaStream_t s);
cudaError_t launch_bf_sweep(const int64_t* row_ptr, const int32_t* col, const double* len, double* dist,
                            const uint32_t* chg_in, uint32_t* chg_out, const uint16_t* pend_in, uint16_t* pend_out,
                            int n, int S, int nsrc, int it, double delta, unsigned int* flags, int grid,
                            cudaStream_t s);
cudaError_t launch_bf_seed(uint32_t* chg, uint16_t* pend, const int* srcs, int nsrc, int S, cudaStream_t s);
cudaError_t launch_bf_store(const double* dist, int n, const int* srcs, int nsrc, int S, int nb, int64_t t0,
                            int64_t t1, uint8_t* D, double* dmax, cudaStream_t s);
cudaError_t launch_dist_rows(const uint8_t* D, int hb, int nb, int64_t t0, int64_t t1, const int* rows, int nrows,
                             int n, float* out, int* missing, cudaStream_t s);
// 4-bit tiles: raw (lo | hi << 4) bytes written by the BFS -> nib_encode bytes
cudaError_t launch_nib_encode(uint8_t* D, size_t bytes, cudaStream_t s);
cudaError_t launch_hop_rows(const uint8_t* D, int hb, int nb, int64_t t0, int64_t t1, const int* rows, int nrows,
                            int n, uint16_t* out, int* missing, cudaStream_t s);
// sum of rank partials (world x len doubles, rank order) into out0/out1 split at D of C
cudaError_t launch_slice_sum(const double* recv, int world, int64_t elems, double* out, cudaStream_t s);
cudaError_t launch_slice_unpack(const double* gath, int world, int64_t rslice, int64_t rows, int C, int D, int inter,
                                double* out0, double* out1, cudaStream_t s);
cudaError_t launch_stress_ranks(const double* parts, int64_t stride, int world, int nsets, DevScalars* sc, int set_cur,
                                cudaStream_t s);
cudaError_t launch_set_sigma_rows(const double* diag, int n, DevScalars* sc, cudaStream_t s);

}  // namespace fdl
