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

namespace fdl {

// ------------------------------------------------------------ tiling
constexpr int kWarps = 4;          // warps per P1/P2 CTA
constexpr int kThreads = 32 * kWarps;
constexpr int kRPT = 2;            // rows per thread
constexpr int kBM = 32 * kWarps * kRPT;  // 256 rows per work item (= FDL_ROW_BLOCK)
constexpr int kRowGroup = 32;      // rows per tile-major row group
constexpr int kVecBytes = 16;      // bytes per (row, column-vector) cell
constexpr int kCellBytes = kRowGroup * kVecBytes;  // 512 B block = 32 rows x 16 B
constexpr int kColPad = 128;       // columns padded to this multiple
constexpr int kStages = 4;         // TMA pipeline depth
constexpr int kRB = 256;           // row block of all fp64 reductions (global-aligned)
constexpr int kBFSWords = 32;      // MS-BFS source batch = 32 words x 32 bits = 1024

// columns per j-tile: keeps the D tile at kBM x kBN x hop_bytes = 16 KB
__host__ __device__ constexpr int bn_for(int hb) { return hb == 1 ? 64 : 32; }

// Tile-major hop matrix: row group g (32 rows), column vector c (16 B worth of
// columns: 16 u8 or 8 u16), lane-major inside the 512-B cell.
__host__ __device__ inline size_t d_offset(int64_t lrow, int64_t col, int64_t Np, int hb)
{
    const int64_t V = kVecBytes / hb;
    return (size_t)(((lrow / kRowGroup) * (Np / V) + col / V) * kCellBytes +
                     (lrow % kRowGroup) * kVecBytes + (col % V) * hb);
}

// Per-launch arguments of the all-pairs kernels.
struct PairArgs {
    const uint8_t* D;      // tile-major hops of the local rows
    const float* pos;      // P1: positions, stride ps floats; P2: p vector, stride ps
    double* part;          // partials [NC][ncomp][Mrows]
    const float* lut;      // P2 u8: w'_h = 1/h^2 (fp32), 256 entries
    int64_t Np;            // padded columns
    int n;                 // vertices
    int row0;              // first global row owned
    int nloc;              // rows owned
    int Mrows;             // padded local rows (multiple of kBM)
    int CK;                // column chunk (multiple of kColPad)
    int NC;                // chunks = ceil(n / CK)
    int nrb;               // local row blocks = Mrows / kBM
    int ps;                // float stride of pos per vertex
};

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
    double sigma;          // regularisation weight: (L + sigma 1 1^T), sigma = mean(diag)/n
    int active[4];
    int done;
    int cg_iters;
    double relres;
    unsigned int anynew;   // MS-BFS level flag
};

// Host-mapped mirror the host reads after a stream sync.
struct HostScalars {
    volatile int done;
    volatile unsigned int anynew;
};

// ------------------------------------------------------------ launchers
// All launchers enqueue on `s` and return the CUDA error of the launch.
cudaError_t launch_p1(const PairArgs& a, int dim, int nsets, int hb, int grid, cudaStream_t s);
cudaError_t launch_p2(const PairArgs& a, int dim, int hb, int grid, cudaStream_t s);
int p1_max_ctas(int dim, int nsets, int hb, int device);   // resident CTAs per SM
int p2_max_ctas(int dim, int hb, int device);

// Sum chunk partials of P1 into R_s (scaled) and per-row stress, block stress partials.
cudaError_t launch_p1_reduce(const double* part, int NC, int Mrows, int nloc, int row0, int dim,
                             int nsets, double* R0, double* R1, double* blk_f, int nblk_global,
                             cudaStream_t s);
// Sum f block partials (fixed order) into sc->f_set[0..nsets).
cudaError_t launch_stress_finalize(const double* blk_f, int nblk, int nsets, DevScalars* sc,
                                   int set_cur, cudaStream_t s);

// MS-BFS
cudaError_t launch_bfs_init(uint32_t* frontier, uint32_t* visited, int n, int s0, cudaStream_t s);
cudaError_t launch_bfs_level(const int64_t* row_ptr, const int32_t* col, const uint32_t* fin,
                             uint32_t* fout, uint32_t* visited, uint8_t* D, int n, int s0, int nsrc,
                             int level, int row0, int row1, int64_t Np, int hb, unsigned int* anynew,
                             cudaStream_t s);
cudaError_t launch_diag(const uint8_t* D, int64_t Np, int hb, int n, int nloc, int row0, double* diag,
                        double* blk, cudaStream_t s);
cudaError_t launch_set_sigma(const double* blk, int nblk, int n, DevScalars* sc, cudaStream_t s);

// staging / vector kernels (dim columns, local rows, global row = row0 + lr)
cudaError_t launch_stage_pos1(const double* X, float* posf, int nloc, int row0, int dim, int ps,
                              cudaStream_t s);
cudaError_t launch_combine(const double* Xk, double* Xn, double* Xt, float* posf, double* blk_max,
                           const double* xpin, int nloc, int row0, int dim, double omega, double cap,
                           int nsets, int ps, cudaStream_t s);
cudaError_t launch_get_pin(const double* x, double* slots, int rank, int dim, int owns_row0, cudaStream_t s);
cudaError_t launch_select(double* Xk, double* Rk, const double* Xn, const double* Xt, const double* R1,
                          const double* R2, const double* blk_f, const double* blk_max, int nblk,
                          int nloc, int dim, int nsets, DevScalars* sc, cudaStream_t s);
cudaError_t launch_cg_begin(const double* Xk, double* x, float* pvec, int nloc, int row0, int dim,
                            int pq, cudaStream_t s);
cudaError_t launch_cg_init(const double* part, int NC, int Mrows, const double* b, const double* x,
                           const double* diag, double* r, double* z, double* p, float* pvec,
                           double* blk, int nblk, int nloc, int row0, int dim, int pq, cudaStream_t s);
cudaError_t launch_cg_ap(const double* part, int NC, int Mrows, const double* p, double* y, double* blk,
                         int nblk, int nloc, int row0, int dim, const DevScalars* sc, cudaStream_t s);
cudaError_t launch_cg_update(double* x, double* r, double* z, const double* p, const double* y,
                             const double* diag, double* blk, int nblk, const DevScalars* sc, int nloc,
                             int row0, int dim, cudaStream_t s);
cudaError_t launch_cg_p(double* p, const double* z, float* pvec, const DevScalars* sc, int nloc, int row0,
                        int dim, int pq, cudaStream_t s);
// mode 0: after init (rz, rr, bb); 1: alpha from pAp; 2: beta + convergence
cudaError_t launch_cg_finalize(const double* blk, int nblk, int dim, int mode, double rtol,
                               DevScalars* sc, HostScalars* hs, cudaStream_t s);
cudaError_t launch_reduce_rows(const double* part, int NC, int Mrows, int nloc, int dim, double* out,
                               cudaStream_t s);
cudaError_t launch_ffma_bench(float* out, int iters, int blocks, int threads, cudaStream_t s);

}  // namespace fdl
