// fdl_kernels.cu -- fp64 vector kernels of the hot path (sm_100a): MS-BFS
// initialisation, staging of the fp32 pair-pass inputs, PCG vector updates and
// scalar steps, pinning, the SOR combine (Eq. 10) and the guard of Algorithm 2.
// The all-pairs passes and the BFS level kernel live in fdl_sym.cu.
//
// Determinism: every reduction has a fixed order independent of the launch:
// warp xor-butterfly -> 8 warps in order -> 256-row blocks in global order.
#include <cfloat>
#include <cstdint>

#include "fdl_internal.h"

namespace fdl {

// Deterministic block sum of one double per thread (256 threads); result in
// thread 0.  Warp xor-butterfly, then warps in order.
__device__ __forceinline__ double block_sum_256(double v, double* red /* >= 8 */)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += red[k];
    return s;
}

__device__ __forceinline__ double block_max_256(double v, double* red)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s = fmax(s, red[k]);
    return s;
}

__global__ void k_bfs_init(uint32_t* frontier, uint32_t* visited, int n, int s0)
{
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)n * kBFSWords) return;
    const int v = (int)(idx / kBFSWords), w = (int)(idx % kBFSWords);
    uint32_t val = 0;
    const int d = v - s0;
    if (d >= 0 && d < 32 * kBFSWords && (d >> 5) == w) val = 1u << (d & 31);
    frontier[idx] = val;
    visited[idx] = val;
}

cudaError_t launch_bfs_init(uint32_t* frontier, uint32_t* visited, int n, int s0, cudaStream_t s)
{
    const int64_t total = (int64_t)n * kBFSWords;
    k_bfs_init<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(frontier, visited, n, s0);
    return cudaGetLastError();
}


// ====================================================== vector kernels (fp64)
__global__ void k_stage_pos1(const double* __restrict__ X, float* posf, int nloc, int row0, int dim, int ps)
{
    const int lr = blockIdx.x * blockDim.x + threadIdx.x;
    if (lr >= nloc) return;
    const int64_t g = stage_slot((int64_t)row0 + lr);
    for (int q = 0; q < ps; ++q) posf[g * ps + q] = q < dim ? (float)X[(size_t)lr * dim + q] : 0.0f;
}

cudaError_t launch_stage_pos1(const double* X, float* posf, int nloc, int row0, int dim, int ps, cudaStream_t s)
{
    k_stage_pos1<<<(nloc + kRB - 1) / kRB, kRB, 0, s>>>(X, posf, nloc, row0, dim, ps);
    return cudaGetLastError();
}

// Pin: X^{k+1} <- x - x_0 ("always taking x_1 = 0").  Then Eq. 10:
// Xt = (1 + w) X^{k+1} - w X^k, optional per-vertex cap of
// ||Xt_i - X^{k+1}_i|| (DESIGN R14), staging of the P1 input and the
// max-displacement diagnostic.  xpin = x_0 of the CG solution.
__global__ void __launch_bounds__(kRB) k_combine(const double* __restrict__ Xk, double* __restrict__ Xn,
                                                 double* __restrict__ Xt, float* posf, double* blk_max,
                                                 const double* __restrict__ xpin, int nloc, int row0, int dim,
                                                 double omega, const double* __restrict__ omega_v, double cap,
                                                 int nsets, int ps)
{
    __shared__ double red[8];
    const int lr = blockIdx.x * kRB + threadIdx.x;
    double disp2 = 0.0;
    if (lr < nloc) {
        const int64_t g = stage_slot((int64_t)row0 + lr);
        if (omega_v) omega = omega_v[row0 + lr];  // per-vertex relax factor
        double v[3], xn[3], n2 = 0.0;
        for (int q = 0; q < dim; ++q) {
            xn[q] = Xn[(size_t)lr * dim + q] - xpin[q];
            Xn[(size_t)lr * dim + q] = xn[q];
            const double xk = Xk[(size_t)lr * dim + q];
            const double dq = xn[q] - xk;
            disp2 += dq * dq;
            v[q] = (1.0 + omega) * xn[q] - omega * xk - xn[q];  // Xt - X^{k+1}
            n2 += v[q] * v[q];
        }
        double sc = 1.0;
        if (cap < INFINITY && n2 > cap * cap) sc = cap / sqrt(n2);
        for (int q = 0; q < dim; ++q) {
            const double xt = (sc == 1.0) ? (1.0 + omega) * xn[q] - omega * Xk[(size_t)lr * dim + q]
                                          : xn[q] + sc * v[q];
            Xt[(size_t)lr * dim + q] = xt;
            if (nsets == 2) {  // sets interleaved per component: {x_n, x_t} pairs for the packed P1
                posf[g * ps + 2 * q] = (float)xn[q];
                posf[g * ps + 2 * q + 1] = (float)xt;
            } else {
                posf[g * ps + q] = (float)xn[q];
            }
        }
        for (int q = nsets * dim; q < ps; ++q) posf[g * ps + q] = 0.0f;
    }
    const double m = block_max_256(disp2, red);
    if (threadIdx.x == 0) blk_max[blockIdx.x] = m;
}

cudaError_t launch_combine(const double* Xk, double* Xn, double* Xt, float* posf, double* blk_max,
                           const double* xpin, int nloc, int row0, int dim, double omega, const double* omega_v,
                           double cap, int nsets, int ps, cudaStream_t s)
{
    k_combine<<<(nloc + kRB - 1) / kRB, kRB, 0, s>>>(Xk, Xn, Xt, posf, blk_max, xpin, nloc, row0, dim, omega,
                                                     omega_v, cap, nsets, ps);
    return cudaGetLastError();
}

// ------------------------------------------------------ enumerating strategy
// Pin X^{k+1} (x_0 = 0) and stage {x'(dim), D(dim)} per vertex for
// k_enum, D = X^{k+1} - X^k; block maxima of |D_i|^2 (maxdisp diagnostic).
__global__ void __launch_bounds__(kRB) k_enum_stage(const double* __restrict__ Xk, double* Xn, float* posf,
                                                    double* blk_max, const double* __restrict__ xpin, int n,
                                                    int dim, int ps)
{
    __shared__ double red[8];
    const int i = blockIdx.x * kRB + threadIdx.x;
    double disp2 = 0.0;
    if (i < n) {
        const int64_t g = stage_slot(i);
        for (int q = 0; q < dim; ++q) {
            const size_t k = (size_t)i * dim + q;
            const double xn = Xn[k] - xpin[q];
            Xn[k] = xn;
            const double dq = xn - Xk[k];
            disp2 += dq * dq;
            posf[g * ps + q] = (float)xn;
            posf[g * ps + ps / 2 + q] = (float)dq;
        }
        for (int q = dim; q < ps / 2; ++q) posf[g * ps + q] = posf[g * ps + ps / 2 + q] = 0.0f;
    }
    const double m = block_max_256(disp2, red);
    if (threadIdx.x == 0) blk_max[blockIdx.x] = m;
}

cudaError_t launch_enum_stage(const double* Xk, double* Xn, float* posf, double* blk_max, const double* xpin, int n,
                              int dim, int ps, cudaStream_t s)
{
    k_enum_stage<<<(n + kRB - 1) / kRB, kRB, 0, s>>>(Xk, Xn, posf, blk_max, xpin, n, dim, ps);
    return cudaGetLastError();
}

// omega* = the first (smallest) argmin of the candidates' stresses (lines
// 286-288; ties to the smaller omega).  Candidate 0 is omega = 0.
__global__ void k_enum_pick(const double* __restrict__ fs, int m, double step, DevScalars* sc)
{
    if (threadIdx.x != 0) return;
    int best = 0;
    for (int c = 1; c < m; ++c)
        if (fs[c] < fs[best]) best = c;
    sc->omega_star = step * best;
    sc->enum_best = best;
    sc->enum_f0 = fs[0];
    sc->enum_fbest = fs[best];
}

cudaError_t launch_enum_pick(const double* fs, int m, double step, DevScalars* sc, cudaStream_t s)
{
    k_enum_pick<<<1, 32, 0, s>>>(fs, m, step, sc);
    return cudaGetLastError();
}

// X~ = X^{k+1} + w* (X^{k+1} - X^k), L^W X~ = (1 + w*) L^W X^{k+1} - w* L^W X^k
// (carried, L linear), staged fp32 X~ for the P1 pass of the chosen point.
__global__ void k_enum_apply(const double* __restrict__ Xn, const double* __restrict__ Xk,
                             const double* __restrict__ An, const double* __restrict__ Ak, double* Xt, double* At,
                             float* posf, const DevScalars* __restrict__ sc, int n, int dim, int ps)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double w = sc->omega_star;
    const int64_t g = stage_slot(i);
    for (int q = 0; q < dim; ++q) {
        const size_t k = (size_t)i * dim + q;
        const double xt = w == 0.0 ? Xn[k] : (1.0 + w) * Xn[k] - w * Xk[k];
        Xt[k] = xt;
        At[k] = w == 0.0 ? An[k] : (1.0 + w) * An[k] - w * Ak[k];
        posf[g * ps + q] = (float)xt;
    }
    for (int q = dim; q < ps; ++q) posf[g * ps + q] = 0.0f;
}

cudaError_t launch_enum_apply(const double* Xn, const double* Xk, const double* An, const double* Ak, double* Xt,
                              double* At, float* posf, const DevScalars* sc, int n, int dim, int ps, cudaStream_t s)
{
    k_enum_apply<<<(n + 255) / 256, 256, 0, s>>>(Xn, Xk, An, Ak, Xt, At, posf, sc, n, dim, ps);
    return cudaGetLastError();
}

// x_0 of the CG solution (global row 0 lives on the rank with row0 == 0) into
// slot `rank` of a world x 4 buffer (all-gathered across ranks afterwards).
__global__ void k_get_pin(const double* __restrict__ x, double* slots, int rank, int dim, int owns_row0)
{
    const int q = threadIdx.x;
    if (q < 4) slots[rank * 4 + q] = (owns_row0 && q < dim) ? x[q] : 0.0;
}

cudaError_t launch_get_pin(const double* x, double* slots, int rank, int dim, int owns_row0, cudaStream_t s)
{
    k_get_pin<<<1, 32, 0, s>>>(x, slots, rank, dim, owns_row0);
    return cudaGetLastError();
}

// Carried L^W X: the PCG recursion gives (L + sigma 1 1^T) d =
// r0 - r_cg with d = x - x0 and r0 = Rk - Ak, so L x = Rk - r_cg - sigma (sum d) 1;
// L is linear, so L Xt = (1 + w) L X^{k+1} - w L X^k.  (The pin x_0 = 0 is a
// translation: L 1 = 0.)
__global__ void k_carry_a(const double* __restrict__ Rk, const double* __restrict__ rcg,
                          const double* __restrict__ Ak, double* An, double* At, const DevScalars* __restrict__ sc,
                          int n, int dim, double omega)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    for (int q = 0; q < dim; ++q) {
        const size_t k = (size_t)i * dim + q;
        const double an = Rk[k] - rcg[k] - sc->sigma * sc->Sd[q];
        An[k] = an;
        At[k] = (1.0 + omega) * an - omega * Ak[k];
    }
}

cudaError_t launch_carry_a(const double* Rk, const double* rcg, const double* Ak, double* An, double* At,
                           const DevScalars* sc, int n, int dim, double omega, cudaStream_t s)
{
    k_carry_a<<<(n + kRB - 1) / kRB, kRB, 0, s>>>(Rk, rcg, Ak, An, At, sc, n, dim, omega);
    return cudaGetLastError();
}

// Guard of Algorithm 2 lines 6-8: accept Xt iff f(Xt) <= f(X^{k+1}) (ties
// accept, raw comparison).  Copies the accepted placement, its R and (when
// carried) its L^W X.
__global__ void __launch_bounds__(kRB) k_select(double* Xk, double* Rk, const double* __restrict__ Xn,
                                                const double* __restrict__ Xt, const double* __restrict__ R1,
                                                const double* __restrict__ R2, const double* __restrict__ blk_max,
                                                int nblk_loc, int nloc, int dim, int nsets, DevScalars* sc,
                                                double* Ak, const double* __restrict__ An,
                                                const double* __restrict__ At)
{
    const double f0 = sc->f_set[0];
    const double f1 = nsets == 2 ? sc->f_set[1] : f0;
    const bool accept = nsets == 2 && (f1 <= f0);
    const int lr = blockIdx.x * kRB + threadIdx.x;
    if (lr < nloc) {
        for (int q = 0; q < dim; ++q) {
            const size_t i = (size_t)lr * dim + q;
            Xk[i] = accept ? Xt[i] : Xn[i];
            Rk[i] = accept ? R2[i] : R1[i];
            if (Ak) Ak[i] = accept ? At[i] : An[i];
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < 32) {
        // max of the block maxima by warp 0 (fmax is exact, so any order gives the same value;
        // one thread walking C5's 782 maxima took ~30 us)
        double m = 0.0;
        for (int b = threadIdx.x; b < nblk_loc; b += 32) m = fmax(m, blk_max[b]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (threadIdx.x != 0) return;
        sc->maxdisp = sqrt(m);
        sc->f_next = f0;
        sc->f_relaxed = nsets == 2 ? f1 : NAN;
        sc->accepted = accept ? 1 : 0;
        const double fc = accept ? f1 : f0;
        sc->f_cur = fc;
        sc->nonfinite = !isfinite(fc);
    }
}

cudaError_t launch_select(double* Xk, double* Rk, const double* Xn, const double* Xt, const double* R1,
                          const double* R2, const double* blk_max, int nloc, int dim, int nsets, DevScalars* sc,
                          double* Ak, const double* An, const double* At, cudaStream_t s)
{
    const int nb = (nloc + kRB - 1) / kRB;
    k_select<<<nb, kRB, 0, s>>>(Xk, Rk, Xn, Xt, R1, R2, blk_max, nb, nloc, dim, nsets, sc, Ak, An, At);
    return cudaGetLastError();
}

// ------------------------------------------------------------------- PCG
// Jacobi-preconditioned CG on Eq. 5, L^W X = L^{X^k} X^k, over all n rows
// (consistent singular system: L^W 1 = 0 and sum_i (L^X X)_i = 0).  CG from a
// warm start converges to a solution of Eq. 5; the translation is fixed
// afterwards by x_0 = 0 in k_combine.  The result is the paper's
// X^{k+1} (unique up to translation); the gauge is chosen after the
// solve instead of by deleting row/column 0, which removes the small
// eigenvalue mean_i w_i0 that pinning introduces (R7).
// All d columns at once with per-column scalars (the d systems of Eq. 2-5
// are independent).
// The correction d = x - x0 solves (L + sigma 1 1^T) d = r0 with r0 = b - L x0:
// r0 is orthogonal to 1 (up to rounding), so d is the zero-mean solution of
// L d = r0 and the rank-one term only makes the operator nonsingular (fp32
// rounding leaves sum_i r_i != 0 otherwise, an unreachable residual floor).
// sum_i p_i is carried by the recurrence S <- sum z + beta S.
// Extrapolated PCG start (DESIGN R23): x0 = X^k + rho (X^k - X^{k-1}),
// L^W x0 = A^k + rho (A^k - A^{k-1}) from the carried products (L linear), so
// no extra pass.  rho is the previous step's least-squares ratio of successive
// corrections (k_rho); valid = 0 -> x0 = X^k.  The solve's result is the same
// minimiser (Eq. 4) to the CG tolerance; only the start changes.
__global__ void k_extrap(const double* __restrict__ Xk, const double* __restrict__ Xprev,
                         const double* __restrict__ Ak, const double* __restrict__ Aprev, double* x, double* y0,
                         const DevScalars* __restrict__ sc, int n, int dim, int valid)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double rho = valid ? sc->rho : 0.0;
    for (int q = 0; q < dim; ++q) {
        const size_t k = (size_t)i * dim + q;
        x[k] = Xk[k] + rho * (Xk[k] - Xprev[k]);
        y0[k] = Ak[k] + rho * (Ak[k] - Aprev[k]);
    }
}

cudaError_t launch_extrap(const double* Xk, const double* Xprev, const double* Ak, const double* Aprev, double* x,
                          double* y0, const DevScalars* sc, int n, int dim, int valid, cudaStream_t s)
{
    k_extrap<<<(n + 255) / 256, 256, 0, s>>>(Xk, Xprev, Ak, Aprev, x, y0, sc, n, dim, valid);
    return cudaGetLastError();
}

// Block partials of a = <X^{k+1} - X^k, X^k - X^{k-1}>, b = |X^k - X^{k-1}|^2
// (pinned gauge), then X^{k-1} <- X^k, A^{k-1} <- A^k for the next step.
__global__ void __launch_bounds__(kRB) k_rho(const double* __restrict__ Xn, const double* __restrict__ Xk,
                                             double* Xprev, const double* __restrict__ Ak, double* Aprev,
                                             double* blk, int n, int dim, int nblk, int valid)
{
    __shared__ double red[8];
    const int i = blockIdx.x * kRB + threadIdx.x;
    double a = 0.0, b = 0.0;
    if (i < n) {
        for (int q = 0; q < dim; ++q) {
            const size_t k = (size_t)i * dim + q;
            const double xk = Xk[k], dp = xk - Xprev[k];
            a += (Xn[k] - xk) * dp;
            b += dp * dp;
            Xprev[k] = xk;
            Aprev[k] = Ak[k];
        }
    }
    if (!valid) a = b = 0.0;
    double t = block_sum_256(a, red);
    if (threadIdx.x == 0) blk[blockIdx.x] = t;
    t = block_sum_256(b, red);
    if (threadIdx.x == 0) blk[nblk + blockIdx.x] = t;
}

__global__ void k_rho_finalize(const double* __restrict__ blk, int nblk, DevScalars* sc)
{
    const int lane = threadIdx.x;
    double a = 0.0, b = 0.0;
    for (int k = lane; k < nblk; k += 32) {
        a += blk[k];
        b += blk[nblk + k];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if (lane == 0) sc->rho = b > 0.0 ? fmin(fmax(a / b, 0.0), 1.0) : 0.0;
}

cudaError_t launch_rho(const double* Xn, const double* Xk, double* Xprev, const double* Ak, double* Aprev,
                       double* blk, int n, int dim, int valid, DevScalars* sc, cudaStream_t s)
{
    const int nblk = (n + kRB - 1) / kRB;
    k_rho<<<nblk, kRB, 0, s>>>(Xn, Xk, Xprev, Ak, Aprev, blk, n, dim, nblk, valid);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_rho_finalize<<<1, 32, 0, s>>>(blk, nblk, sc);
    return cudaGetLastError();
}

// Placement units at the ABI: mode 0 (upload) y = (x - x_0) / k, the pin
// x_0 = 0 of P:125 (fp64 subtract, then divide: the same IEEE operations as on the
// host); mode 1 (download) y = x * k.
__global__ void k_pin_scale(const double* __restrict__ x, double* __restrict__ y, int n, int dim, double k, int mode)
{
    const size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= (size_t)n * dim) return;
    y[g] = mode == 0 ? (x[g] - x[g % dim]) / k : x[g] * k;
}

// fdl_set_positions: does the uploaded placement x (original units) differ from the
// context's X^k as fdl_get_positions returns it (X^k * k, bitwise)?  *differs = 1 if so.
__global__ void k_placement_differs(const double* __restrict__ x, const double* __restrict__ Xk, size_t cnt, double k,
                                    unsigned int* differs)
{
    const size_t g = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool d = g < cnt && x[g] != Xk[g] * k;
    if (__any_sync(0xffffffffu, d) && (threadIdx.x & 31) == 0) *differs = 1u;
}

cudaError_t launch_placement_differs(const double* x, const double* Xk, size_t cnt, double k, unsigned int* differs,
                                     cudaStream_t s)
{
    k_placement_differs<<<(unsigned)((cnt + 255) / 256), 256, 0, s>>>(x, Xk, cnt, k, differs);
    return cudaGetLastError();
}

cudaError_t launch_pin_scale(const double* x, double* y, int n, int dim, double k, int mode, cudaStream_t s)
{
    const size_t cnt = (size_t)n * dim;
    k_pin_scale<<<(unsigned)((cnt + 255) / 256), 256, 0, s>>>(x, y, n, dim, k, mode);
    return cudaGetLastError();
}

// ------------------------------------------------ recycled PCG start (R27)
// L^W is the same matrix at every step, so the directions the run already took
// carry over: the start is the Galerkin (A-norm optimal) correction of X^k over
// the span of the last m step differences v_s = X^{j+1} - X^j, whose products
// L^W v_s are differences of the carried L^W X (no extra pair pass):
//   x0 = X^k + V y,  L^W x0 = A^k + (AV) y,  (V^T AV) y = V^T (b - A^k),  per column.
// The solve still runs to cg_rtol from there: only the start changes.
constexpr int kGalNG = kGalMax * (kGalMax + 1) / 2;  // upper-triangle Gram entries (kGalNV: + right-hand sides)

__device__ __forceinline__ double warp_sum_d(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// block partials of G_st = (v_s.av_t + v_t.av_s)/2 (s <= t) and v_s.r, r = b - A^k
__global__ void __launch_bounds__(kRB) k_gal_partial(const double* __restrict__ V, const double* __restrict__ AV,
                                                     const double* __restrict__ b, const double* __restrict__ Ak,
                                                     double* blk, int n, int dim, int nblk,
                                                     const DevScalars* __restrict__ sc)
{
    __shared__ double red[kRB / 32][3 * kGalNV];
    const int cnt = sc->gal_cnt;
    if (cnt == 0) return;  // k_gal_solve does not read the partials
    const int i = blockIdx.x * kRB + threadIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const size_t nd = (size_t)n * dim;
    for (int c = 0; c < dim; ++c) {
        const size_t k = (size_t)i * dim + c;
        double v[kGalMax], av[kGalMax], r = 0.0;
#pragma unroll
        for (int q = 0; q < kGalMax; ++q) {
            v[q] = (i < n && q < cnt) ? V[q * nd + k] : 0.0;
            av[q] = (i < n && q < cnt) ? AV[q * nd + k] : 0.0;
        }
        if (i < n) r = b[k] - Ak[k];
        int e = c * kGalNV;
#pragma unroll
        for (int q = 0; q < kGalMax; ++q)
#pragma unroll
            for (int t = q; t < kGalMax; ++t, ++e) {
                double g = 0.0;
                if (t < cnt) g = warp_sum_d(0.5 * (v[q] * av[t] + v[t] * av[q]));
                if (lane == 0) red[w][e] = g;
            }
#pragma unroll
        for (int q = 0; q < kGalMax; ++q, ++e) {
            double g = 0.0;
            if (q < cnt) g = warp_sum_d(v[q] * r);
            if (lane == 0) red[w][e] = g;
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < dim * kGalNV; e += kRB) {
        double t = 0.0;
        for (int ww = 0; ww < kRB / 32; ++ww) t += red[ww][e];
        blk[(size_t)e * nblk + blockIdx.x] = t;
    }
}

// one block: fixed-order sums of the partials, then per column an LDL^T solve of
// the cnt x cnt Gram system that skips dependent vectors (pivot below 1e-6 of
// the vector's own A-norm: it adds nothing the earlier ones do not span).
__global__ void __launch_bounds__(256) k_gal_solve(const double* __restrict__ blk, int nblk, int dim, DevScalars* sc)
{
    __shared__ double tot[3 * kGalNV];
    const int cnt = sc->gal_cnt;
    for (int e = threadIdx.x; e < dim * kGalNV && cnt > 0; e += blockDim.x) {
        double t = 0.0;
        for (int q0 = 0; q0 < nblk; q0 += 8) {  // in order; 8 loads in flight (+0.0 padding is exact)
            double v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = q0 + k < nblk ? __ldg(blk + (size_t)e * nblk + q0 + k) : 0.0;
#pragma unroll
            for (int k = 0; k < 8; ++k) t += v[k];
        }
        tot[e] = t;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        const int c = threadIdx.x;
        double y[kGalMax];
        int dropped = 0;
        for (int q = 0; q < kGalMax; ++q) y[q] = 0.0;
        if (c < dim && cnt > 0) {
            double G[kGalMax][kGalMax], L[kGalMax][kGalMax], D[kGalMax], z[kGalMax];
            bool keep[kGalMax];
            const double* T = tot + c * kGalNV;
            int e = 0;
            for (int q = 0; q < kGalMax; ++q)
                for (int t = q; t < kGalMax; ++t, ++e) G[q][t] = G[t][q] = T[e];
            for (int q = 0; q < cnt; ++q) {
                double d = G[q][q];
                for (int k = 0; k < q; ++k)
                    if (keep[k]) d -= L[q][k] * L[q][k] * D[k];
                keep[q] = G[q][q] > 0.0 && d > 1e-6 * G[q][q];
                if (!keep[q]) {
                    ++dropped;
                    continue;
                }
                D[q] = d;
                for (int t = q + 1; t < cnt; ++t) {
                    double g = G[t][q];
                    for (int k = 0; k < q; ++k)
                        if (keep[k]) g -= L[t][k] * L[q][k] * D[k];
                    L[t][q] = g / d;
                }
            }
            for (int q = 0; q < cnt; ++q) {
                if (!keep[q]) continue;
                double v = T[kGalNG + q];
                for (int k = 0; k < q; ++k)
                    if (keep[k]) v -= L[q][k] * z[k];
                z[q] = v;
            }
            for (int q = cnt - 1; q >= 0; --q) {
                if (!keep[q]) continue;
                double v = z[q] / D[q];
                for (int t = q + 1; t < cnt; ++t)
                    if (keep[t]) v -= L[t][q] * y[t];
                y[q] = v;
            }
        }
        for (int q = 0; q < kGalMax; ++q) sc->gal_y[c][q] = y[q];
        if (c == 0) sc->gal_dropped = dropped;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        sc->gal_use = cnt;
        sc->gal_cnt = cnt + 1 < sc->gal_m ? cnt + 1 : sc->gal_m;  // after the next step's push
    }
}

__global__ void k_gal_apply(const double* __restrict__ V, const double* __restrict__ AV,
                            const double* __restrict__ Xk, const double* __restrict__ Ak, double* x, double* y0,
                            const DevScalars* __restrict__ sc, int n, int dim)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int use = sc->gal_use;
    const size_t nd = (size_t)n * dim;
    for (int c = 0; c < dim; ++c) {
        const size_t k = (size_t)i * dim + c;
        double xv = Xk[k], yv = Ak[k];
        for (int q = 0; q < use; ++q) {
            const double g = sc->gal_y[c][q];
            xv += g * V[q * nd + k];
            yv += g * AV[q * nd + k];
        }
        x[k] = xv;
        y0[k] = yv;
    }
}

cudaError_t launch_gal_start(const double* V, const double* AV, const double* b, const double* Xk, const double* Ak,
                             double* x, double* y0, double* blk, int nblk, DevScalars* sc, int n, int dim,
                             cudaStream_t s)
{
    k_gal_partial<<<nblk, kRB, 0, s>>>(V, AV, b, Ak, blk, n, dim, nblk, sc);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_gal_solve<<<1, 256, 0, s>>>(blk, nblk, dim, sc);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_gal_apply<<<(n + 255) / 256, 256, 0, s>>>(V, AV, Xk, Ak, x, y0, sc, n, dim);
    return cudaGetLastError();
}

__global__ void k_gal_push(const double* __restrict__ Xk, const double* __restrict__ Xprev,
                           const double* __restrict__ Ak, const double* __restrict__ Aprev, double* V, double* AV,
                           size_t nd, int m)
{
    const size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nd) return;
    for (int q = m - 1; q > 0; --q) {
        V[q * nd + k] = V[(q - 1) * nd + k];
        AV[q * nd + k] = AV[(q - 1) * nd + k];
    }
    V[k] = Xk[k] - Xprev[k];
    AV[k] = Ak[k] - Aprev[k];
}

cudaError_t launch_gal_push(const double* Xk, const double* Xprev, const double* Ak, const double* Aprev, double* V,
                            double* AV, int n, int dim, int m, cudaStream_t s)
{
    const size_t nd = (size_t)n * dim;
    k_gal_push<<<(unsigned)((nd + 255) / 256), 256, 0, s>>>(Xk, Xprev, Ak, Aprev, V, AV, nd, m);
    return cudaGetLastError();
}

// column means of X -> sc->cmean: the centring of the staged P2 input (product form,
// k_p2_finish).  Block partials over kRB rows (warp butterfly, fixed order), then one
// warp sums the blocks in block order: deterministic and independent of the grid.
// (A single 1024-thread block took 0.14 ms per step at C5: it is on the critical path.)
__global__ void k_colmean_part(const double* __restrict__ X, int n, int dim, double* blk)
{
    __shared__ double red[kRB / 32][4];
    const int i = blockIdx.x * kRB + threadIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int q = 0; q < dim; ++q) {
        double v = i < n ? X[(size_t)i * dim + q] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[w][q] = v;
    }
    __syncthreads();
    if (threadIdx.x < dim) {
        double t = 0.0;
        for (int k = 0; k < kRB / 32; ++k) t += red[k][threadIdx.x];
        blk[(size_t)blockIdx.x * 4 + threadIdx.x] = t;
    }
}

__global__ void k_colmean_fin(const double* __restrict__ blk, int nblk, int n, int dim, DevScalars* sc)
{
    const int lane = threadIdx.x;
    for (int q = 0; q < dim; ++q) {
        double v = 0.0;
        for (int b = lane; b < nblk; b += 32) v += blk[(size_t)b * 4 + q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) sc->cmean[q] = v / n;
    }
}

__global__ void k_cg_begin(const double* __restrict__ Xk, double* x, float* pvec, int nloc, int row0, int dim,
                           int pq, const DevScalars* __restrict__ sc)
{
    const int lr = blockIdx.x * blockDim.x + threadIdx.x;
    if (lr >= nloc) return;
    const int64_t g = stage_slot((int64_t)row0 + lr);
    for (int q = 0; q < pq; ++q) {
        double v = 0.0;
        if (q < dim) {
            v = Xk[(size_t)lr * dim + q];
            x[(size_t)lr * dim + q] = v;
            v -= sc->cmean[q];
        }
        pvec[g * pq + q] = (float)v;
    }
}

// fp32 staging of the first PCG direction p = z, centred by sum(p)/n (sc->S
// after cg_finalize mode 0)
__global__ void k_stage_p(const double* __restrict__ p, float* pvec, const DevScalars* __restrict__ sc, int n,
                          int dim, int pq)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t g = stage_slot(i);
    for (int q = 0; q < pq; ++q)
        pvec[g * pq + q] = q < dim ? (float)(p[(size_t)i * dim + q] - sc->S[q] * sc->inv_n) : 0.0f;
}

cudaError_t launch_stage_p(const double* p, float* pvec, const DevScalars* sc, int n, int dim, int pq,
                           cudaStream_t s)
{
    k_stage_p<<<(n + 255) / 256, 256, 0, s>>>(p, pvec, sc, n, dim, pq);
    return cudaGetLastError();
}

// out_i = diag_i p'_i - S_i: the L^W matvec from the product-form pair sums
// S_i = sum_j w_ij p'_j, with p' the same centred fp32 values the pass read.
__global__ void k_p2_finish(double* out, const float* __restrict__ pvec, const double* __restrict__ diag, int n,
                            int dim, int pq)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t g = stage_slot(i);
    const double d = diag[i];
    for (int q = 0; q < dim; ++q) {
        const size_t k = (size_t)i * dim + q;
        out[k] = d * (double)pvec[g * pq + q] - out[k];
    }
}

cudaError_t launch_p2_finish(double* out, const float* pvec, const double* diag, int n, int dim, int pq,
                             cudaStream_t s)
{
    k_p2_finish<<<(n + 255) / 256, 256, 0, s>>>(out, pvec, diag, n, dim, pq);
    return cudaGetLastError();
}

cudaError_t launch_cg_begin(const double* Xk, double* x, float* pvec, int nloc, int row0, int dim, int pq,
                            DevScalars* sc, double* blk, cudaStream_t s)
{
    const int nblk = (nloc + kRB - 1) / kRB;
    k_colmean_part<<<nblk, kRB, 0, s>>>(Xk, nloc, dim, blk);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_colmean_fin<<<1, 32, 0, s>>>(blk, nblk, nloc, dim, sc);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_cg_begin<<<(nloc + kRB - 1) / kRB, kRB, 0, s>>>(Xk, x, pvec, nloc, row0, dim, pq, sc);
    return cudaGetLastError();
}

// r = b - L x0 (y = L x0 from the symmetric P2 pass), z = r / diag, p = z;
// block partials of r.z, r.r, b.b and sum z.
__global__ void __launch_bounds__(kRB) k_cg_init(const double* __restrict__ y, const double* __restrict__ b,
                                                 const double* __restrict__ diag, double* r, double* z, double* p,
                                                 float* pvec, double* blk, int n, int dim, int pq, int nblk)
{
    __shared__ double red[8];
    const int i = blockIdx.x * kRB + threadIdx.x;
    double rz[3] = {0, 0, 0}, rr[3] = {0, 0, 0}, bb[3] = {0, 0, 0}, zs[3] = {0, 0, 0};
    if (i < n) {
        for (int q = 0; q < dim; ++q) {
            const size_t k = (size_t)i * dim + q;
            const double bv = b[k];
            const double rv = bv - y[k];
            const double zv = rv / diag[i];
            r[k] = rv;
            z[k] = zv;
            p[k] = zv;
            rz[q] = rv * zv;
            rr[q] = rv * rv;
            bb[q] = bv * bv;
            zs[q] = zv;
        }
    }
    for (int q = 0; q < dim; ++q) {
        double t = block_sum_256(rz[q], red);
        if (threadIdx.x == 0) blk[(size_t)(0 * 4 + q) * nblk + blockIdx.x] = t;
        t = block_sum_256(rr[q], red);
        if (threadIdx.x == 0) blk[(size_t)(1 * 4 + q) * nblk + blockIdx.x] = t;
        t = block_sum_256(bb[q], red);
        if (threadIdx.x == 0) blk[(size_t)(2 * 4 + q) * nblk + blockIdx.x] = t;
        t = block_sum_256(zs[q], red);
        if (threadIdx.x == 0) blk[(size_t)(3 * 4 + q) * nblk + blockIdx.x] = t;
    }
}

cudaError_t launch_cg_init(const double* y, const double* b, const double* diag, double* r, double* z, double* p,
                           float* pvec, double* blk, int nblk, int n, int dim, int pq, cudaStream_t s)
{
    k_cg_init<<<(n + kRB - 1) / kRB, kRB, 0, s>>>(y, b, diag, r, z, p, pvec, blk, n, dim, pq, nblk);
    return cudaGetLastError();
}

// y <- L p + sigma (sum p) 1 (rank-one term of the regularised operator, R7);
// block partials of p.y
__global__ void __launch_bounds__(kRB) k_cg_ap(const double* __restrict__ p, double* y, double* blk, int n, int dim,
                                               int nblk, const DevScalars* __restrict__ sc)
{
    __shared__ double red[8];
    const int i = blockIdx.x * kRB + threadIdx.x;
    double py[3] = {0, 0, 0};
    if (i < n) {
        for (int q = 0; q < dim; ++q) {
            const size_t k = (size_t)i * dim + q;
            const double yv = y[k] + sc->sigma * sc->S[q];
            y[k] = yv;
            py[q] = p[k] * yv;
        }
    }
    for (int q = 0; q < dim; ++q) {
        const double t = block_sum_256(py[q], red);
        if (threadIdx.x == 0) blk[(size_t)q * nblk + blockIdx.x] = t;
    }
}

cudaError_t launch_cg_ap(const double* p, double* y, double* blk, int nblk, int n, int dim, const DevScalars* sc,
                         cudaStream_t s)
{
    k_cg_ap<<<(n + kRB - 1) / kRB, kRB, 0, s>>>(p, y, blk, n, dim, nblk, sc);
    return cudaGetLastError();
}

__global__ void __launch_bounds__(kRB) k_cg_update(double* x, double* r, double* z, const double* __restrict__ p,
                                                   const double* __restrict__ y, const double* __restrict__ diag,
                                                   double* blk, const DevScalars* __restrict__ sc, int nloc,
                                                   int row0, int dim, int nblk)
{
    __shared__ double red[8];
    const int lr = blockIdx.x * kRB + threadIdx.x;
    double rz[3] = {0, 0, 0}, rr[3] = {0, 0, 0}, zs[3] = {0, 0, 0};
    if (lr < nloc) {
        for (int q = 0; q < dim; ++q) {
            const size_t i = (size_t)lr * dim + q;
            const double al = sc->alpha[q];
            const double xv = x[i] + al * p[i];
            const double rv = r[i] - al * y[i];
            const double zv = rv / diag[lr];
            x[i] = xv;
            r[i] = rv;
            z[i] = zv;
            rz[q] = rv * zv;
            rr[q] = rv * rv;
            zs[q] = zv;
        }
    }
    const int gb = row0 / kRB + blockIdx.x;
    for (int q = 0; q < dim; ++q) {
        double t = block_sum_256(rz[q], red);
        if (threadIdx.x == 0) blk[(size_t)(0 * 4 + q) * nblk + gb] = t;
        t = block_sum_256(rr[q], red);
        if (threadIdx.x == 0) blk[(size_t)(1 * 4 + q) * nblk + gb] = t;
        t = block_sum_256(zs[q], red);
        if (threadIdx.x == 0) blk[(size_t)(3 * 4 + q) * nblk + gb] = t;
    }
}

cudaError_t launch_cg_update(double* x, double* r, double* z, const double* p, const double* y, const double* diag,
                             double* blk, int nblk, const DevScalars* sc, int nloc, int row0, int dim, cudaStream_t s)
{
    const int nb = (nloc + kRB - 1) / kRB;
    k_cg_update<<<nb, kRB, 0, s>>>(x, r, z, p, y, diag, blk, sc, nloc, row0, dim, nblk);
    return cudaGetLastError();
}

__global__ void k_cg_p(double* p, const double* __restrict__ z, float* pvec, const DevScalars* __restrict__ sc,
                       int nloc, int row0, int dim, int pq)
{
    const int lr = blockIdx.x * blockDim.x + threadIdx.x;
    if (lr >= nloc) return;
    const int64_t g = stage_slot((int64_t)row0 + lr);
    for (int q = 0; q < dim; ++q) {
        const size_t i = (size_t)lr * dim + q;
        double pv = p[i];
        if (sc->active[q]) pv = z[i] + sc->beta[q] * pv;
        p[i] = pv;
        pvec[g * pq + q] = (float)(pv - sc->S[q] * sc->inv_n);  // centred (k_p2_finish)
    }
}

cudaError_t launch_cg_p(double* p, const double* z, float* pvec, const DevScalars* sc, int nloc, int row0, int dim,
                        int pq, cudaStream_t s)
{
    k_cg_p<<<(nloc + kRB - 1) / kRB, kRB, 0, s>>>(p, z, pvec, sc, nloc, row0, dim, pq);
    return cudaGetLastError();
}

// Scalar step of PCG from block partials (summed in global block order by
// one warp, fixed butterfly).  Slots: 0 r.z | p.y (mode 1), 1 r.r, 2 b.b,
// 3 sum z.  mode 0: init; 1: alpha; 2: beta + stop test.
// Scalar PCG step by one warp (lane = threadIdx.x & 31 of warp 0 of the block).
__device__ __forceinline__ void cg_finalize_warp(const double* __restrict__ blk, int nblk, int dim, int mode,
                                                 double rtol, DevScalars* sc, HostScalars* hs,
                                                 cudaGraphConditionalHandle cond, int use_cond, int cg_max)
{
    const int lane = threadIdx.x & 31;
    // per (quantity, column): the lane's partials b = lane, lane + 32, ... summed in that
    // order, then a butterfly.  The loads of a chunk of 4 x 32 partials of every array are
    // staged in registers before the adds, so they are in flight together (a dependent L2
    // round trip per partial made this ~15 us at C5's 782 blocks); the +0.0 padding past
    // nblk leaves the sums bitwise unchanged (they start at +0.0 and never become -0.0)
    const bool use[4] = {true, mode != 1, mode == 0, mode != 1};
    double sums[4][3];
#pragma unroll
    for (int qq = 0; qq < 4; ++qq)
#pragma unroll
        for (int c = 0; c < 3; ++c) sums[qq][c] = 0.0;
    for (int b0 = lane; b0 < nblk; b0 += 4 * 32) {
        double v[4][3][4];
#pragma unroll
        for (int qq = 0; qq < 4; ++qq)
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int bb = b0 + 32 * k;
                    v[qq][c][k] = (use[qq] && c < dim && bb < nblk) ? __ldg(blk + (size_t)(qq * 4 + c) * nblk + bb) : 0.0;
                }
#pragma unroll
        for (int qq = 0; qq < 4; ++qq)
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int k = 0; k < 4; ++k) sums[qq][c] += v[qq][c][k];
    }
#pragma unroll
    for (int qq = 0; qq < 4; ++qq)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            double t = sums[qq][c];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
            sums[qq][c] = t;
        }
    if (lane != 0) return;
    const double rt2 = rtol * rtol;
    if (mode == 0) {
        int any = 0;
        double rel = 0.0;
        for (int c = 0; c < dim; ++c) {
            sc->rz[c] = sums[0][c];
            sc->rr[c] = sums[1][c];
            sc->bb[c] = sums[2][c];
            sc->S[c] = sums[3][c];
            sc->Sd[c] = 0.0;
            const int act = sums[1][c] > rt2 * sums[2][c];
            sc->active[c] = act;
            any |= act;
            rel = fmax(rel, sums[2][c] > 0 ? sqrt(sums[1][c] / sums[2][c]) : 0.0);
        }
        sc->done = !any;
        sc->cg_iters = 0;
        sc->relres = rel;
        hs->done = !any;
        if (use_cond) cudaGraphSetConditional(cond, (any && cg_max > 0) ? 1u : 0u);  // WHILE node of the step graph
    } else if (mode == 1) {
        for (int c = 0; c < dim; ++c) {
            sc->pap[c] = sums[0][c];
            sc->alpha[c] = (sc->active[c] && sums[0][c] > 0.0) ? sc->rz[c] / sums[0][c] : 0.0;
            sc->Sd[c] += sc->alpha[c] * sc->S[c];  // x += alpha p  =>  sum d += alpha sum p
        }
    } else {
        int any = 0;
        double rel = 0.0;
        for (int c = 0; c < dim; ++c) {
            if (sc->active[c]) {
                const double rzn = sums[0][c];
                const double beta = sc->rz[c] != 0.0 ? rzn / sc->rz[c] : 0.0;
                sc->beta[c] = beta;
                sc->rz[c] = rzn;
                sc->rr[c] = sums[1][c];
                sc->S[c] = sums[3][c] + beta * sc->S[c];  // sum of p = z + beta p
                sc->active[c] = sums[1][c] > rt2 * sc->bb[c];
            }
            any |= sc->active[c];
            rel = fmax(rel, sc->bb[c] > 0 ? sqrt(sc->rr[c] / sc->bb[c]) : 0.0);
        }
        sc->cg_iters += 1;
        sc->done = !any;
        sc->relres = rel;
        hs->done = !any;
        if (use_cond) cudaGraphSetConditional(cond, (any && sc->cg_iters < cg_max) ? 1u : 0u);
    }
}

__global__ void k_cg_finalize(const double* __restrict__ blk, int nblk, int dim, int mode, double rtol,
                              DevScalars* sc, HostScalars* hs, cudaGraphConditionalHandle cond, int use_cond,
                              int cg_max)
{
    cg_finalize_warp(blk, nblk, dim, mode, rtol, sc, hs, cond, use_cond, cg_max);
}

// ---------------------------------------------------------- fused PCG tail
// One PCG iteration after the P2 pass (k_p2_finish, k_cg_ap, finalize 1,
// k_cg_update, finalize 2, k_cg_p) in ONE block of 1024 threads, for small n:
// the 256-row blocks are processed four at a time by the four 256-thread
// quarters with the same per-row arithmetic, the same warp butterflies and the
// same warp and block orders as the separate kernels, so the results are
// bitwise those of the multi-kernel sequence (fewer launches per iteration).
__device__ __forceinline__ double quarter_sum(double v, double* red /* 32 */)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if ((threadIdx.x & 255) == 0) {
        const int w0 = (threadIdx.x >> 8) * 8;
        for (int k = 0; k < 8; ++k) t += red[w0 + k];
    }
    return t;
}

__global__ void __launch_bounds__(1024) k_cg_tail(double* y, const float* __restrict__ pvec_in,
                                                 const double* __restrict__ diag, double* x, double* r, double* z,
                                                 double* p, float* pvec, double* blk, int n, int dim, int nblk,
                                                 int pq, double rtol, DevScalars* sc, HostScalars* hs,
                                                 cudaGraphConditionalHandle cond, int use_cond, int cg_max)
{
    __shared__ double red[32];
    const int quarter = threadIdx.x >> 8, tq = threadIdx.x & 255;
    // (1) y = diag p' - S (k_p2_finish), y += sigma S_p (k_cg_ap), p.y partials
    for (int b0 = 0; b0 < nblk; b0 += 4) {
        const int b = b0 + quarter;
        const int i = b * kRB + tq;
        double py[3] = {0, 0, 0};
        if (b < nblk && i < n) {
            const int64_t g = stage_slot(i);
            const double d = diag[i];
            for (int q = 0; q < dim; ++q) {
                const size_t k = (size_t)i * dim + q;
                double yv = d * (double)pvec_in[g * pq + q] - y[k];
                yv = yv + sc->sigma * sc->S[q];
                y[k] = yv;
                py[q] = p[k] * yv;
            }
        }
        for (int q = 0; q < dim; ++q) {
            const double t = quarter_sum(py[q], red);
            if (tq == 0 && b < nblk) blk[(size_t)q * nblk + b] = t;
        }
    }
    __syncthreads();
    if (threadIdx.x < 32) cg_finalize_warp(blk, nblk, dim, 1, rtol, sc, hs, cond, 0, cg_max);
    __syncthreads();
    // (2) x += alpha p, r -= alpha y, z = r / diag, dot partials (k_cg_update)
    for (int b0 = 0; b0 < nblk; b0 += 4) {
        const int b = b0 + quarter;
        const int i = b * kRB + tq;
        double rz[3] = {0, 0, 0}, rr[3] = {0, 0, 0}, zs[3] = {0, 0, 0};
        if (b < nblk && i < n) {
            for (int q = 0; q < dim; ++q) {
                const size_t k = (size_t)i * dim + q;
                const double al = sc->alpha[q];
                const double xv = x[k] + al * p[k];
                const double rv = r[k] - al * y[k];
                const double zv = rv / diag[i];
                x[k] = xv;
                r[k] = rv;
                z[k] = zv;
                rz[q] = rv * zv;
                rr[q] = rv * rv;
                zs[q] = zv;
            }
        }
        for (int q = 0; q < dim; ++q) {
            double t = quarter_sum(rz[q], red);
            if (tq == 0 && b < nblk) blk[(size_t)(0 * 4 + q) * nblk + b] = t;
            t = quarter_sum(rr[q], red);
            if (tq == 0 && b < nblk) blk[(size_t)(1 * 4 + q) * nblk + b] = t;
            t = quarter_sum(zs[q], red);
            if (tq == 0 && b < nblk) blk[(size_t)(3 * 4 + q) * nblk + b] = t;
        }
    }
    __syncthreads();
    if (threadIdx.x < 32) cg_finalize_warp(blk, nblk, dim, 2, rtol, sc, hs, cond, use_cond, cg_max);
    __syncthreads();
    // (3) p = z + beta p (active columns), fp32 staging centred by S/n (k_cg_p)
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int64_t g = stage_slot(i);
        for (int q = 0; q < dim; ++q) {
            const size_t k = (size_t)i * dim + q;
            double pv = p[k];
            if (sc->active[q]) pv = z[k] + sc->beta[q] * pv;
            p[k] = pv;
            pvec[g * pq + q] = (float)(pv - sc->S[q] * sc->inv_n);
        }
    }
}

cudaError_t launch_cg_tail(double* y, const float* pvec_in, const double* diag, double* x, double* r, double* z,
                           double* p, float* pvec, double* blk, int n, int dim, int nblk, int pq, double rtol,
                           DevScalars* sc, HostScalars* hs, cudaStream_t s, unsigned long long cond, int use_cond,
                           int cg_max)
{
    k_cg_tail<<<1, 1024, 0, s>>>(y, pvec_in, diag, x, r, z, p, pvec, blk, n, dim, nblk, pq, rtol, sc, hs,
                                 (cudaGraphConditionalHandle)cond, use_cond, cg_max);
    return cudaGetLastError();
}

cudaError_t launch_cg_finalize(const double* blk, int nblk, int dim, int mode, double rtol, DevScalars* sc,
                               HostScalars* hs, cudaStream_t s, unsigned long long cond, int use_cond, int cg_max)
{
    k_cg_finalize<<<1, 32, 0, s>>>(blk, nblk, dim, mode, rtol, sc, hs, (cudaGraphConditionalHandle)cond, use_cond,
                                   cg_max);
    return cudaGetLastError();
}

// IF node of the step graph: the epilogue (lines 5-8) runs only when the solve
// converged, so a capped PCG leaves X^k, R^k, A^k as the eager step leaves them
__global__ void k_cond_done(const DevScalars* sc, cudaGraphConditionalHandle cond)
{
    cudaGraphSetConditional(cond, sc->done ? 1u : 0u);
}

cudaError_t launch_cond_done(const DevScalars* sc, cudaStream_t s, unsigned long long cond)
{
    k_cond_done<<<1, 1, 0, s>>>(sc, (cudaGraphConditionalHandle)cond);
    return cudaGetLastError();
}

// ============================================================ FFMA roofline
// Peak FP32 microbenchmark: 8 independent FFMA chains per thread.
__global__ void k_ffma(float* out, int iters)
{
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-7f + k;
    const float m = 0.9999999f, c = 1e-7f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], m, c);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 12345.f) out[threadIdx.x] = s;
}

cudaError_t launch_ffma_bench(float* out, int iters, int blocks, int threads, cudaStream_t s)
{
    k_ffma<<<blocks, threads, 0, s>>>(out, iters);
    return cudaGetLastError();
}

}  // namespace fdl
