// fdl_kernels.cu -- sm_100a kernels of the SOR stress-majorization hot path.
//
// Paper quantities (PAPER.md, arXiv 1711.01228), in device units of k
// (positions X' = X/k, ideal distance d' = hop h, weight w' = h^-2):
//   P1  per row i, for one or two position sets (X^{k+1} and the relaxed Xt):
//         R_i = sum_{j != i} (x_i - x_j) / (h_ij r_ij)      = (L^X X)_i   (Eq. 2-5 rhs)
//         s_i = sum_{j != i} (r_ij / h_ij - 1)^2              f = s.sum()/2  (Eq. 1)
//       one hop read feeds both sets (Algorithm 2 lines 4-6 evaluate f twice).
//   P2  y_i = sum_{j != i} w_ij (p_i - p_j), p_0 = 0           = (L^W_red p)_i
//   MS-BFS   hop(i,j) = graph distance (DESIGN R1), 1024 sources per batch.
//   CG / combine / select: fp64 vector kernels of PCG, Eq. 10 and the
//   guard of Algorithm 2 lines 6-8.
// FP32 CUDA cores only: the pair terms are non-linear (rsqrt) with no
// K-reduction, so there is no dense contraction for tcgen05.  Hop tiles and
// position tiles are staged in shared memory by cp.async.bulk (TMA, SASS
// UBLKCP) through a kStages-deep mbarrier ring.
//
// Determinism: every sum has a fixed order independent of grid size and of
// the number of GPUs: fp32 over one j-tile (<= 64 terms) -> fp64 per row per
// column chunk -> fp64 over chunks in chunk order -> fixed 256-row blocks ->
// blocks in global order.
#include <cfloat>
#include <cstdint>

#include "fdl_internal.h"

namespace fdl {

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity)
{
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    while (!mbar_try_wait(bar, parity)) {
    }
}

// 1-D bulk tensor copy global -> shared, completion counted on `bar`.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ float rsqrt_approx(float x)
{
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float rcp_approx(float x)
{
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Hop count of entry e of a 32-bit word as an exact float: one PRMT builds
// 0x4B0000hh (= 2^23 + h) and one FADD removes 2^23.
template <int HB>
__device__ __forceinline__ float hop_float(uint32_t word, int e)
{
    uint32_t bits;
    if (HB == 1)
        bits = __byte_perm(word, 0x4B000000u, 0x7650u + (uint32_t)e);
    else
        bits = __byte_perm(word, 0x4B000000u, e == 0 ? 0x7610u : 0x7632u);
    return __uint_as_float(bits) - 8388608.0f;
}

__device__ __forceinline__ uint32_t word_of(const uint4& v, int q)
{
    return q == 0 ? v.x : (q == 1 ? v.y : (q == 2 ? v.z : v.w));
}

template <int DIM, int NSETS>
__host__ __device__ constexpr int p1_stride()
{
    return DIM == 2 ? (NSETS == 1 ? 2 : 4) : (NSETS == 1 ? 4 : 8);
}

template <int DIM>
__host__ __device__ constexpr int p2_stride()
{
    return DIM == 2 ? 2 : 4;
}

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

// ================================================================= P1 / P2
// Work item = (row block rb of kBM local rows, column chunk c).  Each CTA runs
// items blockIdx.x, blockIdx.x + gridDim.x, ...; the tiles of its items form
// one stream fed by a kStages-deep TMA ring.  Thread (warp w, lane l) owns
// rows (w*kRPT + m)*32 + l of the item, m < kRPT: row-group-aligned, so its
// 16-byte hop cells are a lane-contiguous 512-byte run in shared memory.
struct TileIter {
    int item, t, nt;
};

template <int BN>
__device__ __forceinline__ int tiles_of_item(const PairArgs& a, int item)
{
    const int c = item % a.NC;
    const int cols = min(a.CK, a.n - c * a.CK);
    return (cols + BN - 1) / BN;
}

template <int BN>
__device__ __forceinline__ void iter_advance(const PairArgs& a, TileIter& it, int items)
{
    if (++it.t == it.nt) {
        it.t = 0;
        it.item += gridDim.x;
        it.nt = it.item < items ? tiles_of_item<BN>(a, it.item) : 0;
    }
}

template <int HB, int BN, int PSB /* bytes of pos per vertex */>
__device__ __forceinline__ void issue_tile(const PairArgs& a, const TileIter& it, uint8_t* stage_base,
                                           uint64_t* bar)
{
    constexpr int V = kVecBytes / HB;
    constexpr int NV = BN / V;
    constexpr int DT = kBM * BN * HB;
    constexpr int PT = BN * PSB;
    const int rb = it.item / a.NC, c = it.item % a.NC;
    const int64_t j0 = (int64_t)c * a.CK + (int64_t)it.t * BN;
    const int64_t cells_per_group = a.Np / V;
    fence_proxy_async();
    mbar_arrive_expect_tx(bar, DT + PT);
#pragma unroll
    for (int g = 0; g < kBM / kRowGroup; ++g) {
        const uint8_t* src =
            a.D + ((int64_t)(rb * (kBM / kRowGroup) + g) * cells_per_group + j0 / V) * kCellBytes;
        tma_load_1d(stage_base + g * NV * kCellBytes, src, NV * kCellBytes, bar);
    }
    tma_load_1d(stage_base + DT, reinterpret_cast<const uint8_t*>(a.pos) + j0 * PSB, PT, bar);
}

// ----------------------------------------------------------------- P1 pair
template <int DIM, bool SAFE>
__device__ __forceinline__ void p1_pair(const float* xi, const float* xj, float h2, float* acc)
{
    float d[DIM];
    float r2 = FLT_MIN;  // keeps r2 > 0 for coincident points: x_i == x_j -> zero R term
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        d[c] = xi[c] - xj[c];
        r2 = fmaf(d[c], d[c], r2);
    }
    float q = rsqrt_approx(r2 * h2);  // 1 / (h r)  = w' d' / r
    float u = fmaf(r2, q, -1.0f);     // r/h - 1    (stress term is u^2, w' d'^2 = 1)
    if (SAFE) {                        // h == 0: diagonal or padding column -> no pair
        const bool valid = h2 > 0.0f;
        q = valid ? q : 0.0f;
        u = valid ? u : 0.0f;
    }
#pragma unroll
    for (int c = 0; c < DIM; ++c) acc[c] = fmaf(q, d[c], acc[c]);
    acc[DIM] = fmaf(u, u, acc[DIM]);
}

template <int DIM, int NSETS, int HB, bool SAFE>
__device__ __forceinline__ void p1_tile(const uint8_t* sD, const float* sP, int warp, int lane,
                                        const float (&xi)[kRPT][NSETS][DIM],
                                        float (&acc)[kRPT][NSETS][DIM + 1])
{
    constexpr int BN = bn_for(HB);
    constexpr int V = kVecBytes / HB;
    constexpr int NV = BN / V;
    constexpr int PS = p1_stride<DIM, NSETS>();
    constexpr int EPW = 4 / HB;  // entries per 32-bit word
#pragma unroll 1
    for (int v = 0; v < NV; ++v) {
        uint4 dv[kRPT];
#pragma unroll
        for (int m = 0; m < kRPT; ++m)
            dv[m] = *reinterpret_cast<const uint4*>(sD + ((warp * kRPT + m) * NV + v) * kCellBytes + lane * 16);
#pragma unroll
        for (int e = 0; e < V; ++e) {
            const int j = v * V + e;
            float xj[PS];
            if (PS == 2) {
                const float2 t = *reinterpret_cast<const float2*>(sP + j * PS);
                xj[0] = t.x; xj[1] = t.y;
            } else {
#pragma unroll
                for (int q = 0; q < PS / 4; ++q) {
                    const float4 t = *reinterpret_cast<const float4*>(sP + j * PS + 4 * q);
                    xj[4 * q + 0] = t.x; xj[4 * q + 1] = t.y; xj[4 * q + 2] = t.z; xj[4 * q + 3] = t.w;
                }
            }
#pragma unroll
            for (int m = 0; m < kRPT; ++m) {
                const float hf = hop_float<HB>(word_of(dv[m], e / EPW), e % EPW);
                const float h2 = hf * hf;
#pragma unroll
                for (int s = 0; s < NSETS; ++s) p1_pair<DIM, SAFE>(xi[m][s], xj + s * DIM, h2, acc[m][s]);
            }
        }
    }
}

template <int DIM, int NSETS, int HB>
__global__ void __launch_bounds__(kThreads) k_p1(const PairArgs a)
{
    constexpr int BN = bn_for(HB);
    constexpr int PS = p1_stride<DIM, NSETS>();
    constexpr int DT = kBM * BN * HB;
    constexpr int STAGE = DT + BN * PS * 4;
    constexpr int NCOMP = NSETS * (DIM + 1);
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t full[kStages];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int items = a.nrb * a.NC;
    if ((int)blockIdx.x >= items) return;
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    TileIter cit{(int)blockIdx.x, 0, tiles_of_item<BN>(a, blockIdx.x)};
    TileIter pit = cit;
    if (tid == 0) {
        for (int s = 0; s < kStages - 1 && pit.item < items; ++s) {
            issue_tile<HB, BN, PS * 4>(a, pit, smem + s * STAGE, &full[s]);
            iter_advance<BN>(a, pit, items);
        }
    }

    float xi[kRPT][NSETS][DIM];
    double acc64[kRPT][NSETS][DIM + 1];
    int stage = 0;
    uint32_t phase = 0;
    while (cit.item < items) {
        if (tid == 0 && pit.item < items) {
            const int ps = (stage + kStages - 1) % kStages;
            issue_tile<HB, BN, PS * 4>(a, pit, smem + ps * STAGE, &full[ps]);
            iter_advance<BN>(a, pit, items);
        }
        const int rb = cit.item / a.NC, c = cit.item % a.NC;
        if (cit.t == 0) {
#pragma unroll
            for (int m = 0; m < kRPT; ++m) {
                const int64_t gr = (int64_t)a.row0 + rb * kBM + (warp * kRPT + m) * 32 + lane;
#pragma unroll
                for (int s = 0; s < NSETS; ++s)
#pragma unroll
                    for (int q = 0; q < DIM; ++q) xi[m][s][q] = a.pos[gr * PS + s * DIM + q];
#pragma unroll
                for (int s = 0; s < NSETS; ++s)
#pragma unroll
                    for (int q = 0; q <= DIM; ++q) acc64[m][s][q] = 0.0;
            }
        }
        const int64_t j0 = (int64_t)c * a.CK + (int64_t)cit.t * BN;
        const int64_t gi0 = (int64_t)a.row0 + (int64_t)rb * kBM;
        const bool safe = (j0 + BN > a.n) || (j0 < gi0 + kBM && j0 + BN > gi0);
        float acc[kRPT][NSETS][DIM + 1];
#pragma unroll
        for (int m = 0; m < kRPT; ++m)
#pragma unroll
            for (int s = 0; s < NSETS; ++s)
#pragma unroll
                for (int q = 0; q <= DIM; ++q) acc[m][s][q] = 0.0f;

        mbar_wait(&full[stage], phase);
        const uint8_t* sD = smem + stage * STAGE;
        const float* sP = reinterpret_cast<const float*>(sD + DT);
        if (safe)
            p1_tile<DIM, NSETS, HB, true>(sD, sP, warp, lane, xi, acc);
        else
            p1_tile<DIM, NSETS, HB, false>(sD, sP, warp, lane, xi, acc);
#pragma unroll
        for (int m = 0; m < kRPT; ++m)
#pragma unroll
            for (int s = 0; s < NSETS; ++s)
#pragma unroll
                for (int q = 0; q <= DIM; ++q) acc64[m][s][q] += (double)acc[m][s][q];

        if (cit.t == cit.nt - 1) {
#pragma unroll
            for (int m = 0; m < kRPT; ++m) {
                const int lr = rb * kBM + (warp * kRPT + m) * 32 + lane;
#pragma unroll
                for (int s = 0; s < NSETS; ++s)
#pragma unroll
                    for (int q = 0; q <= DIM; ++q)
                        a.part[((size_t)c * NCOMP + s * (DIM + 1) + q) * a.Mrows + lr] = acc64[m][s][q];
            }
        }
        __syncthreads();  // stage fully consumed -> producer may refill it
        iter_advance<BN>(a, cit, items);
        if (++stage == kStages) {
            stage = 0;
            phase ^= 1u;
        }
    }
}

// ----------------------------------------------------------------- P2 pair
template <int DIM, int HB, bool SAFE>
__device__ __forceinline__ void p2_tile(const uint8_t* sD, const float* sP, const float* lut, int warp,
                                        int lane, const float (&pi)[kRPT][DIM], float (&acc)[kRPT][DIM])
{
    constexpr int BN = bn_for(HB);
    constexpr int V = kVecBytes / HB;
    constexpr int NV = BN / V;
    constexpr int PQ = p2_stride<DIM>();
    constexpr int EPW = 4 / HB;
#pragma unroll 1
    for (int v = 0; v < NV; ++v) {
        uint4 dv[kRPT];
#pragma unroll
        for (int m = 0; m < kRPT; ++m)
            dv[m] = *reinterpret_cast<const uint4*>(sD + ((warp * kRPT + m) * NV + v) * kCellBytes + lane * 16);
#pragma unroll
        for (int e = 0; e < V; ++e) {
            const int j = v * V + e;
            float pj[PQ];
            if (PQ == 2) {
                const float2 t = *reinterpret_cast<const float2*>(sP + j * PQ);
                pj[0] = t.x; pj[1] = t.y;
            } else {
                const float4 t = *reinterpret_cast<const float4*>(sP + j * PQ);
                pj[0] = t.x; pj[1] = t.y; pj[2] = t.z; pj[3] = t.w;
            }
#pragma unroll
            for (int m = 0; m < kRPT; ++m) {
                const uint32_t word = word_of(dv[m], e / EPW);
                float w;
                if (HB == 1) {
                    w = lut[__byte_perm(word, 0u, 0x4440u + (uint32_t)(e % EPW))];  // lut[0] = 0
                } else {
                    const float hf = hop_float<HB>(word, e % EPW);
                    w = rcp_approx(hf * hf);
                    if (SAFE) w = hf > 0.0f ? w : 0.0f;
                }
#pragma unroll
                for (int q = 0; q < DIM; ++q) acc[m][q] = fmaf(w, pi[m][q] - pj[q], acc[m][q]);
            }
        }
    }
}

template <int DIM, int HB>
__global__ void __launch_bounds__(kThreads) k_p2(const PairArgs a)
{
    constexpr int BN = bn_for(HB);
    constexpr int PQ = p2_stride<DIM>();
    constexpr int DT = kBM * BN * HB;
    constexpr int STAGE = DT + BN * PQ * 4;
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t full[kStages];
    __shared__ float lut[256];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int items = a.nrb * a.NC;
    if ((int)blockIdx.x >= items) return;
    if (HB == 1)
        for (int t = tid; t < 256; t += kThreads) lut[t] = a.lut[t];
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();

    TileIter cit{(int)blockIdx.x, 0, tiles_of_item<BN>(a, blockIdx.x)};
    TileIter pit = cit;
    if (tid == 0) {
        for (int s = 0; s < kStages - 1 && pit.item < items; ++s) {
            issue_tile<HB, BN, PQ * 4>(a, pit, smem + s * STAGE, &full[s]);
            iter_advance<BN>(a, pit, items);
        }
    }
    float pi[kRPT][DIM];
    double acc64[kRPT][DIM];
    int stage = 0;
    uint32_t phase = 0;
    while (cit.item < items) {
        if (tid == 0 && pit.item < items) {
            const int ps = (stage + kStages - 1) % kStages;
            issue_tile<HB, BN, PQ * 4>(a, pit, smem + ps * STAGE, &full[ps]);
            iter_advance<BN>(a, pit, items);
        }
        const int rb = cit.item / a.NC, c = cit.item % a.NC;
        if (cit.t == 0) {
#pragma unroll
            for (int m = 0; m < kRPT; ++m) {
                const int64_t gr = (int64_t)a.row0 + rb * kBM + (warp * kRPT + m) * 32 + lane;
#pragma unroll
                for (int q = 0; q < DIM; ++q) {
                    pi[m][q] = a.pos[gr * PQ + q];
                    acc64[m][q] = 0.0;
                }
            }
        }
        const int64_t j0 = (int64_t)c * a.CK + (int64_t)cit.t * BN;
        const int64_t gi0 = (int64_t)a.row0 + (int64_t)rb * kBM;
        const bool safe = (j0 + BN > a.n) || (j0 < gi0 + kBM && j0 + BN > gi0);
        float acc[kRPT][DIM];
#pragma unroll
        for (int m = 0; m < kRPT; ++m)
#pragma unroll
            for (int q = 0; q < DIM; ++q) acc[m][q] = 0.0f;
        mbar_wait(&full[stage], phase);
        const uint8_t* sD = smem + stage * STAGE;
        const float* sP = reinterpret_cast<const float*>(sD + DT);
        if (HB == 2 && safe)
            p2_tile<DIM, HB, true>(sD, sP, lut, warp, lane, pi, acc);
        else
            p2_tile<DIM, HB, false>(sD, sP, lut, warp, lane, pi, acc);
#pragma unroll
        for (int m = 0; m < kRPT; ++m)
#pragma unroll
            for (int q = 0; q < DIM; ++q) acc64[m][q] += (double)acc[m][q];
        if (cit.t == cit.nt - 1) {
#pragma unroll
            for (int m = 0; m < kRPT; ++m) {
                const int lr = rb * kBM + (warp * kRPT + m) * 32 + lane;
#pragma unroll
                for (int q = 0; q < DIM; ++q) a.part[((size_t)c * DIM + q) * a.Mrows + lr] = acc64[m][q];
            }
        }
        __syncthreads();
        iter_advance<BN>(a, cit, items);
        if (++stage == kStages) {
            stage = 0;
            phase ^= 1u;
        }
    }
}

template <int DIM, int NSETS, int HB>
static size_t p1_smem()
{
    return (size_t)kStages * (kBM * bn_for(HB) * HB + bn_for(HB) * p1_stride<DIM, NSETS>() * 4);
}
template <int DIM, int HB>
static size_t p2_smem()
{
    return (size_t)kStages * (kBM * bn_for(HB) * HB + bn_for(HB) * p2_stride<DIM>() * 4);
}

template <int DIM, int NSETS, int HB>
static cudaError_t launch_p1_t(const PairArgs& a, int grid, cudaStream_t s)
{
    const size_t sm = p1_smem<DIM, NSETS, HB>();
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_p1<DIM, NSETS, HB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sm);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    k_p1<DIM, NSETS, HB><<<grid, kThreads, sm, s>>>(a);
    return cudaGetLastError();
}

template <int DIM, int HB>
static cudaError_t launch_p2_t(const PairArgs& a, int grid, cudaStream_t s)
{
    const size_t sm = p2_smem<DIM, HB>();
    static bool attr = false;
    if (!attr) {
        cudaError_t e =
            cudaFuncSetAttribute(k_p2<DIM, HB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    k_p2<DIM, HB><<<grid, kThreads, sm, s>>>(a);
    return cudaGetLastError();
}

#define FDL_DISPATCH_P1(D_, S_, H_) \
    if (dim == D_ && nsets == S_ && hb == H_) return launch_p1_t<D_, S_, H_>(a, grid, s);
cudaError_t launch_p1(const PairArgs& a, int dim, int nsets, int hb, int grid, cudaStream_t s)
{
    FDL_DISPATCH_P1(2, 1, 1) FDL_DISPATCH_P1(2, 2, 1) FDL_DISPATCH_P1(3, 1, 1) FDL_DISPATCH_P1(3, 2, 1)
    FDL_DISPATCH_P1(2, 1, 2) FDL_DISPATCH_P1(2, 2, 2) FDL_DISPATCH_P1(3, 1, 2) FDL_DISPATCH_P1(3, 2, 2)
    return cudaErrorInvalidValue;
}

cudaError_t launch_p2(const PairArgs& a, int dim, int hb, int grid, cudaStream_t s)
{
    if (dim == 2 && hb == 1) return launch_p2_t<2, 1>(a, grid, s);
    if (dim == 3 && hb == 1) return launch_p2_t<3, 1>(a, grid, s);
    if (dim == 2 && hb == 2) return launch_p2_t<2, 2>(a, grid, s);
    if (dim == 3 && hb == 2) return launch_p2_t<3, 2>(a, grid, s);
    return cudaErrorInvalidValue;
}

template <typename K>
static int occ(K kern, size_t smem, int device)
{
    (void)device;
    int n = 0;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kThreads, smem) != cudaSuccess) n = 1;
    return n > 0 ? n : 1;
}

int p1_max_ctas(int dim, int nsets, int hb, int device)
{
#define FDL_OCC1(D_, S_, H_) \
    if (dim == D_ && nsets == S_ && hb == H_) return occ(k_p1<D_, S_, H_>, p1_smem<D_, S_, H_>(), device);
    FDL_OCC1(2, 1, 1) FDL_OCC1(2, 2, 1) FDL_OCC1(3, 1, 1) FDL_OCC1(3, 2, 1)
    FDL_OCC1(2, 1, 2) FDL_OCC1(2, 2, 2) FDL_OCC1(3, 1, 2) FDL_OCC1(3, 2, 2)
    return 1;
}

int p2_max_ctas(int dim, int hb, int device)
{
    if (dim == 2 && hb == 1) return occ(k_p2<2, 1>, p2_smem<2, 1>(), device);
    if (dim == 3 && hb == 1) return occ(k_p2<3, 1>, p2_smem<3, 1>(), device);
    if (dim == 2 && hb == 2) return occ(k_p2<2, 2>, p2_smem<2, 2>(), device);
    if (dim == 3 && hb == 2) return occ(k_p2<3, 2>, p2_smem<3, 2>(), device);
    return 1;
}

// ============================================================ reductions
// Rows are processed in fixed global blocks of kRB = 256; local block b of a
// rank starting at row0 (a multiple of kRB) is global block row0/kRB + b.

__global__ void __launch_bounds__(kRB) k_p1_reduce(const double* __restrict__ part, int NC, int Mrows, int nloc,
                                                   int row0, int dim, int nsets, double* R0, double* R1,
                                                   double* blk_f, int nblk)
{
    __shared__ double red[8];
    const int lr = blockIdx.x * kRB + threadIdx.x;
    const int ncomp = nsets * (dim + 1);
    double srow[2] = {0.0, 0.0};
    if (lr < nloc) {
        for (int s = 0; s < nsets; ++s) {
            double* R = s == 0 ? R0 : R1;
            for (int q = 0; q <= dim; ++q) {
                double v = 0.0;
                for (int c = 0; c < NC; ++c) v += part[((size_t)c * ncomp + s * (dim + 1) + q) * Mrows + lr];
                if (q < dim)
                    R[(size_t)lr * dim + q] = v;
                else
                    srow[s] = v;
            }
        }
    }
    const int gb = row0 / kRB + blockIdx.x;
    for (int s = 0; s < nsets; ++s) {
        const double t = block_sum_256(srow[s], red);
        if (threadIdx.x == 0) blk_f[(size_t)s * nblk + gb] = t;
    }
}

cudaError_t launch_p1_reduce(const double* part, int NC, int Mrows, int nloc, int row0, int dim, int nsets,
                             double* R0, double* R1, double* blk_f, int nblk_global, cudaStream_t s)
{
    const int nb = (nloc + kRB - 1) / kRB;
    k_p1_reduce<<<nb, kRB, 0, s>>>(part, NC, Mrows, nloc, row0, dim, nsets, R0, R1, blk_f, nblk_global);
    return cudaGetLastError();
}

// f = 1/2 sum_i s_i (Eq. 1 counts each unordered pair once).  One warp,
// lane-strided partial sums then a fixed butterfly: deterministic.
__global__ void k_stress_finalize(const double* __restrict__ blk_f, int nblk, int nsets, DevScalars* sc,
                                  int set_cur)
{
    const int lane = threadIdx.x;
    for (int s = 0; s < nsets; ++s) {
        double v = 0.0;
        for (int b = lane; b < nblk; b += 32) v += blk_f[(size_t)s * nblk + b];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) {
            sc->f_set[s] = 0.5 * v;
            if (set_cur) {
                sc->f_cur = 0.5 * v;
                sc->nonfinite = !isfinite(0.5 * v);
            }
        }
    }
}

cudaError_t launch_stress_finalize(const double* blk_f, int nblk, int nsets, DevScalars* sc, int set_cur,
                                   cudaStream_t s)
{
    k_stress_finalize<<<1, 32, 0, s>>>(blk_f, nblk, nsets, sc, set_cur);
    return cudaGetLastError();
}

// y = sum over chunks (generic, for A = L^W X)
__global__ void __launch_bounds__(kRB) k_reduce_rows(const double* __restrict__ part, int NC, int Mrows, int nloc,
                                                     int dim, double* out)
{
    const int lr = blockIdx.x * kRB + threadIdx.x;
    if (lr >= nloc) return;
    for (int q = 0; q < dim; ++q) {
        double v = 0.0;
        for (int c = 0; c < NC; ++c) v += part[((size_t)c * dim + q) * Mrows + lr];
        out[(size_t)lr * dim + q] = v;
    }
}

cudaError_t launch_reduce_rows(const double* part, int NC, int Mrows, int nloc, int dim, double* out,
                               cudaStream_t s)
{
    k_reduce_rows<<<(nloc + kRB - 1) / kRB, kRB, 0, s>>>(part, NC, Mrows, nloc, dim, out);
    return cudaGetLastError();
}

// ================================================================ MS-BFS
// Bit-parallel multi-source BFS: batch of up to 1024 sources s0..s0+1023;
// vertex v keeps a 1024-bit frontier / visited mask (32 words, word = lane).
// Level L: next(v) = OR_{u in N(v)} frontier(u) & ~visited(v); newly set bit b
// of word l means hop(v, s0 + 32 l + b) = L.  One warp per vertex: lanes read
// 32 neighbour ids at a time (coalesced), then OR each neighbour's 128-byte
// mask (one line per neighbour, coalesced).
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

template <int HB>
__global__ void __launch_bounds__(256) k_bfs_level(const int64_t* __restrict__ row_ptr,
                                                   const int32_t* __restrict__ col,
                                                   const uint32_t* __restrict__ fin, uint32_t* __restrict__ fout,
                                                   uint32_t* __restrict__ visited, uint8_t* __restrict__ D, int n,
                                                   int s0, int nsrc, int level, int row0, int row1, int64_t Np,
                                                   unsigned int* anynew)
{
    const int v = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (v >= n) return;
    const int nl = min(max(nsrc - 32 * lane, 0), 32);
    const uint32_t full = nl == 32 ? 0xffffffffu : ((1u << nl) - 1u);
    const uint32_t vis = visited[(int64_t)v * kBFSWords + lane];
    if (__all_sync(0xffffffffu, (vis & full) == full)) {
        fout[(int64_t)v * kBFSWords + lane] = 0u;
        return;
    }
    uint32_t acc = 0;
    const int64_t beg = row_ptr[v], end = row_ptr[v + 1];
    for (int64_t e0 = beg; e0 < end; e0 += 32) {
        const int myu = (e0 + lane < end) ? col[e0 + lane] : 0;
        const int cnt = (int)min((int64_t)32, end - e0);
#pragma unroll 4
        for (int k = 0; k < cnt; ++k) {
            const int u = __shfl_sync(0xffffffffu, myu, k);
            acc |= fin[(int64_t)u * kBFSWords + lane];
        }
    }
    uint32_t nw = acc & ~vis & full;
    fout[(int64_t)v * kBFSWords + lane] = nw;
    if (nw) visited[(int64_t)v * kBFSWords + lane] = vis | nw;
    if (__any_sync(0xffffffffu, nw != 0u) && lane == 0) *anynew = 1u;
    if (v >= row0 && v < row1) {
        const int64_t lv = v - row0;
        const int64_t cbase = (int64_t)s0 + 32 * lane;
        while (nw) {
            const int b = __ffs(nw) - 1;
            nw &= nw - 1u;
            const size_t off = d_offset(lv, cbase + b, Np, HB);
            if (HB == 1)
                D[off] = (uint8_t)level;
            else
                *reinterpret_cast<uint16_t*>(D + off) = (uint16_t)level;
        }
    }
}

cudaError_t launch_bfs_level(const int64_t* row_ptr, const int32_t* col, const uint32_t* fin, uint32_t* fout,
                             uint32_t* visited, uint8_t* D, int n, int s0, int nsrc, int level, int row0,
                             int row1, int64_t Np, int hb, unsigned int* anynew, cudaStream_t s)
{
    const int64_t threads = (int64_t)n * 32;
    const unsigned grid = (unsigned)((threads + 255) / 256);
    if (hb == 1)
        k_bfs_level<1><<<grid, 256, 0, s>>>(row_ptr, col, fin, fout, visited, D, n, s0, nsrc, level, row0, row1, Np,
                                            anynew);
    else
        k_bfs_level<2><<<grid, 256, 0, s>>>(row_ptr, col, fin, fout, visited, D, n, s0, nsrc, level, row0, row1, Np,
                                            anynew);
    return cudaGetLastError();
}

// Jacobi diagonal sum_{j != i} w'_ij, w' = fp32(1/h^2) (h = 0 -> 0), one
// thread per local row summing its row sequentially in fp64 (row-group
// coalesced 16-byte cell reads).
template <int HB>
__global__ void __launch_bounds__(256) k_diag(const uint8_t* __restrict__ D, int64_t Np, int nloc, double* diag,
                                              double* blk, int row0)
{
    __shared__ double red[8];
    const int64_t lr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    constexpr int V = kVecBytes / HB;
    const int64_t cells = Np / V;
    const uint8_t* base = D + (lr / kRowGroup) * cells * kCellBytes + (lr % kRowGroup) * kVecBytes;
    double s = 0.0;
    for (int64_t c = 0; c < cells; ++c) {
        const uint4 cell = *reinterpret_cast<const uint4*>(base + c * kCellBytes);
#pragma unroll
        for (int e = 0; e < V; ++e) {
            const float hf = hop_float<HB>(word_of(cell, e / (4 / HB)), e % (4 / HB));
            const float w = hf > 0.0f ? __frcp_rn(hf * hf) : 0.0f;
            s += (double)w;
        }
    }
    if (lr < nloc) diag[lr] = s;
    const double t = block_sum_256(lr < nloc ? s : 0.0, red);
    if (threadIdx.x == 0) blk[row0 / kRB + blockIdx.x] = t;
}

cudaError_t launch_diag(const uint8_t* D, int64_t Np, int hb, int n, int nloc, int row0, double* diag, double* blk,
                        cudaStream_t s)
{
    (void)n;
    const unsigned grid = (unsigned)((nloc + 255) / 256);
    if (hb == 1)
        k_diag<1><<<grid, 256, 0, s>>>(D, Np, nloc, diag, blk, row0);
    else
        k_diag<2><<<grid, 256, 0, s>>>(D, Np, nloc, diag, blk, row0);
    return cudaGetLastError();
}

// ====================================================== vector kernels (fp64)
__global__ void k_stage_pos1(const double* __restrict__ X, float* posf, int nloc, int row0, int dim, int ps)
{
    const int lr = blockIdx.x * blockDim.x + threadIdx.x;
    if (lr >= nloc) return;
    const int64_t g = (int64_t)row0 + lr;
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
                                                 double omega, double cap, int nsets, int ps)
{
    __shared__ double red[8];
    const int lr = blockIdx.x * kRB + threadIdx.x;
    double disp2 = 0.0;
    if (lr < nloc) {
        const int64_t g = (int64_t)row0 + lr;
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
            posf[g * ps + q] = (float)xn[q];
            if (nsets == 2) posf[g * ps + dim + q] = (float)xt;
        }
        for (int q = nsets * dim; q < ps; ++q) posf[g * ps + q] = 0.0f;
    }
    const double m = block_max_256(disp2, red);
    if (threadIdx.x == 0) blk_max[blockIdx.x] = m;
}

cudaError_t launch_combine(const double* Xk, double* Xn, double* Xt, float* posf, double* blk_max,
                           const double* xpin, int nloc, int row0, int dim, double omega, double cap, int nsets,
                           int ps, cudaStream_t s)
{
    k_combine<<<(nloc + kRB - 1) / kRB, kRB, 0, s>>>(Xk, Xn, Xt, posf, blk_max, xpin, nloc, row0, dim, omega, cap,
                                                     nsets, ps);
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

// Guard of Algorithm 2 lines 6-8: accept Xt iff f(Xt) <= f(X^{k+1}) (ties
// accept, raw comparison).  Copies the accepted placement and its R.
__global__ void __launch_bounds__(kRB) k_select(double* Xk, double* Rk, const double* __restrict__ Xn,
                                                const double* __restrict__ Xt, const double* __restrict__ R1,
                                                const double* __restrict__ R2, const double* __restrict__ blk_max,
                                                int nblk_loc, int nloc, int dim, int nsets, DevScalars* sc)
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
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        double m = 0.0;
        for (int b = 0; b < nblk_loc; ++b) m = fmax(m, blk_max[b]);
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
                          const double* R2, const double* blk_f, const double* blk_max, int nblk, int nloc, int dim,
                          int nsets, DevScalars* sc, cudaStream_t s)
{
    (void)blk_f;
    (void)nblk;
    const int nb = (nloc + kRB - 1) / kRB;
    k_select<<<nb, kRB, 0, s>>>(Xk, Rk, Xn, Xt, R1, R2, blk_max, nb, nloc, dim, nsets, sc);
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
__global__ void k_cg_begin(const double* __restrict__ Xk, double* x, float* pvec, int nloc, int row0, int dim,
                           int pq)
{
    const int lr = blockIdx.x * blockDim.x + threadIdx.x;
    if (lr >= nloc) return;
    const int64_t g = (int64_t)row0 + lr;
    for (int q = 0; q < pq; ++q) {
        double v = 0.0;
        if (q < dim) {
            v = Xk[(size_t)lr * dim + q];
            x[(size_t)lr * dim + q] = v;
        }
        pvec[g * pq + q] = (float)v;
    }
}

cudaError_t launch_cg_begin(const double* Xk, double* x, float* pvec, int nloc, int row0, int dim, int pq,
                            cudaStream_t s)
{
    k_cg_begin<<<(nloc + kRB - 1) / kRB, kRB, 0, s>>>(Xk, x, pvec, nloc, row0, dim, pq);
    return cudaGetLastError();
}

__device__ __forceinline__ double chunk_sum(const double* __restrict__ part, int NC, int Mrows, int dim, int q,
                                            int lr)
{
    double v = 0.0;
    for (int c = 0; c < NC; ++c) v += part[((size_t)c * dim + q) * Mrows + lr];
    return v;
}

// r = b - L x0, z = r / diag, p = z; block partials of r.z, r.r, b.b
__global__ void __launch_bounds__(kRB) k_cg_init(const double* __restrict__ part, int NC, int Mrows,
                                                 const double* __restrict__ b, const double* __restrict__ x,
                                                 const double* __restrict__ diag, double* r, double* z, double* p,
                                                 float* pvec, double* blk, int nloc, int row0, int dim, int pq,
                                                 int nblk)
{
    __shared__ double red[8];
    const int lr = blockIdx.x * kRB + threadIdx.x;
    const int64_t g = (int64_t)row0 + lr;
    double rz[3] = {0, 0, 0}, rr[3] = {0, 0, 0}, bb[3] = {0, 0, 0}, zs[3] = {0, 0, 0};
    if (lr < nloc) {
        for (int q = 0; q < dim; ++q) {
            const size_t i = (size_t)lr * dim + q;
            const double bv = b[i];
            const double rv = bv - chunk_sum(part, NC, Mrows, dim, q, lr);
            const double zv = rv / diag[lr];
            r[i] = rv;
            z[i] = zv;
            p[i] = zv;
            pvec[g * pq + q] = (float)zv;
            rz[q] = rv * zv;
            rr[q] = rv * rv;
            bb[q] = bv * bv;
            zs[q] = zv;
        }
        for (int q = dim; q < pq; ++q) pvec[g * pq + q] = 0.0f;
    }
    const int gb = row0 / kRB + blockIdx.x;
    for (int q = 0; q < dim; ++q) {
        double t = block_sum_256(rz[q], red);
        if (threadIdx.x == 0) blk[(size_t)(0 * 4 + q) * nblk + gb] = t;
        t = block_sum_256(rr[q], red);
        if (threadIdx.x == 0) blk[(size_t)(1 * 4 + q) * nblk + gb] = t;
        t = block_sum_256(bb[q], red);
        if (threadIdx.x == 0) blk[(size_t)(2 * 4 + q) * nblk + gb] = t;
        t = block_sum_256(zs[q], red);
        if (threadIdx.x == 0) blk[(size_t)(3 * 4 + q) * nblk + gb] = t;
    }
}

cudaError_t launch_cg_init(const double* part, int NC, int Mrows, const double* b, const double* x,
                           const double* diag, double* r, double* z, double* p, float* pvec, double* blk, int nblk,
                           int nloc, int row0, int dim, int pq, cudaStream_t s)
{
    const int nb = (nloc + kRB - 1) / kRB;
    k_cg_init<<<nb, kRB, 0, s>>>(part, NC, Mrows, b, x, diag, r, z, p, pvec, blk, nloc, row0, dim, pq, nblk);
    return cudaGetLastError();
}

// y = L p (sum of chunk partials); block partials of p.y
__global__ void __launch_bounds__(kRB) k_cg_ap(const double* __restrict__ part, int NC, int Mrows,
                                               const double* __restrict__ p, double* y, double* blk, int nloc,
                                               int row0, int dim, int nblk, const DevScalars* __restrict__ sc)
{
    __shared__ double red[8];
    const int lr = blockIdx.x * kRB + threadIdx.x;
    double py[3] = {0, 0, 0};
    if (lr < nloc) {
        for (int q = 0; q < dim; ++q) {
            const size_t i = (size_t)lr * dim + q;
            const double yv = chunk_sum(part, NC, Mrows, dim, q, lr) + sc->sigma * sc->S[q];
            y[i] = yv;
            py[q] = p[i] * yv;
        }
    }
    const int gb = row0 / kRB + blockIdx.x;
    for (int q = 0; q < dim; ++q) {
        const double t = block_sum_256(py[q], red);
        if (threadIdx.x == 0) blk[(size_t)q * nblk + gb] = t;
    }
}

cudaError_t launch_cg_ap(const double* part, int NC, int Mrows, const double* p, double* y, double* blk, int nblk,
                         int nloc, int row0, int dim, const DevScalars* sc, cudaStream_t s)
{
    const int nb = (nloc + kRB - 1) / kRB;
    k_cg_ap<<<nb, kRB, 0, s>>>(part, NC, Mrows, p, y, blk, nloc, row0, dim, nblk, sc);
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
    const int64_t g = (int64_t)row0 + lr;
    for (int q = 0; q < dim; ++q) {
        const size_t i = (size_t)lr * dim + q;
        double pv = p[i];
        if (sc->active[q]) pv = z[i] + sc->beta[q] * pv;
        p[i] = pv;
        pvec[g * pq + q] = (float)pv;
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
__global__ void k_cg_finalize(const double* __restrict__ blk, int nblk, int dim, int mode, double rtol,
                              DevScalars* sc, HostScalars* hs)
{
    const int lane = threadIdx.x;
    double sums[4][3];
    for (int qq = 0; qq < 4; ++qq)
        for (int c = 0; c < dim; ++c) {
            sums[qq][c] = 0.0;
            if (mode == 1 && qq > 0) continue;
            if (mode == 2 && qq == 2) continue;
            const double* src = blk + (size_t)(qq * 4 + c) * nblk;
            double v = 0.0;
            for (int b = lane; b < nblk; b += 32) v += src[b];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            sums[qq][c] = v;
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
            const int act = sums[1][c] > rt2 * sums[2][c];
            sc->active[c] = act;
            any |= act;
            rel = fmax(rel, sums[2][c] > 0 ? sqrt(sums[1][c] / sums[2][c]) : 0.0);
        }
        sc->done = !any;
        sc->cg_iters = 0;
        sc->relres = rel;
        hs->done = !any;
    } else if (mode == 1) {
        for (int c = 0; c < dim; ++c) {
            sc->pap[c] = sums[0][c];
            sc->alpha[c] = (sc->active[c] && sums[0][c] > 0.0) ? sc->rz[c] / sums[0][c] : 0.0;
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
    }
}

// sigma = (sum_i diag_i) / n^2 from per-block partial sums of diag
__global__ void k_set_sigma(const double* __restrict__ blk, int nblk, double n, DevScalars* sc)
{
    const int lane = threadIdx.x;
    double v = 0.0;
    for (int b = lane; b < nblk; b += 32) v += blk[b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sc->sigma = v / (n * n);
}

cudaError_t launch_set_sigma(const double* blk, int nblk, int n, DevScalars* sc, cudaStream_t s)
{
    k_set_sigma<<<1, 32, 0, s>>>(blk, nblk, (double)n, sc);
    return cudaGetLastError();
}

cudaError_t launch_cg_finalize(const double* blk, int nblk, int dim, int mode, double rtol, DevScalars* sc,
                               HostScalars* hs, cudaStream_t s)
{
    k_cg_finalize<<<1, 32, 0, s>>>(blk, nblk, dim, mode, rtol, sc, hs);
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
