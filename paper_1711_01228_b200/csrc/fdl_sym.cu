// fdl_sym.cu -- symmetric (upper-triangle) all-pairs kernels for sm_100a.
//
// The pair terms of the method are symmetric in (i, j): d_ij = d_ji, w_ij = w_ji
// (P:48), the stress term of Eq. 1 is counted once per unordered pair
// (sum over i < j), and the L^Y / L^W products are antisymmetric
// (x_i - x_j) sums.  So each unordered pair is evaluated ONCE and feeds both
// rows: R_i += q (x_i - x_j) and R_j -= q (x_i - x_j) (Newton's third law),
// s += u^2.  Only the upper triangle of the hop matrix is stored: half the
// HBM bytes and half the pair arithmetic of a row-by-row evaluation.
//
// Geometry: tiles of kT x kT (128 x 128) vertices, tile (I, J) with I <= J,
// numbered row-major over the triangle.  A CTA of 256 threads = 16 x 16 grid;
// thread (ty, tx) owns the 8 x 8 sub-block rows 8 ty.., cols 8 tx.. of the
// tile; its 64 (u8) / 128 (u16) hop bytes are stored as 16-byte chunks
// interleaved across threads ((chunk * 256 + thread) * 16), so both the TMA
// bulk copy (one contiguous 16/32 KB run per tile) and the LDS.128 reads are
// conflict-free.
//
// Work item = strip segment: row block I and up to kSeg consecutive column
// blocks J (the rank's tile range in triangle order); CTA b takes the items
// order[b], order[b + grid], ... (longest first, dealt in snake order: item_order).  i-side sums stay in
// registers over the segment; j-side sums are reduced across the 16 thread
// rows through padded shared memory after every tile.  Outputs are fp32 tile
// partials (j side, per tile) and fp64 segment partials (i side, stress),
// summed per row in a fixed order by k_sym_reduce: deterministic, no atomics.
#include <algorithm>
#include <atomic>
#include <cfloat>
#include <cstdint>

#include "fdl_internal.h"

#ifndef FDL_PACKED_FMA
#define FDL_PACKED_FMA 1  // 0: two scalar FFMAs instead of fma.rn.f32x2 (measured slower)
#endif
#ifndef FDL_P2_SHFL
#define FDL_P2_SHFL 0  // 1: P2 hop weights by warp shuffle (experiment; slower in k_sym)
#endif
#ifndef FDL_P1_SHFL
#define FDL_P1_SHFL 0  // 1: P1 hop decode by warp shuffle (experiment; slower)
#endif
#ifndef FDL_BFS_UNROLL
#define FDL_BFS_UNROLL 16  // neighbour frontier loads in flight per warp (MS-BFS)
#endif
constexpr int kBfsUnroll = FDL_BFS_UNROLL;
#ifndef FDL_P1S_CTAS
#define FDL_P1S_CTAS 2  // CTAs per SM of the 2-D line-6 pass
#endif
#ifndef FDL_P1A_CTAS
#define FDL_P1A_CTAS 2  // CTAs per SM of the 2-D fused evaluation pass
#endif
#ifndef FDL_P2_SHFLRED_CTAS
#define FDL_P2_SHFLRED_CTAS 2  // CTAs per SM of the 2-D PCG matvec pass with the butterfly (16 more live registers)
#endif
#ifndef FDL_P2_CTAS
#define FDL_P2_CTAS 3  // CTAs per SM of the 2-D PCG matvec pass
#endif
#ifndef FDL_TPS_P1
#define FDL_TPS_P1 1  // 4-bit P1 (fused / one set) and P1A: tiles per TMA stage
#endif
#ifndef FDL_TPS_P2
#define FDL_TPS_P2 2  // 4-bit P2: tiles of one work item per TMA stage (one mbarrier wait / refill each)
#endif
#ifndef FDL_P2_SHFLRED
#define FDL_P2_SHFLRED 0  // 1: 4-bit 2-D P2 j-side column sums by a warp butterfly (measured slower)
#endif
#ifndef FDL_P2_PBFLY
#define FDL_P2_PBFLY 0  // 1: 4-bit 2-D P2 j-side column sums by a progressive warp butterfly (no j-side buffer)
#endif
#ifndef FDL_P2_MUFU_COLS
// 4-bit P2: bit cc set -> column cc of each 16-byte chunk (4 columns per chunk) takes
// its weights from the MUFU (rcp.approx(h^2), bitwise the table's fp32(1/h^2) for
// h <= 15) instead of the shared-memory table: moves that share of the table's
// shared-memory wavefronts to the otherwise idle XU pipe
#define FDL_P2_MUFU_COLS 0  // measured slower for every share: 0x8 -> 1762, 0xA -> 1613, 0xF -> 1377 vs 1913 GB/s
#endif
#ifndef FDL_P1S_SQRT
#define FDL_P1S_SQRT 0  // 1: P1S stress of X^{k+1} by MUFU.SQRT and 1/h (experiment)
#endif
#ifndef FDL_P1R_SCALAR
#define FDL_P1R_SCALAR 0  // 1: the 2-D one-set R updates (P1R, 1-set P1) as scalar FFMAs instead of FFMA2
#endif
#ifndef FDL_P1S_PACKR
#define FDL_P1S_PACKR 0  // 1: the line-6 pass's R updates of set 1 as FFMA2 on (x, y) instead of 4 FFMA
#endif
#ifndef FDL_MAXST
#define FDL_MAXST 4  // deepest TMA ring of the pair passes
#endif

namespace fdl {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
#ifndef FDL_MBAR_HINT
#define FDL_MBAR_HINT 0  // > 0: suspend-time hint (ns) of the stage waits (the warp sleeps instead of re-polling)
#endif
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity)
{
    uint32_t ok;
#if FDL_MBAR_HINT > 0
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "n"(FDL_MBAR_HINT)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
#endif
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    while (!mbar_try_wait(bar, parity)) {
    }
}
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
__device__ __forceinline__ uint32_t word_of(const uint4& v, int q)
{
    return q == 0 ? v.x : (q == 1 ? v.y : (q == 2 ? v.z : v.w));
}

// hop of entry (row r, column cc of the chunk) of one 16-byte chunk as an
// exact float: one PRMT builds 0x4B0000hh (= 2^23 + h), one FADD removes 2^23.
// u8 chunk: columns 2k, 2k+1, byte cc*8 + r; u16 chunk: column k, bytes 2r, 2r+1.
// `magic` holds 0x4B000000 in a register (a kernel parameter, opaque to
// constant folding) so the selector can be the PRMT immediate: one PRMT per
// hop, no selector materialisation.
template <int SEL>
__device__ __forceinline__ uint32_t prmt_imm(uint32_t a, uint32_t b)
{
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "n"(SEL));
    return d;
}

template <int HB>
__device__ __forceinline__ float chunk_hop(const uint4& ch, int r, int cc, uint32_t magic)
{
    uint32_t bits;
    if (HB == 1) {
        const int byte = cc * 8 + r;
        const uint32_t w = word_of(ch, byte >> 2);
        switch (byte & 3) {
            case 0: bits = prmt_imm<0x7650>(w, magic); break;
            case 1: bits = prmt_imm<0x7651>(w, magic); break;
            case 2: bits = prmt_imm<0x7652>(w, magic); break;
            default: bits = prmt_imm<0x7653>(w, magic); break;
        }
    } else {
        const uint32_t w = word_of(ch, r >> 1);
        bits = (r & 1) ? prmt_imm<0x7632>(w, magic) : prmt_imm<0x7610>(w, magic);
    }
    return __uint_as_float(bits) - 8388608.0f;
}

}  // namespace

// number of output components per mode
template <int MODE, int DIM, int NSETS>
__host__ __device__ constexpr int sym_ncomp()
{
    return MODE == kSymP1 ? NSETS * DIM
                          : (MODE == kSymP1A ? 2 * DIM : ((MODE == kSymP2 || MODE == kSymP1S || MODE == kSymP1R) ? DIM : 1));
}

// floats per vertex in the staged position vector
template <int MODE, int DIM, int NSETS>
__host__ __device__ constexpr int sym_ps()
{
    return (MODE == kSymP1 || MODE == kSymP1S || MODE == kSymP1A || MODE == kSymP1R)
               ? (DIM == 2 ? (NSETS == 1 ? 2 : 4) : (NSETS == 1 ? 4 : 8))
                          : (MODE == kSymP2 ? (DIM == 2 ? 2 : 4) : 4);
}


// tiles per TMA stage: 2 for the 4-bit matvec pass (its per-tile work is short, so halving
// the mbarrier waits and refills pays: C5 P2 1820 -> 1913 GB/s), 1 elsewhere (the line-6 pass
// got slower with 2, and wider tiles would not fit two per stage)
template <int MODE, int HB>
__host__ __device__ constexpr int sym_tps()
{
    return (MODE == kSymP2 && HB == 0) ? FDL_TPS_P2
                                       : ((MODE == kSymP1 || MODE == kSymP1A || MODE == kSymP1R) && HB == 0 ? FDL_TPS_P1 : 1);
}

template <int MODE, int DIM, int NSETS, int HB>
__host__ __device__ constexpr int sym_stage_bytes()
{
    return (int)tile_bytes(HB) + kT * sym_ps<MODE, DIM, NSETS>() * 4;
}

// j-side column sums of the tile by a warp butterfly (registers + SHFL) instead of
// shared-memory stores and the warp flush: the 4-bit 2-D matvec pass, whose
// shared-memory wavefronts bound it
template <int MODE, int DIM, int NSETS, int HB>
__host__ __device__ constexpr bool sym_shflred()
{
    return FDL_P2_SHFLRED && MODE == kSymP2 && DIM == 2 && NSETS == 1 && HB == 0;
}

// floats per lane row of a warp's j-side buffer: 9C keeps the 16 rows of a
// half-warp on distinct banks for the C-wide vector stores
// ... the same butterfly done column by column inside the tile (sym_tile): after
// each column the pair of rows (ty, ty^1) is combined, after each column pair
// the rows (ty, ty^2), and so on, so at most ~3 partial values are live per
// lane (the end-of-tile butterfly holds 16 and needs 2 CTAs/SM); no j-side
// shared-memory buffer, so the TMA ring gets its space
template <int MODE, int DIM, int NSETS, int HB>
__host__ __device__ constexpr bool sym_pbfly()
{
    return FDL_P2_PBFLY && !FDL_P2_SHFLRED && MODE == kSymP2 && DIM == 2 && NSETS == 1 && HB == 0;
}

template <int MODE, int DIM, int NSETS>
__host__ __device__ constexpr int sym_jpitch()
{
    return 9 * sym_ncomp<MODE, DIM, NSETS>();
}

template <int MODE, int DIM, int NSETS>
__host__ __device__ constexpr size_t sym_red_floats()  // the j-side warp buffers
{
    return (size_t)8 * 2 * (16 * sym_jpitch<MODE, DIM, NSETS>() + 16);
}

// CTAs per SM the pass is built for (register budget of __launch_bounds__)
template <int MODE, int DIM>
__host__ __device__ constexpr int sym_ctas_per_sm()
{
    return (MODE == kSymP2 && DIM == 2)    ? (FDL_P2_SHFLRED ? FDL_P2_SHFLRED_CTAS : FDL_P2_CTAS)
           : (MODE == kSymP1A && DIM == 2) ? FDL_P1A_CTAS
           : (MODE == kSymP1S && DIM == 2) ? FDL_P1S_CTAS
                                           : ((DIM == 2 || (MODE != kSymP1 && MODE != kSymP1S && MODE != kSymP1A &&
                                                            MODE != kSymP1R)) ? 2 : 1);
}

// TMA ring depth: as many stages (2..4) as the shared memory left by the
// reduction buffers allows at sym_ctas_per_sm CTAs per SM (228 KB per SM,
// ~1 KB per CTA reserved, ~4 KB static).
template <int MODE, int DIM, int NSETS, int HB>
__host__ __device__ constexpr size_t sym_red_floats_hb()  // j-side warp buffers of this pass (none with sym_pbfly)
{
    return sym_pbfly<MODE, DIM, NSETS, HB>() ? 0 : sym_red_floats<MODE, DIM, NSETS>();
}

template <int MODE, int DIM, int NSETS, int HB>
__host__ __device__ constexpr int sym_stages()
{
    constexpr int budget = 228 * 1024 / sym_ctas_per_sm<MODE, DIM>() - 5 * 1024 -
                           (int)sym_red_floats_hb<MODE, DIM, NSETS, HB>() * 4;
    constexpr int st = budget / (sym_tps<MODE, HB>() * sym_stage_bytes<MODE, DIM, NSETS, HB>());
    return st < 2 ? 2 : (st > FDL_MAXST ? FDL_MAXST : st);
}

template <int MODE, int DIM, int NSETS, int HB>
__host__ __device__ constexpr size_t sym_smem_bytes()
{
    return (size_t)sym_stages<MODE, DIM, NSETS, HB>() * sym_tps<MODE, HB>() * sym_stage_bytes<MODE, DIM, NSETS, HB>() +
           sym_red_floats_hb<MODE, DIM, NSETS, HB>() * 4;
}

// ------------------------------------------------------------ packed FP32x2
// sm_100 executes fp32 pairs as one instruction (FADD2 / FFMA2 / FMUL2, with
// free negation, immediate and scalar-broadcast operands).  The two position
// sets of P1 (X^{k+1}, Xt) and the x/y coordinates of P2 run as pairs: half the
// issue slots of the scalar code for the same fp32 arithmetic (round-to-nearest
// per element, bitwise equal to the scalar ops).
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float lo, float hi)
{
    u64 d;
    asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
    return d;
}
__device__ __forceinline__ void upk(u64 v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
__device__ __forceinline__ u64 fsub2(u64 a, u64 b)
{
    u64 d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c)
{
#if FDL_PACKED_FMA
    u64 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
#else
    // two scalar FFMAs (same IEEE operation per element).  Alone, an FFMA2 with three
    // register pairs issues at ~3.1 cycles per warp against 2 x 1.1 for the scalar pair
    // (scripts/pipe_rates.cu), but inside k_sym the scalar form is slower (more issue
    // slots; C5 P2 1846 -> 1681 GB/s, P1S 15.58 -> 15.70 ms)
    float al, ah, bl, bh, cl, ch;
    upk(a, al, ah);
    upk(b, bl, bh);
    upk(c, cl, ch);
    return pk(fmaf(al, bl, cl), fmaf(ah, bh, ch));
#endif
}
__device__ __forceinline__ u64 fmul2(u64 a, u64 b)
{
    u64 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

// One unordered pair.  Layouts (C components per vertex):
//   P1, 2 sets: [x_s0, x_s1, y_s0, y_s1 (, z_s0, z_s1)]  (sets interleaved, packed)
//   P1, 1 set and P2: [x, y (, z)];  DIAG: [w]
// MODE P1: a_i += q d, a_j += q d (j side negated at the flush), s += u^2
// MODE P2: a_i += w d, a_j += w d;   MODE DIAG: a_i += w, a_j += w
template <int MODE, int DIM, int NSETS, bool SAFE>
__device__ __forceinline__ void sym_pair(const float* xi, const float* xj, float h2, float wlut, bool valid,
                                         float* ai, float* aj, float* s)
{
    if (MODE == kSymP1S && FDL_P1S_SQRT) {
        // experiment: set 0 (stress only) as r0 = sqrt(r2) and u0 = r0 / h - 1 with 1/h from
        // the table (wlut), so only set 1 needs r2 h^2 for its rsqrt
        u64 d[DIM];
        u64 r2 = pk(FLT_MIN, FLT_MIN);
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            d[c] = fsub2(pk(xi[2 * c], xi[2 * c + 1]), pk(xj[2 * c], xj[2 * c + 1]));
            r2 = ffma2(d[c], d[c], r2);
        }
        float r20, r21;
        upk(r2, r20, r21);
        float r0;
        asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(r20));
        float q1 = rsqrt_approx(r21 * h2);
        if (SAFE) q1 = valid ? q1 : 0.0f;
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            float dlo, dhi;
            upk(d[c], dlo, dhi);
            ai[c] = fmaf(q1, dhi, ai[c]);
            aj[c] = fmaf(q1, dhi, aj[c]);
        }
        float u0 = fmaf(r0, wlut, -1.0f), u1 = fmaf(r21, q1, -1.0f);
        if (SAFE) {
            u0 = valid ? u0 : 0.0f;
            u1 = valid ? u1 : 0.0f;
        }
        float s0, s1;
        upk(ffma2(pk(u0, u1), pk(u0, u1), pk(s[0], s[1])), s0, s1);
        s[0] = s0;
        s[1] = s1;
    } else if (MODE == kSymP1S) {
        // two sets, stress of both, R of set 1 only (Xt; R(X^{k+1}) is needed only
        // when the guard rejects, and is then computed by a 1-set pass): the
        // stress arithmetic is the packed 2-set code, R the scalar FMAs of set 1
        u64 d[DIM];
        u64 r2 = pk(FLT_MIN, FLT_MIN);
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            d[c] = fsub2(pk(xi[2 * c], xi[2 * c + 1]), pk(xj[2 * c], xj[2 * c + 1]));
            r2 = ffma2(d[c], d[c], r2);
        }
        float t0, t1;
        upk(fmul2(r2, pk(h2, h2)), t0, t1);
        float q0 = rsqrt_approx(t0), q1 = rsqrt_approx(t1);
        if (SAFE) {
            q0 = valid ? q0 : 0.0f;
            q1 = valid ? q1 : 0.0f;
        }
        if (FDL_P1S_PACKR && DIM == 2) {
            // R of set 1 as two FFMA2 on (x, y) with q1 broadcast (same fma per element)
            float dx0, dx1, dy0, dy1;
            upk(d[0], dx0, dx1);
            upk(d[1], dy0, dy1);
            const u64 d1 = pk(dx1, dy1), qq = pk(q1, q1);
            float lo, hi;
            upk(ffma2(qq, d1, pk(ai[0], ai[1])), lo, hi);
            ai[0] = lo;
            ai[1] = hi;
            upk(ffma2(qq, d1, pk(aj[0], aj[1])), lo, hi);
            aj[0] = lo;
            aj[1] = hi;
        } else {
#pragma unroll
            for (int c = 0; c < DIM; ++c) {
                float dlo, dhi;
                upk(d[c], dlo, dhi);
                ai[c] = fmaf(q1, dhi, ai[c]);
                aj[c] = fmaf(q1, dhi, aj[c]);
            }
        }
        float u0, u1;
        upk(ffma2(r2, pk(q0, q1), pk(-1.0f, -1.0f)), u0, u1);
        if (SAFE) {
            u0 = valid ? u0 : 0.0f;
            u1 = valid ? u1 : 0.0f;
        }
        float s0, s1;
        upk(ffma2(pk(u0, u1), pk(u0, u1), pk(s[0], s[1])), s0, s1);
        s[0] = s0;
        s[1] = s1;
    } else if (MODE == kSymP1 && NSETS == 2) {
        u64 d[DIM];
        u64 r2 = pk(FLT_MIN, FLT_MIN);  // r^2 > 0 for coincident points: zero R term
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            d[c] = fsub2(pk(xi[2 * c], xi[2 * c + 1]), pk(xj[2 * c], xj[2 * c + 1]));
            r2 = ffma2(d[c], d[c], r2);
        }
        float t0, t1;
        upk(fmul2(r2, pk(h2, h2)), t0, t1);
        float q0 = rsqrt_approx(t0), q1 = rsqrt_approx(t1);  // 1/(h r) per set
        if (SAFE) {
            q0 = valid ? q0 : 0.0f;
            q1 = valid ? q1 : 0.0f;
        }
        const u64 q = pk(q0, q1);
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            float lo, hi;
            upk(ffma2(q, d[c], pk(ai[2 * c], ai[2 * c + 1])), lo, hi);
            ai[2 * c] = lo;
            ai[2 * c + 1] = hi;
            upk(ffma2(q, d[c], pk(aj[2 * c], aj[2 * c + 1])), lo, hi);
            aj[2 * c] = lo;
            aj[2 * c + 1] = hi;
        }
        float u0, u1;
        upk(ffma2(r2, q, pk(-1.0f, -1.0f)), u0, u1);  // r/h - 1 per set
        if (SAFE) {
            u0 = valid ? u0 : 0.0f;
            u1 = valid ? u1 : 0.0f;
        }
        const u64 u = pk(u0, u1);
        float s0, s1;
        upk(ffma2(u, u, pk(s[0], s[1])), s0, s1);
        s[0] = s0;
        s[1] = s1;
    } else if ((MODE == kSymP1 || MODE == kSymP1R) && DIM == 2) {
        // one set, 2-D: (x, y) as a packed pair for delta and the R updates (same
        // per-element IEEE operations and order as the scalar code below); P1R: R only
        const u64 d = fsub2(pk(xi[0], xi[1]), pk(xj[0], xj[1]));
        float dx, dy;
        upk(d, dx, dy);
        const float r2 = fmaf(dy, dy, fmaf(dx, dx, FLT_MIN));
        float q = rsqrt_approx(r2 * h2);
        float u = fmaf(r2, q, -1.0f);
        if (SAFE) {
            q = valid ? q : 0.0f;
            u = valid ? u : 0.0f;
        }
        if (FDL_P1R_SCALAR) {
            // four scalar FFMAs (the same IEEE fma per element as the packed pair)
            ai[0] = fmaf(q, dx, ai[0]);
            ai[1] = fmaf(q, dy, ai[1]);
            aj[0] = fmaf(q, dx, aj[0]);
            aj[1] = fmaf(q, dy, aj[1]);
        } else {
            const u64 qq = pk(q, q);
            float lo, hi;
            upk(ffma2(qq, d, pk(ai[0], ai[1])), lo, hi);
            ai[0] = lo;
            ai[1] = hi;
            upk(ffma2(qq, d, pk(aj[0], aj[1])), lo, hi);
            aj[0] = lo;
            aj[1] = hi;
        }
        if (MODE == kSymP1) s[0] = fmaf(u, u, s[0]);
    } else if (MODE == kSymP1 || MODE == kSymP1R) {
        float d[DIM];
        float r2 = FLT_MIN;
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            d[c] = xi[c] - xj[c];
            r2 = fmaf(d[c], d[c], r2);
        }
        float q = rsqrt_approx(r2 * h2);  // 1/(h r) = w' d' / r
        float u = fmaf(r2, q, -1.0f);     // r/h - 1
        if (SAFE) {
            q = valid ? q : 0.0f;
            u = valid ? u : 0.0f;
        }
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            ai[c] = fmaf(q, d[c], ai[c]);
            aj[c] = fmaf(q, d[c], aj[c]);
        }
        if (MODE == kSymP1) s[0] = fmaf(u, u, s[0]);
    } else if (MODE == kSymP1A) {
        // one set: stress and R as the 1-set P1 pass (same operations and order, so
        // R and f are bitwise those of kSymP1), plus (L^W X)_i = sum_j w_ij (x_i - x_j)
        // in difference form on the same delta (w = wlut = 1/h^2, the P2 table value)
        float d[DIM];
        float r2 = FLT_MIN;
        float q, u;
        float w = wlut;
        if (DIM == 2) {
            const u64 dd = fsub2(pk(xi[0], xi[1]), pk(xj[0], xj[1]));
            upk(dd, d[0], d[1]);
            r2 = fmaf(d[1], d[1], fmaf(d[0], d[0], FLT_MIN));
            q = rsqrt_approx(r2 * h2);
            u = fmaf(r2, q, -1.0f);
            if (SAFE) {
                q = valid ? q : 0.0f;
                u = valid ? u : 0.0f;
                w = valid ? w : 0.0f;
            }
            float lo, hi;
            upk(ffma2(pk(q, q), dd, pk(ai[0], ai[1])), lo, hi);
            ai[0] = lo;
            ai[1] = hi;
            upk(ffma2(pk(q, q), dd, pk(aj[0], aj[1])), lo, hi);
            aj[0] = lo;
            aj[1] = hi;
            upk(ffma2(pk(w, w), dd, pk(ai[2], ai[3])), lo, hi);
            ai[2] = lo;
            ai[3] = hi;
            upk(ffma2(pk(w, w), dd, pk(aj[2], aj[3])), lo, hi);
            aj[2] = lo;
            aj[3] = hi;
        } else {
#pragma unroll
            for (int c = 0; c < DIM; ++c) {
                d[c] = xi[c] - xj[c];
                r2 = fmaf(d[c], d[c], r2);
            }
            q = rsqrt_approx(r2 * h2);
            u = fmaf(r2, q, -1.0f);
            if (SAFE) {
                q = valid ? q : 0.0f;
                u = valid ? u : 0.0f;
                w = valid ? w : 0.0f;
            }
#pragma unroll
            for (int c = 0; c < DIM; ++c) {
                ai[c] = fmaf(q, d[c], ai[c]);
                aj[c] = fmaf(q, d[c], aj[c]);
                ai[DIM + c] = fmaf(w, d[c], ai[DIM + c]);
                aj[DIM + c] = fmaf(w, d[c], aj[DIM + c]);
            }
        }
        s[0] = fmaf(u, u, s[0]);
    } else if (MODE == kSymP2) {
        // Product form of the L^W matvec: (L^W p)_i = diag_i p_i - sum_j w_ij p_j
        // (P:65-68), so a pair adds w p_j to row i and w p_i to row j; the
        // diagonal term is applied after the reduction (k_p2_finish) on the
        // same fp32 staged values, which are centred (p - mean p; L 1 = 0) so
        // the sums carry no common offset.
        float w = wlut;  // w' = 1/h^2 (table for u8 / 4-bit, MUFU rcp for u16; 0 for h = 0)
        if (SAFE) w = valid ? w : 0.0f;
        const u64 wp = pk(w, w);
        float lo, hi;
        upk(ffma2(wp, pk(xj[0], xj[1]), pk(ai[0], ai[1])), lo, hi);
        ai[0] = lo;
        ai[1] = hi;
        upk(ffma2(wp, pk(xi[0], xi[1]), pk(aj[0], aj[1])), lo, hi);
        aj[0] = lo;
        aj[1] = hi;
        if (DIM == 3) {
            ai[2] = fmaf(w, xj[2], ai[2]);
            aj[2] = fmaf(w, xi[2], aj[2]);
        }
    } else {
        // DIAG: w' = fp32(1/h^2) correctly rounded -- the table value at 4 bits (the
        // P2 table), __frcp_rn(h^2) at 8/16 bits (sym_tile); the same number either way
        float w = wlut;
        if (SAFE) w = valid ? w : 0.0f;
        ai[0] += w;
        aj[0] += w;
    }
}

// General weights (NEXT-3: weighted graphs, any alpha): d = the stored fp32
// path length (device units), w = d^alpha = 2^(alpha log2 d) (MUFU LG2/EX2),
// w d for the L^X coefficient.  P1 per set: q = 1/r, R += (w d q) delta,
// s += w (r - d)^2 (Eq. 1); P2: w p_j / w p_i (product form); DIAG: w.
__device__ __forceinline__ float lg2_approx(float x)
{
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float ex2_approx(float x)
{
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int MODE, int DIM, int NSETS, bool SAFE>
__device__ __forceinline__ void gen_pair(const float* xi, const float* xj, float d, float alpha, bool valid,
                                         float* ai, float* aj, float* s)
{
    float w = ex2_approx(alpha * lg2_approx(d));
    if (SAFE) w = valid ? w : 0.0f;
    if (MODE == kSymP1) {
        const float c = w * d;
#pragma unroll
        for (int k = 0; k < NSETS; ++k) {
            float dl[DIM];
            float r2 = FLT_MIN;
#pragma unroll
            for (int q = 0; q < DIM; ++q) {
                dl[q] = xi[q * NSETS + k] - xj[q * NSETS + k];
                r2 = fmaf(dl[q], dl[q], r2);
            }
            const float q1 = rsqrt_approx(r2);
            const float coef = c * q1;
#pragma unroll
            for (int q = 0; q < DIM; ++q) {
                ai[q * NSETS + k] = fmaf(coef, dl[q], ai[q * NSETS + k]);
                aj[q * NSETS + k] = fmaf(coef, dl[q], aj[q * NSETS + k]);
            }
            const float u = fmaf(r2, q1, -d);
            s[k] = fmaf(w * u, u, s[k]);
        }
    } else if (MODE == kSymP2) {
#pragma unroll
        for (int q = 0; q < DIM; ++q) {
            ai[q] = fmaf(w, xj[q], ai[q]);
            aj[q] = fmaf(w, xi[q], aj[q]);
        }
    } else {
        ai[0] += w;
        aj[0] += w;
    }
}

template <int MODE, int DIM, int NSETS, int HB, bool SAFE>
__device__ __forceinline__ void sym_tile(const uint8_t* sD, const float* sP, const float* lut, const float2* lut2,
                                         const float2* lutw, uint32_t magic, float alpha, int ty, int tx, bool diag,
                                         const float (&xi)[8][NSETS * DIM], float (&ai)[8][sym_ncomp<MODE, DIM, NSETS>()],
                                         float* myred, float (&sf)[2][NSETS], float (&jv)[8 * sym_ncomp<MODE, DIM, NSETS>()])
{
    constexpr int C = sym_ncomp<MODE, DIM, NSETS>();
    constexpr bool BFLY = sym_shflred<MODE, DIM, NSETS, HB>();
    constexpr bool PBFLY = sym_pbfly<MODE, DIM, NSETS, HB>();
    constexpr int PS = sym_ps<MODE, DIM, NSETS>();
    constexpr int NCH = HB ? 4 * HB : 2;  // 16-byte chunks per thread
    constexpr int CPC = HB ? 2 / HB : 4;  // columns per chunk
    const int tid = tx * 16 + ty;  // chunk owner index of the tile layout (sym_offset)
    if (HB == kHbDist) {
        // fp32 path lengths: column c = chunks 2c, 2c+1 (rows 0-3, 4-7)
#pragma unroll 1
        for (int c = 0; c < 8; ++c) {
            const float4 d0 = *reinterpret_cast<const float4*>(sD + ((size_t)(2 * c) * 256 + tid) * 16);
            const float4 d1 = *reinterpret_cast<const float4*>(sD + ((size_t)(2 * c + 1) * 256 + tid) * 16);
            const float dv[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
            const int jl = tx * 8 + c;
            const int js = c * 16 + tx;
            float xj[PS];
#pragma unroll
            for (int q = 0; q < PS; ++q) xj[q] = sP[js * PS + q];
            float aj[C];
#pragma unroll
            for (int v = 0; v < C; ++v) aj[v] = 0.0f;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                bool valid = true;
                if (SAFE) valid = (dv[r] > 0.0f) && (!diag || (ty * 8 + r < jl));
                const float dd = (SAFE && !valid) ? 1.0f : dv[r];
                gen_pair<MODE, DIM, NSETS, SAFE>(&xi[r][0], xj, dd, alpha, valid, &ai[r][0], aj, &sf[r & 1][0]);
            }
#pragma unroll
            for (int v = 0; v < C; ++v) myred[c * C + v] = aj[v];
        }
        return;
    }
    if (HB == 0) {
        // 4-bit tiles: one byte = hops of rows (2p, 2p+1) of a column, one 8-byte
        // LUT entry per byte gives both decoded values (h^2 for P1/DIAG, w' = 1/h^2
        // for P2): 2 ALU ops + 1 LDS.64 per two pairs, no FP32-pipe decode work.
        // Both chunks are loaded up front and the 8 columns fully unrolled, so the
        // LUT loads of the next column overlap the FP work of this one; the
        // j-side sum of a column is split over even/odd rows (two 4-long FFMA
        // chains instead of one 8-long chain).
        uint4 chs[NCH];
        float pv1[8], pv2[4], pv3[2];  // progressive butterfly partials (PBFLY)
        const bool b0 = ty & 1, b1 = ty & 2, b2 = ty & 4, b3 = ty & 8;
        const float wtab = MODE == kSymP2 ? lut[threadIdx.x & 15]  // w'_h for h = lane & 15 (w'_0 = 0)
                                          : (float)((threadIdx.x & 15) * (threadIdx.x & 15));  // h^2 (shuffle experiments)
#pragma unroll
        for (int kc = 0; kc < NCH; ++kc) chs[kc] = *reinterpret_cast<const uint4*>(sD + ((size_t)kc * 256 + tid) * 16);
#pragma unroll
        for (int kc = 0; kc < NCH; ++kc) {
            const uint4 ch = chs[kc];
#pragma unroll
            for (int cc = 0; cc < CPC; ++cc) {
                const int c = kc * CPC + cc;
                const int jl = tx * 8 + c;
                const int js = c * 16 + tx;
                float xj[PS];
                if (PS == 2) {
                    const float2 t = *reinterpret_cast<const float2*>(sP + js * PS);
                    xj[0] = t.x; xj[1] = t.y;
                } else {
#pragma unroll
                    for (int q = 0; q < PS / 4; ++q) {
                        const float4 t = *reinterpret_cast<const float4*>(sP + js * PS + 4 * q);
                        xj[4 * q] = t.x; xj[4 * q + 1] = t.y; xj[4 * q + 2] = t.z; xj[4 * q + 3] = t.w;
                    }
                }
                float aj[2][C];
#pragma unroll
                for (int v = 0; v < C; ++v) aj[0][v] = aj[1][v] = 0.0f;
                const uint32_t w = word_of(ch, cc);
                float2 e[4], ew[4];
                if (MODE == kSymP2 && ((FDL_P2_MUFU_COLS >> cc) & 1)) {
                    // the four bytes of the word at once: hi nibbles H, lo = (lo' - 4 hi) mod 16
                    // per byte lane (lo' | 64 keeps each byte's difference from borrowing)
                    const uint32_t H = (w >> 4) & 0x0F0F0F0Fu;
                    const uint32_t L = (((w & 0x0F0F0F0Fu) | 0x40404040u) - (H << 2)) & 0x0F0F0F0Fu;
#pragma unroll
                    for (int rp = 0; rp < 4; ++rp) {
                        uint32_t bl, bh;  // 0x4B0000hh = 2^23 + h
                        switch (rp) {
                            case 0: bl = prmt_imm<0x7650>(L, magic); bh = prmt_imm<0x7650>(H, magic); break;
                            case 1: bl = prmt_imm<0x7651>(L, magic); bh = prmt_imm<0x7651>(H, magic); break;
                            case 2: bl = prmt_imm<0x7652>(L, magic); bh = prmt_imm<0x7652>(H, magic); break;
                            default: bl = prmt_imm<0x7653>(L, magic); bh = prmt_imm<0x7653>(H, magic); break;
                        }
                        const float hl = __uint_as_float(bl) - 8388608.0f, hh = __uint_as_float(bh) - 8388608.0f;
                        float wl = rcp_approx(hl * hl), wh = rcp_approx(hh * hh);
                        if (SAFE) {  // h = 0 (diagonal, padding): weight 0, as the table's entry
                            wl = hl > 0.0f ? wl : 0.0f;
                            wh = hh > 0.0f ? wh : 0.0f;
                        }
                        e[rp] = make_float2(wl, wh);
                    }
                } else
#pragma unroll
                for (int rp = 0; rp < 4; ++rp) {
                    const uint32_t off = rp == 0 ? ((w << 3) & 0x7f8u) : ((w >> (8 * rp - 3)) & 0x7f8u);
                    if (MODE == kSymP1A || (MODE == kSymP1S && FDL_P1S_SQRT))  // w' = 1/h^2 (P1A) or 1/h (P1S exp.)
                        ew[rp] = *reinterpret_cast<const float2*>(reinterpret_cast<const char*>(lutw) + off);
                    if ((FDL_P2_SHFL && MODE == kSymP2) || (FDL_P1_SHFL && (MODE == kSymP1 || MODE == kSymP1S))) {
                        // experiment (off): weights by warp shuffle from a 16-entry register
                        // table (lane h holds w'_h or h^2) instead of the shared-memory table.
                        // The shuffle reads lane (index mod 32) and the table repeats every 16
                        // lanes, so only the low 4 bits of each index matter: hi = the shifted
                        // word, lo = ((b & 15) - 4 hi) mod 16 = x - 4 y (nib_decode_lo).  P2's
                        // per-tile work alone gets 21% faster, but inside k_sym the pass gets
                        // 14% slower (two SHFL per byte load the MIO queue the warp flush also
                        // uses); P1S 7% slower
                        const uint32_t x = rp == 0 ? w : (w >> (8 * rp)), y = w >> (8 * rp + 4);
                        e[rp] = make_float2(__shfl_sync(0xffffffffu, wtab, (int)(x - 4u * y)),
                                            __shfl_sync(0xffffffffu, wtab, (int)y));
                        continue;
                    }
                    e[rp] = *reinterpret_cast<const float2*>(reinterpret_cast<const char*>(lut2) + off);
                }
#pragma unroll
                for (int rp = 0; rp < 4; ++rp) {
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        const int r = 2 * rp + hh;
                        const float v = hh ? e[rp].y : e[rp].x;
                        const float vw = (MODE == kSymP1A || (MODE == kSymP1S && FDL_P1S_SQRT))
                                             ? (hh ? ew[rp].y : ew[rp].x) : v;
                        bool valid = true;
                        if (SAFE) valid = (v > 0.0f) && (!diag || (ty * 8 + r < jl));
                        sym_pair<MODE, DIM, NSETS, SAFE>(&xi[r][0], xj, v, vw, valid, &ai[r][0], &aj[hh][0], &sf[hh][0]);
                    }
                }
                if constexpr (PBFLY) {
                    // rows (ty, ty^1) of column c: the lane keeps component b0; then column
                    // pairs with lane ty^2 (keeps column 2m + b1), column quads with ty^4,
                    // the two halves with ty^8: the pairs added are those of
                    // sym_flush_warp's tree, so the sums are bitwise the same, and lane ty
                    // ends with output (column 4 b3 + 2 b2 + b1, component b0) = e = ty
                    const float s0 = aj[0][0] + aj[1][0], s1 = aj[0][1] + aj[1][1];
                    pv1[c] = (b0 ? s1 : s0) + __shfl_xor_sync(0xffffffffu, b0 ? s0 : s1, 1);
                    if (c & 1) {
                        const float lo = pv1[c - 1], hi = pv1[c];
                        pv2[c >> 1] = (b1 ? hi : lo) + __shfl_xor_sync(0xffffffffu, b1 ? lo : hi, 2);
                    }
                    if ((c & 3) == 3) {
                        const float lo = pv2[(c >> 1) - 1], hi = pv2[c >> 1];
                        pv3[c >> 2] = (b2 ? hi : lo) + __shfl_xor_sync(0xffffffffu, b2 ? lo : hi, 4);
                    }
                    if (c == 7) jv[0] = (b3 ? pv3[1] : pv3[0]) + __shfl_xor_sync(0xffffffffu, b3 ? pv3[0] : pv3[1], 8);
                } else {
#pragma unroll
                    for (int v = 0; v < C; ++v) {
                        if (BFLY)
                            jv[c * C + v] = aj[0][v] + aj[1][v];
                        else
                            myred[c * C + v] = aj[0][v] + aj[1][v];
                    }
                }
            }
        }
        return;
    }
#pragma unroll 1
    for (int kc = 0; kc < NCH; ++kc) {
        const uint4 ch = *reinterpret_cast<const uint4*>(sD + ((size_t)kc * 256 + tid) * 16);
#pragma unroll
        for (int cc = 0; cc < CPC; ++cc) {
            const int c = kc * CPC + cc;
            const int jl = tx * 8 + c;
            const int js = c * 16 + tx;  // staged slot of column jl (stage_slot)
            float xj[PS];
            if (PS == 2) {
                const float2 t = *reinterpret_cast<const float2*>(sP + js * PS);
                xj[0] = t.x; xj[1] = t.y;
            } else {
#pragma unroll
                for (int q = 0; q < PS / 4; ++q) {
                    const float4 t = *reinterpret_cast<const float4*>(sP + js * PS + 4 * q);
                    xj[4 * q] = t.x; xj[4 * q + 1] = t.y; xj[4 * q + 2] = t.z; xj[4 * q + 3] = t.w;
                }
            }
            float aj[2][C];  // even / odd rows (same split and order as the 4-bit path)
#pragma unroll
            for (int v = 0; v < C; ++v) aj[0][v] = aj[1][v] = 0.0f;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                float hf, h2, wl = 0.0f;
                if (MODE == kSymP2 && HB == 1) {
                    const int byte = cc * 8 + r;
                    const uint32_t hb8 = __byte_perm(word_of(ch, byte >> 2), 0u, 0x4440u + (uint32_t)(byte & 3));
                    wl = lut[hb8];
                    h2 = wl;  // only its sign (h > 0) is used below
                } else {
                    hf = chunk_hop<HB>(ch, r, cc, magic);
                    h2 = hf * hf;
                    if (MODE == kSymP2) wl = rcp_approx(h2);
                    if (MODE == kSymDiag) wl = __frcp_rn(h2);
                    if (MODE == kSymP1A) wl = HB == 1 ? lut[(int)hf] : rcp_approx(h2);  // as P2 at this width
                }
                bool valid = true;
                if (SAFE) valid = (h2 > 0.0f) && (!diag || (ty * 8 + r < jl));
                sym_pair<MODE, DIM, NSETS, SAFE>(&xi[r][0], xj, h2, wl, valid, &ai[r][0], &aj[r & 1][0], &sf[r & 1][0]);
            }
#pragma unroll
            for (int v = 0; v < C; ++v) myred[c * C + v] = aj[0][v] + aj[1][v];
        }
    }
}

// j-side column sums by a warp butterfly: lane (h = tx & 1, ty) holds jv[e] =
// its 8-row partial of output e = c * C + v (column tx * 8 + c).  Four halving
// exchanges with lanes ty ^ 1, ^ 2, ^ 4, ^ 8 (each lane keeps the half of the
// vector picked by that bit of ty and adds the partner's copy) leave lane ty
// with the 16-row sum of output e = 8 b0 + 4 b1 + 2 b2 + b3 (b_k = bit k of ty).
// The pairs added at each level are those of sym_flush_warp's tree (rows r and
// r + w for w = 1, 2, 4, 8), so the sums are bitwise the same.  Needs 8C = 16.
template <int MODE, int DIM, int NSETS>
__device__ __forceinline__ void sym_bfly_warp(const float (&jv)[16], float* jpart_warp, int lane)
{
    const int ty = lane & 15, h = lane >> 4;
    const bool b0 = ty & 1, b1 = ty & 2, b2 = ty & 4, b3 = ty & 8;
    float l0[8], l1[4], l2[2];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const float send = b0 ? jv[i] : jv[8 + i], keep = b0 ? jv[8 + i] : jv[i];
        l0[i] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float send = b1 ? l0[i] : l0[4 + i], keep = b1 ? l0[4 + i] : l0[i];
        l1[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const float send = b2 ? l1[i] : l1[2 + i], keep = b2 ? l1[2 + i] : l1[i];
        l2[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    const float send = b3 ? l2[0] : l2[1], keep = b3 ? l2[1] : l2[0];
    const float tot = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    const int e = (b0 ? 8 : 0) + (b1 ? 4 : 0) + (b2 ? 2 : 0) + (b3 ? 1 : 0);
    jpart_warp[h * 16 + e] = tot;  // P2: symmetric, no sign
}

// j-side flush of one tile by one warp (no CTA barrier): the warp's lanes are
// (h = tx & 1, ty = 0..15); lane (h, ty) wrote its 8 x C column partials to
// row ty of half h of the warp buffer.  Output e = h * 8C + c * C + v (column
// tx * 8 + c, component v) is the fixed-order tree sum over the 16 rows, stored
// as fp32 jpart[tile][col][C]; the warp's outputs are one contiguous run of 16C
// floats.  The j-side sign: P1 accumulates +term for row i and -term for row j
// (antisymmetric); P2 (product form) and DIAG are symmetric.
template <int MODE, int DIM, int NSETS>
__device__ __forceinline__ void sym_flush_warp(const float* wbuf, float* jpart_warp, int lane)
{
    constexpr int C = sym_ncomp<MODE, DIM, NSETS>();
    constexpr int P = sym_jpitch<MODE, DIM, NSETS>();
    constexpr float SIGN = (MODE == kSymP1 || MODE == kSymP1S || MODE == kSymP1A || MODE == kSymP1R)
                               ? -1.0f : 1.0f;  // P1 antisymmetric; P2, DIAG symmetric
    __syncwarp();
#pragma unroll
    for (int e0 = 0; e0 < 16 * C; e0 += 32) {
        const int e = e0 + lane;
        if (16 * C % 32 == 0 || e < 16 * C) {
            const int h = e / (8 * C), o = e % (8 * C);
            const float* src = wbuf + h * (16 * P + 16) + o;
            float v[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = src[r * P];
#pragma unroll
            for (int w = 1; w < 16; w *= 2)
#pragma unroll
                for (int r = 0; r < 16; r += 2 * w) v[r] += v[r + w];
            jpart_warp[e] = SIGN * v[0];
        }
    }
    __syncwarp();  // the buffer is rewritten by the next tile
}

template <int MODE, int DIM, int NSETS, int HB>
__global__ void __launch_bounds__(256, sym_ctas_per_sm<MODE, DIM>()) k_sym(const SymArgs a)
{
    constexpr int C = sym_ncomp<MODE, DIM, NSETS>();
    constexpr int PS = sym_ps<MODE, DIM, NSETS>();
    constexpr int STAGE = sym_stage_bytes<MODE, DIM, NSETS, HB>();
    constexpr int DT = (int)tile_bytes(HB);
    constexpr int JP = sym_jpitch<MODE, DIM, NSETS>();
    constexpr int NST = sym_stages<MODE, DIM, NSETS, HB>();
    constexpr int NW = 8;  // warps
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t full[NST];
    __shared__ int drained[NST];  // warps done with the stage's current tile
    __shared__ int prod[2];       // producer cursor {item, tile in item}
    __shared__ float lut[256];
    __shared__ float2 lut2[HB == 0 ? 256 : 1];
    __shared__ float2 lutw2[(HB == 0 && (MODE == kSymP1A || (MODE == kSymP1S && FDL_P1S_SQRT))) ? 256 : 1];
    constexpr int TPS = sym_tps<MODE, HB>();
    constexpr int SLOT = TPS * STAGE;  // one stage: up to TPS consecutive tiles of one item
    float* red = reinterpret_cast<float*>(smem + (size_t)NST * SLOT);

    // Thread (ty, tx) owns rows ty*8.. and columns tx*8.. of a tile; a warp holds
    // two thread columns (tx = 2w, 2w+1) x all 16 thread rows, so the j-side sum
    // over ty stays inside the warp.
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int ty = lane & 15, tx = tid >> 4;
    if ((int)blockIdx.x >= a.nitems) return;
    lut[tid] = tid ? 1.0f / (float)(tid * tid) : 0.0f;  // w'_h = fp32(1/h^2), correctly rounded
    if (HB == 0) {  // entry of encoded byte tid: (row 2p, row 2p+1) -> h^2 (P1, DIAG) or w' (P2)
        const int lo = (int)nib_decode_lo((uint32_t)tid), hi = (int)nib_decode_hi((uint32_t)tid);
        lut2[tid] = (MODE == kSymP2 || MODE == kSymDiag)
                        ? make_float2(lo ? 1.0f / (float)(lo * lo) : 0.0f, hi ? 1.0f / (float)(hi * hi) : 0.0f)
                        : make_float2((float)(lo * lo), (float)(hi * hi));
        if (MODE == kSymP1A)
            lutw2[tid] = make_float2(lo ? 1.0f / (float)(lo * lo) : 0.0f, hi ? 1.0f / (float)(hi * hi) : 0.0f);
        if (MODE == kSymP1S && FDL_P1S_SQRT)
            lutw2[tid] = make_float2(lo ? 1.0f / (float)lo : 0.0f, hi ? 1.0f / (float)hi : 0.0f);
    }
    // producer: the next tile of this CTA's items (cursor in shared memory; it is
    // advanced by whichever warp frees a stage last, see below)
    auto issue = [&](int stage) {
        int p_item = prod[0], p_t = prod[1];
        if (p_item >= a.nitems) return;
        const int4 it = a.items[a.order[p_item]];  // {I, J0, ntiles, first local tile}
        const int cnt = min(TPS, it.z - p_t);  // tiles of this item in the stage
        fence_proxy_async();
        mbar_arrive_expect_tx(&full[stage], cnt * STAGE);
        for (int k = 0; k < cnt; ++k) {
            const int J = it.y + p_t + k;
            const int64_t lt = (int64_t)it.w + p_t + k;
            uint8_t* base = smem + (size_t)stage * SLOT + (size_t)k * STAGE;
            FDL_DCHECK(lt >= 0 && lt < a.ntiles && J >= 0 && (int64_t)(J + 1) * kT <= a.nstage);
            tma_load_1d(base, a.D + lt * DT, DT, &full[stage]);
            tma_load_1d(base + DT, a.pos + (int64_t)J * kT * PS, kT * PS * 4, &full[stage]);
        }
        p_t += cnt;
        if (p_t == it.z) {
            p_t = 0;
            p_item += gridDim.x;
        }
        prod[0] = p_item;
        prod[1] = p_t;
    };
    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 1);
            drained[s] = 0;
        }
        fence_mbar_init();
        prod[0] = blockIdx.x;
        prod[1] = 0;
        for (int s = 0; s < NST; ++s) issue(s);
    }
    __syncthreads();

    float* wrow = red + wid * 2 * (16 * JP + 16) + (tx & 1) * (16 * JP + 16) + ty * JP;  // this lane's j row
    const float* wbuf = red + wid * 2 * (16 * JP + 16);
    int stage = 0;
    uint32_t phase = 0;
    for (int slot = blockIdx.x; slot < a.nitems; slot += gridDim.x) {
        const int item = a.order[slot];  // outputs are indexed by item: any schedule gives the same sums
        const int4 it = a.items[item];
        const int I = it.x;
        FDL_DCHECK(it.z >= 1 && it.w >= 0 && (int64_t)it.w + it.z <= a.ntiles && I <= it.y &&
                   (int64_t)(I + 1) * kT <= a.nstage);
        float xi[8][NSETS * DIM];
        float ai[8][C];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int64_t gi = stage_slot((int64_t)I * kT + ty * 8 + r);
#pragma unroll
            for (int q = 0; q < NSETS * DIM; ++q) xi[r][q] = a.pos[gi * PS + q];
#pragma unroll
            for (int v = 0; v < C; ++v) ai[r][v] = 0.0f;
        }
        double s64[NSETS];
#pragma unroll
        for (int s = 0; s < NSETS; ++s) s64[s] = 0.0;
        for (int t = 0; t < it.z; ++t) {
            const int J = it.y + t;
            const bool diag = (J == I);
            const bool safe = diag || (int64_t)(J + 1) * kT > a.n || (int64_t)(I + 1) * kT > a.n;
            const int k = t % TPS;                            // tile within its stage
            const bool last = k == TPS - 1 || t == it.z - 1;  // the stage's last tile
            if (k == 0) mbar_wait(&full[stage], phase);
            const uint8_t* sD = smem + (size_t)stage * SLOT + (size_t)k * STAGE;
            const float* sP = reinterpret_cast<const float*>(sD + DT);
            float sf[2][NSETS];  // stress of the tile, even / odd rows (two independent FMA chains)
#pragma unroll
            for (int s = 0; s < NSETS; ++s) sf[0][s] = sf[1][s] = 0.0f;
            float jv[8 * C];  // j-side column partials (butterfly mode)
            if (safe)
                sym_tile<MODE, DIM, NSETS, HB, true>(sD, sP, lut, lut2, lutw2, a.magic, a.alpha, ty, tx, diag, xi, ai, wrow, sf, jv);
            else
                sym_tile<MODE, DIM, NSETS, HB, false>(sD, sP, lut, lut2, lutw2, a.magic, a.alpha, ty, tx, diag, xi, ai, wrow, sf, jv);
#pragma unroll
            for (int s = 0; s < NSETS; ++s) s64[s] += (double)sf[0][s] + (double)sf[1][s];
            // stage consumed by this warp; the last of the 8 warps refills it
            if (last) {
                __syncwarp();
                if (lane == 0) {
                    __threadfence_block();
                    if (atomicAdd(&drained[stage], 1) == NW - 1) {
                        __threadfence_block();
                        drained[stage] = 0;
                        issue(stage);
                    }
                }
            }
            FDL_DCHECK((int64_t)it.w + t < a.ntiles);
            if constexpr (sym_shflred<MODE, DIM, NSETS, HB>())
                sym_bfly_warp<MODE, DIM, NSETS>(jv, a.jpart + ((size_t)it.w + t) * kT * C + wid * 16 * C, lane);
            else if constexpr (sym_pbfly<MODE, DIM, NSETS, HB>())
                a.jpart[((size_t)it.w + t) * kT * C + wid * 16 * C + lane] = jv[0];  // P2: symmetric, no sign
            else
                sym_flush_warp<MODE, DIM, NSETS>(wbuf, a.jpart + ((size_t)it.w + t) * kT * C + wid * 16 * C, lane);
            if (last && ++stage == NST) {
                stage = 0;
                phase ^= 1u;
            }
        }
        // i-side, per warp (no CTA barrier): the warp's two thread columns (lanes
        // ty and ty + 16) are summed by one xor-shuffle, and lane (ty, h) writes
        // rows ty*8 + 4h .. +3 of the warp's partial [item][warp][row][C] (fp32;
        // k_sym_reduce sums items and warps in a fixed order, in fp64).
        {
            float* ip = a.ipart + ((size_t)item * 8 + wid) * kT * C + (size_t)ty * 8 * C;
            const int h = lane >> 4;
#pragma unroll
            for (int r = 0; r < 8; ++r)
#pragma unroll
                for (int v = 0; v < C; ++v) {
                    const float tot = ai[r][v] + __shfl_xor_sync(0xffffffffu, ai[r][v], 16);
                    if ((r >> 2) == h) ip[r * C + v] = tot;
                }
        }
        if (MODE == kSymP1 || MODE == kSymP1S || MODE == kSymP1A) {
            // stress of the warp's share of the segment: fixed-order warp butterfly of
            // the fp64 thread sums -> spart[item][warp][set]
#pragma unroll
            for (int s = 0; s < NSETS; ++s) {
                double v = s64[s];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0) a.spart[((size_t)item * 8 + wid) * NSETS + s] = v;
            }
        }
    }
}

// Opt-in dynamic shared memory of a kernel, once per device (thread-safe: contexts of
// several ranks may launch from several host threads, e.g. the loopback group)
template <typename K>
static cudaError_t ensure_smem_attr(K* fn, size_t sm, std::atomic<uint32_t>& done)
{
    int dev = 0;
    cudaGetDevice(&dev);
    // one flag bit per ordinal 0..31; other ordinals set the attribute on every launch
    const bool flagged = dev >= 0 && dev < 32;
    const uint32_t bit = flagged ? 1u << dev : 0u;
    if (flagged && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e == cudaSuccess && flagged) done.fetch_or(bit, std::memory_order_release);
    return e;
}

template <int MODE, int DIM, int NSETS, int HB>
static cudaError_t launch_sym_t(const SymArgs& a, int grid, cudaStream_t s)
{
    const size_t sm = sym_smem_bytes<MODE, DIM, NSETS, HB>();
    static std::atomic<uint32_t> attr{0};
    const cudaError_t e = ensure_smem_attr(k_sym<MODE, DIM, NSETS, HB>, sm, attr);
    if (e != cudaSuccess) return e;
    k_sym<MODE, DIM, NSETS, HB><<<grid, 256, sm, s>>>(a);
    return cudaGetLastError();
}

#define FDL_SYM_CASE(M_, D_, S_, H_) \
    if (mode == M_ && dim == D_ && nsets == S_ && hb == H_) return launch_sym_t<M_, D_, S_, H_>(a, grid, s);
#define FDL_SYM_ALLHB(M_, D_, S_) FDL_SYM_CASE(M_, D_, S_, 0) FDL_SYM_CASE(M_, D_, S_, 1) FDL_SYM_CASE(M_, D_, S_, 2)

cudaError_t launch_sym(const SymArgs& a, int mode, int dim, int nsets, int hb, int grid, cudaStream_t s)
{
    FDL_SYM_ALLHB(kSymP1, 2, 1) FDL_SYM_ALLHB(kSymP1, 2, 2) FDL_SYM_ALLHB(kSymP1, 3, 1) FDL_SYM_ALLHB(kSymP1, 3, 2)
    FDL_SYM_ALLHB(kSymP1S, 2, 2) FDL_SYM_ALLHB(kSymP1S, 3, 2)
    FDL_SYM_ALLHB(kSymP1A, 2, 1) FDL_SYM_ALLHB(kSymP1A, 3, 1)
    FDL_SYM_ALLHB(kSymP1R, 2, 1) FDL_SYM_ALLHB(kSymP1R, 3, 1)
    FDL_SYM_CASE(kSymP1, 2, 1, 4) FDL_SYM_CASE(kSymP1, 2, 2, 4) FDL_SYM_CASE(kSymP1, 3, 1, 4)
    FDL_SYM_CASE(kSymP1, 3, 2, 4) FDL_SYM_CASE(kSymP2, 2, 1, 4) FDL_SYM_CASE(kSymP2, 3, 1, 4)
    FDL_SYM_CASE(kSymDiag, 2, 1, 4) FDL_SYM_CASE(kSymDiag, 3, 1, 4)
    FDL_SYM_ALLHB(kSymP2, 2, 1) FDL_SYM_ALLHB(kSymP2, 3, 1)
    FDL_SYM_ALLHB(kSymDiag, 2, 1) FDL_SYM_ALLHB(kSymDiag, 3, 1)
    return cudaErrorInvalidValue;
}

// ------------------------------------------- P1S arithmetic ceiling (diagnostic)
// A pass's per-tile work alone -- sym_tile (the same function k_sym runs: hop
// decode from shared memory, pair arithmetic, j-side stores) on one resident
// 4-bit tile and position block, at k_sym's occupancy -- without the TMA ring,
// HBM, the warp flushes or the reductions: the ceiling the instruction mix
// itself allows (fdl_bench_p1s_mix for the line-6 pass, bench.py; P2 alike).
template <int MODE, int NSETS>
__global__ void __launch_bounds__(256, sym_ctas_per_sm<MODE, 2>()) k_tile_mix(const float* __restrict__ pos,
                                                                              float* out, int iters)
{
    constexpr int C = sym_ncomp<MODE, 2, NSETS>();
    constexpr int PS = sym_ps<MODE, 2, NSETS>();
    constexpr int JP = sym_jpitch<MODE, 2, NSETS>();
    __shared__ __align__(128) uint8_t sD[tile_bytes(0)];
    __shared__ __align__(16) float sP[kT * PS];
    __shared__ float lut[256];
    __shared__ float2 lut2[256];
    __shared__ float red[sym_red_floats<MODE, 2, NSETS>()];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int ty = lane & 15, tx = tid >> 4;
    lut[tid] = tid ? 1.0f / (float)(tid * tid) : 0.0f;
    {
        const int lo = (int)nib_decode_lo((uint32_t)tid), hi = (int)nib_decode_hi((uint32_t)tid);
        lut2[tid] = MODE == kSymP2 ? make_float2(lo ? 1.0f / (float)(lo * lo) : 0.0f, hi ? 1.0f / (float)(hi * hi) : 0.0f)
                                   : make_float2((float)(lo * lo), (float)(hi * hi));
    }
    for (int k = tid; k < kT * PS; k += 256) sP[k] = pos[k % (kT * 4)];
    for (int k = tid; k < (int)tile_bytes(0); k += 256) {  // hops 1..8 (C5's range)
        const uint32_t z = (uint32_t)k * 2654435761u + blockIdx.x * 40503u;
        sD[k] = (uint8_t)nib_encode(1u + ((z >> 7) & 7u), 1u + ((z >> 17) & 7u));
    }
    __syncthreads();
    float xi[8][PS], ai[8][C];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
        for (int q = 0; q < PS; ++q) xi[r][q] = pos[((ty * 8 + r) * PS + q) % (kT * 4)] + 0.37f;
#pragma unroll
        for (int v = 0; v < C; ++v) ai[r][v] = 0.0f;
    }
    float* wrow = red + wid * 2 * (16 * JP + 16) + (tx & 1) * (16 * JP + 16) + ty * JP;
    double s64 = 0.0;
    for (int it = 0; it < iters; ++it) {
        float sf[2][NSETS];
#pragma unroll
        for (int q = 0; q < NSETS; ++q) sf[0][q] = sf[1][q] = 0.0f;
        float jv[8 * C];
        sym_tile<MODE, 2, NSETS, 0, false>(sD, sP, lut, lut2, lut2, 0x4B000000u, -2.0f, ty, tx, false, xi, ai, wrow, sf,
                                           jv);
        if constexpr (sym_shflred<MODE, 2, NSETS, 0>())
            sym_bfly_warp<MODE, 2, NSETS>(jv, red + wid * 2 * (16 * JP + 16), lane);  // the pass stores one float per lane
        else if constexpr (sym_pbfly<MODE, 2, NSETS, 0>())
            red[wid * 2 * (16 * JP + 16) + lane] = jv[0];
        s64 += (double)sf[0][0] + (double)sf[1][NSETS - 1];
        __syncwarp();
    }
    __syncwarp();
    float t = (float)s64 + red[wid * 2 * (16 * JP + 16) + lane];  // keeps the j-side stores
#pragma unroll
    for (int r = 0; r < 8; ++r) t += ai[r][0] + ai[r][C - 1];
    out[blockIdx.x * 256 + tid] = t;
}

cudaError_t launch_tile_mix(int mode, const float* pos, float* out, int iters, int blocks, cudaStream_t s)
{
    if (mode == kSymP1S)
        k_tile_mix<kSymP1S, 2><<<blocks, 256, 0, s>>>(pos, out, iters);
    else if (mode == kSymP2)
        k_tile_mix<kSymP2, 1><<<blocks, 256, 0, s>>>(pos, out, iters);
    else
        return cudaErrorInvalidValue;
    return cudaGetLastError();
}

int tile_mix_ctas_per_sm(int mode) { return mode == kSymP2 ? sym_ctas_per_sm<kSymP2, 2>() : sym_ctas_per_sm<kSymP1S, 2>(); }

// ------------------------------------------------------ enumerating strategy
// Stress of NC relaxed candidates X~(w_c) = X^{k+1} + w_c (X^{k+1} - X^k) in
// one pass over the stored triangle (the exhaustive
// search over the relax factor).  Staged per vertex: {x'(DIM), D(DIM)} with
// x' = X^{k+1}, D = X^{k+1} - X^k (padded to 4 / 8 floats), so per pair
// delta(w) = (x'_i - x'_j) + w (D_i - D_j) exactly as Eq. 10 forms it, and
// s_c += (|delta(w_c)| / h - 1)^2 (Eq. 1, w' d'^2 = 1).  No force outputs:
// only per-item stress partials [item][NC].  MUFU (rsqrt) bound: one per
// candidate per pair.
template <int DIM>
__host__ __device__ constexpr int enum_ps()
{
    return DIM == 2 ? 4 : 8;
}

template <int DIM, int HB>
__host__ __device__ constexpr int enum_stage_bytes()
{
    return (int)tile_bytes(HB) + kT * enum_ps<DIM>() * 4;
}

constexpr int kEnumStages = 3;

template <int DIM, int NC, bool SAFE>
__device__ __forceinline__ void enum_pair(const float* xi, const float* xj, float h2, bool valid, const float* om,
                                          float* sf)
{
    float dp[DIM], dd[DIM];
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        dp[c] = xi[c] - xj[c];
        dd[c] = xi[DIM + c] - xj[DIM + c];
    }
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        float r2 = FLT_MIN;
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            const float d = fmaf(om[k], dd[c], dp[c]);
            r2 = fmaf(d, d, r2);
        }
        const float q = rsqrt_approx(r2 * h2);
        float u = fmaf(r2, q, -1.0f);
        if (SAFE) u = valid ? u : 0.0f;
        sf[k] = fmaf(u, u, sf[k]);
    }
}

template <int DIM, int HB, int NC, bool SAFE>
__device__ __forceinline__ void enum_tile(const uint8_t* sD, const float* sP, const float2* lut2, uint32_t magic,
                                          int ty, int tx, bool diag, const float (&xi)[8][2 * DIM], const float* om,
                                          float* sf)
{
    constexpr int PS = enum_ps<DIM>();
    constexpr int NCH = HB ? 4 * HB : 2;
    constexpr int CPC = HB ? 2 / HB : 4;
    const int tid = tx * 16 + ty;
#pragma unroll 1
    for (int kc = 0; kc < NCH; ++kc) {
        const uint4 ch = *reinterpret_cast<const uint4*>(sD + ((size_t)kc * 256 + tid) * 16);
#pragma unroll
        for (int cc = 0; cc < CPC; ++cc) {
            const int c = kc * CPC + cc;
            const int jl = tx * 8 + c;
            const int js = c * 16 + tx;
            float xj[PS];
#pragma unroll
            for (int q = 0; q < PS / 4; ++q) {
                const float4 t = *reinterpret_cast<const float4*>(sP + js * PS + 4 * q);
                xj[4 * q] = t.x; xj[4 * q + 1] = t.y; xj[4 * q + 2] = t.z; xj[4 * q + 3] = t.w;
            }
            float xjc[2 * DIM];
#pragma unroll
            for (int q = 0; q < DIM; ++q) {
                xjc[q] = xj[q];
                xjc[DIM + q] = xj[(PS / 2) + q];
            }
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                float h2;
                if (HB == 0) {
                    const float2 e = *reinterpret_cast<const float2*>(
                        reinterpret_cast<const char*>(lut2) +
                        ((r >> 1) == 0 ? ((word_of(ch, cc) << 3) & 0x7f8u)
                                       : ((word_of(ch, cc) >> (8 * (r >> 1) - 3)) & 0x7f8u)));
                    h2 = (r & 1) ? e.y : e.x;
                } else {
                    const float hf = chunk_hop<HB>(ch, r, cc, magic);
                    h2 = hf * hf;
                }
                bool valid = true;
                if (SAFE) valid = (h2 > 0.0f) && (!diag || (ty * 8 + r < jl));
                enum_pair<DIM, NC, SAFE>(&xi[r][0], xjc, h2, valid, om, sf);
            }
        }
    }
}

template <int DIM, int HB, int NC>
__global__ void __launch_bounds__(256, 2) k_enum(const SymArgs a, const EnumOmegas w)
{
    constexpr int PS = enum_ps<DIM>();
    constexpr int STAGE = enum_stage_bytes<DIM, HB>();
    constexpr int DT = (int)tile_bytes(HB);
    constexpr int NST = kEnumStages;
    constexpr int NW = 8;
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t full[NST];
    __shared__ int drained[NST];
    __shared__ int prod[2];
    __shared__ double sred[8][NC];
    __shared__ float2 lut2[HB == 0 ? 256 : 1];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int ty = lane & 15, tx = tid >> 4;
    if ((int)blockIdx.x >= a.nitems) return;
    if (HB == 0) {
        const int lo = (int)nib_decode_lo((uint32_t)tid), hi = (int)nib_decode_hi((uint32_t)tid);
        lut2[tid] = make_float2((float)(lo * lo), (float)(hi * hi));
    }
    float om[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) om[k] = w.w[k];
    auto issue = [&](int stage) {
        int p_item = prod[0], p_t = prod[1];
        if (p_item >= a.nitems) return;
        const int4 it = a.items[a.order[p_item]];
        const int J = it.y + p_t;
        const int64_t lt = (int64_t)it.w + p_t;
        uint8_t* base = smem + (size_t)stage * STAGE;
        fence_proxy_async();
        mbar_arrive_expect_tx(&full[stage], STAGE);
        FDL_DCHECK(lt >= 0 && lt < a.ntiles && J >= 0 && (int64_t)(J + 1) * kT <= a.nstage);
        tma_load_1d(base, a.D + lt * DT, DT, &full[stage]);
        tma_load_1d(base + DT, a.pos + (int64_t)J * kT * PS, kT * PS * 4, &full[stage]);
        if (++p_t == it.z) {
            p_t = 0;
            p_item += gridDim.x;
        }
        prod[0] = p_item;
        prod[1] = p_t;
    };
    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], 1);
            drained[s] = 0;
        }
        fence_mbar_init();
        prod[0] = blockIdx.x;
        prod[1] = 0;
        for (int s = 0; s < NST; ++s) issue(s);
    }
    __syncthreads();
    int stage = 0;
    uint32_t phase = 0;
    for (int slot = blockIdx.x; slot < a.nitems; slot += gridDim.x) {
        const int item = a.order[slot];  // outputs are indexed by item: any schedule gives the same sums
        const int4 it = a.items[item];
        const int I = it.x;
        float xi[8][2 * DIM];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int64_t gi = stage_slot((int64_t)I * kT + ty * 8 + r);
#pragma unroll
            for (int q = 0; q < DIM; ++q) {
                xi[r][q] = a.pos[gi * PS + q];
                xi[r][DIM + q] = a.pos[gi * PS + PS / 2 + q];
            }
        }
        double s64[NC];
#pragma unroll
        for (int k = 0; k < NC; ++k) s64[k] = 0.0;
        for (int t = 0; t < it.z; ++t) {
            const int J = it.y + t;
            const bool diag = (J == I);
            const bool safe = diag || (int64_t)(J + 1) * kT > a.n || (int64_t)(I + 1) * kT > a.n;
            mbar_wait(&full[stage], phase);
            const uint8_t* sD = smem + (size_t)stage * STAGE;
            const float* sP = reinterpret_cast<const float*>(sD + DT);
            float sf[NC];
#pragma unroll
            for (int k = 0; k < NC; ++k) sf[k] = 0.0f;
            if (safe)
                enum_tile<DIM, HB, NC, true>(sD, sP, lut2, a.magic, ty, tx, diag, xi, om, sf);
            else
                enum_tile<DIM, HB, NC, false>(sD, sP, lut2, a.magic, ty, tx, diag, xi, om, sf);
#pragma unroll
            for (int k = 0; k < NC; ++k) s64[k] += (double)sf[k];
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                if (atomicAdd(&drained[stage], 1) == NW - 1) {
                    __threadfence_block();
                    drained[stage] = 0;
                    issue(stage);
                }
            }
            if (++stage == NST) {
                stage = 0;
                phase ^= 1u;
            }
        }
#pragma unroll
        for (int k = 0; k < NC; ++k) {
            double v = s64[k];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) sred[wid][k] = v;
        }
        __syncthreads();
        if (tid < NC) {
            double v = 0.0;
            for (int ww = 0; ww < NW; ++ww) v += sred[ww][tid];
            a.spart[(size_t)item * NC + tid] = v;
        }
        __syncthreads();
    }
}

template <int DIM, int HB>
static cudaError_t launch_enum_t(const SymArgs& a, const EnumOmegas& w, int grid, cudaStream_t s)
{
    constexpr size_t sm = (size_t)kEnumStages * enum_stage_bytes<DIM, HB>();
    static std::atomic<uint32_t> attr{0};
    const cudaError_t e = ensure_smem_attr(k_enum<DIM, HB, kEnumNC>, sm, attr);
    if (e != cudaSuccess) return e;
    k_enum<DIM, HB, kEnumNC><<<grid, 256, sm, s>>>(a, w);
    return cudaGetLastError();
}

cudaError_t launch_enum(const SymArgs& a, const EnumOmegas& w, int dim, int hb, int grid, cudaStream_t s)
{
    if (dim == 2) {
        if (hb == 0) return launch_enum_t<2, 0>(a, w, grid, s);
        if (hb == 1) return launch_enum_t<2, 1>(a, w, grid, s);
        return launch_enum_t<2, 2>(a, w, grid, s);
    }
    if (hb == 0) return launch_enum_t<3, 0>(a, w, grid, s);
    if (hb == 1) return launch_enum_t<3, 1>(a, w, grid, s);
    return launch_enum_t<3, 2>(a, w, grid, s);
}

template <int MODE, int DIM, int NSETS, int HB>
static int sym_occ_t()
{
    const size_t sm = sym_smem_bytes<MODE, DIM, NSETS, HB>();
    int n = 0;
    cudaFuncSetAttribute(k_sym<MODE, DIM, NSETS, HB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_sym<MODE, DIM, NSETS, HB>, 256, sm) != cudaSuccess) n = 1;
    return n > 0 ? n : 1;
}

#define FDL_SYM_OCC(M_, D_, S_, H_) \
    if (mode == M_ && dim == D_ && nsets == S_ && hb == H_) return sym_occ_t<M_, D_, S_, H_>();
int sym_max_ctas(int mode, int dim, int nsets, int hb)
{
#define FDL_SYM_OCC3(M_, D_, S_) FDL_SYM_OCC(M_, D_, S_, 0) FDL_SYM_OCC(M_, D_, S_, 1) FDL_SYM_OCC(M_, D_, S_, 2)
    FDL_SYM_OCC3(kSymP1, 2, 1) FDL_SYM_OCC3(kSymP1, 2, 2) FDL_SYM_OCC3(kSymP1, 3, 1) FDL_SYM_OCC3(kSymP1, 3, 2)
    FDL_SYM_OCC3(kSymP1S, 2, 2) FDL_SYM_OCC3(kSymP1S, 3, 2)
    FDL_SYM_OCC3(kSymP1A, 2, 1) FDL_SYM_OCC3(kSymP1A, 3, 1)
    FDL_SYM_OCC3(kSymP1R, 2, 1) FDL_SYM_OCC3(kSymP1R, 3, 1)
    FDL_SYM_OCC(kSymP1, 2, 1, 4) FDL_SYM_OCC(kSymP1, 2, 2, 4) FDL_SYM_OCC(kSymP1, 3, 1, 4)
    FDL_SYM_OCC(kSymP1, 3, 2, 4) FDL_SYM_OCC(kSymP2, 2, 1, 4) FDL_SYM_OCC(kSymP2, 3, 1, 4)
    FDL_SYM_OCC(kSymDiag, 2, 1, 4) FDL_SYM_OCC(kSymDiag, 3, 1, 4)
    FDL_SYM_OCC3(kSymP2, 2, 1) FDL_SYM_OCC3(kSymP2, 3, 1)
    FDL_SYM_OCC3(kSymDiag, 2, 1) FDL_SYM_OCC3(kSymDiag, 3, 1)
    return 1;
}

// ---------------------------------------------------------------- reduction
// Per row of block B: sum, in a fixed order, the j-side tile partials of the
// local tiles (I, B), I = 0..B, and the i-side per-warp partials of strip B
// (items it_lo[B]..it_hi[B], 8 warps each).  8 groups of 128 threads: group g
// takes tiles I = g mod 8 and items it_lo + g mod 8; the group sums are
// combined in group order (fp64).  Blocks run largest B first.
// Output: dense fp64 rank partial, components [0, D) -> out0, [D, C) -> out1.
constexpr int kRedGroups = 8;
#ifndef FDL_RED_UNROLL
#define FDL_RED_UNROLL 4  // j-side tile partials in flight per thread (k_sym_reduce)
#endif
constexpr int kRedUnroll = FDL_RED_UNROLL;

template <int C>
__global__ void __launch_bounds__(kRedGroups * kT) k_sym_reduce(const float* __restrict__ ipart,
                                                                const float* __restrict__ jpart,
                                                                const int* __restrict__ it_lo,
                                                                const int* __restrict__ it_hi, int nb, int64_t t0,
                                                                int64_t t1, int Ilo, int Ihi, int D, int inter,
                                                                double* out0, double* out1)
{
    __shared__ double gsum[kRedGroups][kT][C];
    const int B = nb - 1 - (int)blockIdx.x;
    const int g = threadIdx.x / kT, r = threadIdx.x % kT;
    double acc[C];
#pragma unroll
    for (int v = 0; v < C; ++v) acc[v] = 0.0;
    // only the local row blocks [Ilo, Ihi] (the rank's tile range); group g keeps I = g mod 8
    const int Ifirst = Ilo + ((g - Ilo) % kRedGroups + kRedGroups) % kRedGroups;
    const int Ilast = min(B, Ihi);
#pragma unroll kRedUnroll
    for (int I = Ifirst; I <= Ilast; I += kRedGroups) {
        const int64_t t = tri_index(I, B, nb);
        if (t < t0 || t >= t1) continue;
        const float* src = jpart + ((size_t)(t - t0) * kT + r) * C;
#pragma unroll
        for (int v = 0; v < C; ++v) acc[v] += (double)src[v];
    }
    for (int item = it_lo[B] + g; item < it_hi[B]; item += kRedGroups)
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            const float* src = ipart + (((size_t)item * 8 + w) * kT + r) * C;
#pragma unroll
            for (int v = 0; v < C; ++v) acc[v] += (double)src[v];
        }
#pragma unroll
    for (int v = 0; v < C; ++v) gsum[g][r][v] = acc[v];
    __syncthreads();
    if (g != 0) return;
    double tot[C];
#pragma unroll
    for (int v = 0; v < C; ++v) tot[v] = 0.0;
    for (int gg = 0; gg < kRedGroups; ++gg)
#pragma unroll
        for (int v = 0; v < C; ++v) tot[v] += gsum[gg][r][v];
    const size_t row = (size_t)B * kT + r;
#pragma unroll
    for (int v = 0; v < C; ++v) {
        if (inter)  // two sets interleaved per component: set v&1, component v>>1
            ((v & 1) ? out1 : out0)[row * D + (v >> 1)] = tot[v];
        else if (v < D)
            out0[row * D + v] = tot[v];
        else
            out1[row * (C - D) + (v - D)] = tot[v];
    }
}

cudaError_t launch_sym_reduce(const float* ipart, const float* jpart, const int* it_lo, const int* it_hi, int nb,
                              int64_t t0, int64_t t1, int Ilo, int Ihi, int C, int D, int inter, double* out0,
                              double* out1, cudaStream_t s)
{
#define FDL_RED_CASE(C_)                                                                                        \
    if (C == C_) {                                                                                              \
        k_sym_reduce<C_><<<nb, kRedGroups * kT, 0, s>>>(ipart, jpart, it_lo, it_hi, nb, t0, t1, Ilo, Ihi, D, inter, \
                                                        out0, out1);                                           \
        return cudaGetLastError();                                                                              \
    }
    FDL_RED_CASE(1) FDL_RED_CASE(2) FDL_RED_CASE(3) FDL_RED_CASE(4) FDL_RED_CASE(6)
#undef FDL_RED_CASE
    return cudaErrorInvalidValue;
}

// sum of rank partials in rank order (multi-GPU): parts[world][rows][C]
// Row-slice exchange of several ranks (fdl_api.cu run_sym): out[i] = sum over
// source ranks g = 0..world-1, in rank order, of recv[g][i] (this rank's rows of
// every rank's partial, as the all-to-all delivered them).
__global__ void k_slice_sum(const double* __restrict__ recv, int world, int64_t elems, double* out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= elems) return;
    double s = 0.0;
    for (int g = 0; g < world; ++g) s += recv[(size_t)g * elems + i];
    out[i] = s;
}

cudaError_t launch_slice_sum(const double* recv, int world, int64_t elems, double* out, cudaStream_t s)
{
    k_slice_sum<<<(unsigned)((elems + 255) / 256), 256, 0, s>>>(recv, world, elems, out);
    return cudaGetLastError();
}

// The all-gathered reduced slices ([world][rslice * C + 2]: rows of rank g's slice,
// then its 2 stress partials) -> the dense outputs (components [0, D) -> out0, the
// rest -> out1; inter: components interleaved by position set, out0 = set 0).
__global__ void k_slice_unpack(const double* __restrict__ gath, int64_t rslice, int64_t rows, int C, int D, int inter,
                               double* out0, double* out1)
{
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= rows * C) return;
    const int64_t row = idx / C;
    const int v = (int)(idx % C);
    const int64_t g = row / rslice;
    const double s = gath[(size_t)g * (rslice * C + 2) + (row - g * rslice) * C + v];
    if (inter)
        ((v & 1) ? out1 : out0)[row * D + (v >> 1)] = s;
    else if (v < D)
        out0[row * D + v] = s;
    else
        out1[row * (C - D) + (v - D)] = s;
}

cudaError_t launch_slice_unpack(const double* gath, int world, int64_t rslice, int64_t rows, int C, int D, int inter,
                                double* out0, double* out1, cudaStream_t s)
{
    (void)world;
    const int64_t total = rows * C;
    k_slice_unpack<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(gath, rslice, rows, C, D, inter, out0, out1);
    return cudaGetLastError();
}

// f = sum over ranks (rank order) of the rank stress partials (rank g's pair at
// parts + g * stride); Eq. 1 counts each unordered pair once, as the symmetric
// pass does.
__global__ void k_stress_ranks(const double* __restrict__ parts, int64_t stride, int world, int nsets, DevScalars* sc,
                               int set_cur)
{
    if (threadIdx.x != 0) return;
    for (int s = 0; s < nsets; ++s) {
        double v = 0.0;
        for (int g = 0; g < world; ++g) v += parts[(size_t)g * stride + s];
        sc->f_set[s] = v;
        if (set_cur && s == 0) {
            sc->f_cur = v;
            sc->nonfinite = !isfinite(v);
        }
    }
}

cudaError_t launch_stress_ranks(const double* parts, int64_t stride, int world, int nsets, DevScalars* sc, int set_cur,
                                cudaStream_t s)
{
    k_stress_ranks<<<1, 32, 0, s>>>(parts, stride, world, nsets, sc, set_cur);
    return cudaGetLastError();
}

// sigma = (sum_i diag_i) / n^2, one block, fixed order
__global__ void k_sigma_rows(const double* __restrict__ diag, int n, DevScalars* sc)
{
    __shared__ double red[32];
    double v = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) v += diag[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
        sc->sigma = s / ((double)n * (double)n);
        sc->inv_n = 1.0 / (double)n;
    }
}

cudaError_t launch_set_sigma_rows(const double* diag, int n, DevScalars* sc, cudaStream_t s)
{
    k_sigma_rows<<<1, 1024, 0, s>>>(diag, n, sc);
    return cudaGetLastError();
}

// Dense hop rows (uint16) gathered from the triangle tiles: out[r][j] = hop(rows[r], j);
// entries whose tile is not local set *missing.
__global__ void k_hop_rows(const uint8_t* __restrict__ D, int hb, int nb, int64_t t0, int64_t t1,
                           const int* __restrict__ rows, int nrows, int n, uint16_t* out, int* missing)
{
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)nrows * n) return;
    const int r = (int)(idx / n), j = (int)(idx % n);
    int a = rows[r], b = j;
    if (a / kT > b / kT) {
        const int tmp = a;
        a = b;
        b = tmp;
    }
    const int64_t t = tri_index(a / kT, b / kT, nb);
    if (t < t0 || t >= t1) {
        *missing = 1;
        out[idx] = 0;
        return;
    }
    const size_t off = sym_offset(t - t0, a % kT, b % kT, hb);
    if (hb == 0)
        out[idx] = (uint16_t)((a & 1) ? nib_decode_hi(D[off]) : nib_decode_lo(D[off]));
    else
        out[idx] = hb == 1 ? D[off] : (uint16_t)(D[off] | (D[off + 1] << 8));
}

cudaError_t launch_hop_rows(const uint8_t* D, int hb, int nb, int64_t t0, int64_t t1, const int* rows, int nrows,
                            int n, uint16_t* out, int* missing, cudaStream_t s)
{
    const int64_t total = (int64_t)nrows * n;
    k_hop_rows<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(D, hb, nb, t0, t1, rows, nrows, n, out, missing);
    return cudaGetLastError();
}

// stress partial of the rank: fixed-order two-stage reduction of the
// [item(x warp)][nsets] partials -- stage 1: block b sums the fixed chunk
// [b*kStressChunk, (b+1)*kStressChunk) (thread stride, warp butterfly, warps in
// order); stage 2: one block sums the chunk sums in the same pattern.
constexpr int kStressChunk = 8192;

__device__ __forceinline__ double block_sum_1024(double v, double* red)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    __syncthreads();
    return t;
}

__global__ void __launch_bounds__(1024) k_sym_stress1(const double* __restrict__ spart, int nitems, int nsets,
                                                      double* chunk_sums)
{
    __shared__ double red[32];
    const int b = blockIdx.x;
    const int lo = b * kStressChunk, hi = min(nitems, lo + kStressChunk);
    for (int s = 0; s < nsets; ++s) {
        double v = 0.0;
        for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) v += spart[(size_t)i * nsets + s];
        const double t = block_sum_1024(v, red);
        if (threadIdx.x == 0) chunk_sums[(size_t)b * nsets + s] = t;
    }
}

__global__ void __launch_bounds__(1024) k_sym_stress2(const double* __restrict__ chunk_sums, int nchunks, int nsets,
                                                      double* out)
{
    __shared__ double red[32];
    for (int s = 0; s < nsets; ++s) {
        double v = 0.0;
        for (int i = threadIdx.x; i < nchunks; i += blockDim.x) v += chunk_sums[(size_t)i * nsets + s];
        const double t = block_sum_1024(v, red);
        if (threadIdx.x == 0) out[s] = t;
    }
}

int sym_stress_chunks(int nitems) { return std::max(1, (nitems + kStressChunk - 1) / kStressChunk); }

cudaError_t launch_sym_stress(const double* spart, int nitems, int nsets, double* out, double* scratch,
                              cudaStream_t s)
{
    const int nc = sym_stress_chunks(nitems);
    k_sym_stress1<<<nc, 1024, 0, s>>>(spart, nitems, nsets, scratch);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_sym_stress2<<<1, 1024, 0, s>>>(scratch, nc, nsets, out);
    return cudaGetLastError();
}

// MS-BFS level: vertex v ORs its neighbours' 1024-source frontier words
// (warp per vertex, lane = 32 sources, coalesced neighbour reads), keeps the
// new bits, and records their level in the batch buffer bbuf[v][source] (cells
// of the stored width, each lane's 32 cells contiguous: one vector
// read-modify-write per lane and level).  k_bfs_retile then moves the batch's
// rows into the triangle tiles with coalesced 16-byte chunk stores.
// Bit k of the low bits of x moved to the lowest bit of cell k (cells of 4, 8 or 16
// bits); times the level, each cell of a set bit holds the level (no carries: the
// level fits the cell).
__device__ __forceinline__ uint32_t spread_nib(uint32_t x)  // 8 bits -> 8 nibbles
{
    x &= 0xffu;
    x = (x | (x << 12)) & 0x000F000Fu;
    x = (x | (x << 6)) & 0x03030303u;
    return (x | (x << 3)) & 0x11111111u;
}
__device__ __forceinline__ uint32_t spread_byte(uint32_t x)  // 4 bits -> 4 bytes
{
    x &= 0xfu;
    x = (x | (x << 14)) & 0x00030003u;
    return (x | (x << 7)) & 0x01010101u;
}

template <int HB>
__device__ __forceinline__ void bfs_record(uint8_t* cells, uint32_t nw, int level)
{
    const uint32_t L = (uint32_t)level;
    if (HB == 0) {  // 32 nibbles = 16 bytes
        uint4 c = *reinterpret_cast<uint4*>(cells);
        c.x |= spread_nib(nw) * L;
        c.y |= spread_nib(nw >> 8) * L;
        c.z |= spread_nib(nw >> 16) * L;
        c.w |= spread_nib(nw >> 24) * L;
        *reinterpret_cast<uint4*>(cells) = c;
    } else if (HB == 1) {  // 32 bytes
        uint4* p = reinterpret_cast<uint4*>(cells);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint4 c = p[h];
            c.x |= spread_byte(nw >> (16 * h)) * L;
            c.y |= spread_byte(nw >> (16 * h + 4)) * L;
            c.z |= spread_byte(nw >> (16 * h + 8)) * L;
            c.w |= spread_byte(nw >> (16 * h + 12)) * L;
            p[h] = c;
        }
    } else {  // 32 x uint16 = 64 bytes
        uint4* p = reinterpret_cast<uint4*>(cells);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            uint4 c = p[h];
            uint32_t w[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t b = nw >> (8 * h + 2 * q);
                w[q] |= ((b & 1u) | ((b & 2u) << 15)) * L;
            }
            p[h] = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
}

template <int HB>
__host__ __device__ constexpr int bfs_row_bytes()  // batch-buffer bytes per vertex (1024 sources)
{
    return HB == 0 ? 512 : 1024 * HB;
}

// One level of the batch's BFS, with no host round trip: flags[L] = 1 when
// level L found a new (vertex, source) pair, and a level whose predecessor
// found none returns at once (the batch's search is over; diam <= 2 ecc(0)
// bounds how many levels the host enqueues).  Grid-stride over vertices (warp
// per vertex), so a finished level costs one short launch.  Gather bytes of
// the level (neighbour frontier words + visited read + new-frontier write,
// 128 B each per vertex searched) are added to *bytes (MS-BFS roofline).
template <int HB>
__device__ __forceinline__ uint32_t bfs_gather(const int32_t* __restrict__ col, const uint32_t* __restrict__ fin,
                                               int64_t beg, int64_t end, int64_t stride, int lane)
{
    // OR of the neighbours' frontier words over col[beg, end) in chunks of 32 neighbours
    // `stride` apart; kBfsUnroll independent 128-byte loads in flight per warp
    uint32_t acc = 0;
    const uint32_t* fl = fin + lane;
    for (int64_t e0 = beg; e0 < end; e0 += stride) {
        const int myu = (e0 + lane < end) ? col[e0 + lane] : 0;
        const int cnt = (int)min((int64_t)32, end - e0);  // warp-uniform
        if (cnt <= 8) {  // the usual degree: 8 slots instead of kBfsUnroll predicated ones
            uint32_t t[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t u = (uint32_t)__shfl_sync(0xffffffffu, myu, k);
                t[k] = k < cnt ? __ldcg(fl + (size_t)u * kBFSWords) : 0u;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) acc |= t[k];
            continue;
        }
        for (int k0 = 0; k0 < cnt; k0 += kBfsUnroll) {
            uint32_t t[kBfsUnroll];
#pragma unroll
            for (int k = 0; k < kBfsUnroll; ++k) {
                const uint32_t u = (uint32_t)__shfl_sync(0xffffffffu, myu, (k0 + k) & 31);
                t[k] = (k0 + k < cnt) ? __ldcg(fl + (size_t)u * kBFSWords) : 0u;
            }
#pragma unroll
            for (int k = 0; k < kBfsUnroll; ++k) acc |= t[k];
        }
    }
    return acc;
}

// One level of the batch's BFS, with no host round trip: flags[L] = 1 when
// level L found a new (vertex, source) pair, and a level whose predecessor
// found none returns at once (the batch's search is over; diam <= 2 ecc(0)
// bounds how many levels the host enqueues).  Blocks [0, nhub) take one hub
// (degree > kBfsHubDeg) each, its neighbour list split over the 8 warps (a
// scale-free graph's hubs would otherwise be one warp's chain of deg / unroll
// L2 round trips per level); the other blocks stride over the remaining
// vertices, warp per vertex.  Gather bytes of the level (neighbour frontier
// words + visited read + new-frontier write, 128 B each per vertex searched)
// are added to *bytes (MS-BFS roofline).
template <int HB>
__global__ void __launch_bounds__(256) k_bfs_level_sym(const int64_t* __restrict__ row_ptr,
                                                       const int32_t* __restrict__ col,
                                                       const uint32_t* __restrict__ fin, uint32_t* __restrict__ fout,
                                                       uint32_t* __restrict__ visited, uint8_t* __restrict__ bbuf,
                                                       int n, int nsrc, int level, unsigned int* flags,
                                                       unsigned long long* bytes, const int* __restrict__ hubs,
                                                       int nhub)
{
    if (level > 1 && *(volatile unsigned int*)&flags[level - 1] == 0u) return;  // uniform over the grid
    __shared__ unsigned long long blk_bytes;
    __shared__ unsigned int blk_new;
    __shared__ uint32_t hub_acc[32];
    __shared__ int hub_skip;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        blk_bytes = 0ull;
        blk_new = 0u;
    }
    const int nl = min(max(nsrc - 32 * lane, 0), 32);
    const uint32_t full = nl == 32 ? 0xffffffffu : ((1u << nl) - 1u);
    if ((int)blockIdx.x < nhub) {
        const int v = hubs[blockIdx.x];
        if (wid == 0) {
            const uint32_t vis = visited[(int64_t)v * kBFSWords + lane];
            const bool done = __all_sync(0xffffffffu, (vis & full) == full);
            hub_acc[lane] = 0u;
            if (lane == 0) hub_skip = done ? 1 : 0;
        }
        __syncthreads();
        const int64_t beg = row_ptr[v], end = row_ptr[v + 1];
        if (!hub_skip) {
            const uint32_t acc = bfs_gather<HB>(col, fin, beg + 32 * wid, end, 256, lane);
            if (acc) atomicOr(&hub_acc[lane], acc);
        }
        __syncthreads();
        if (wid == 0) {
            const uint32_t vis = visited[(int64_t)v * kBFSWords + lane];
            if (hub_skip) {
                fout[(int64_t)v * kBFSWords + lane] = 0u;
            } else {
                const uint32_t nw = hub_acc[lane] & ~vis & full;
                fout[(int64_t)v * kBFSWords + lane] = nw;
                if (nw) {
                    visited[(int64_t)v * kBFSWords + lane] = vis | nw;
                    bfs_record<HB>(bbuf + (int64_t)v * bfs_row_bytes<HB>() + lane * (bfs_row_bytes<HB>() / 32), nw,
                                   level);
                }
                if (__any_sync(0xffffffffu, nw != 0u) && lane == 0) flags[level] = 1u;
                if (lane == 0) atomicAdd(bytes, (unsigned long long)(end - beg + 2) * 128ull);
            }
        }
        return;
    }
    __syncthreads();
    const int64_t nwarps = (int64_t)(gridDim.x - nhub) * (blockDim.x >> 5);
    unsigned long long my_bytes = 0ull;
    bool found = false;
    for (int64_t vv = ((int64_t)(blockIdx.x - nhub) * blockDim.x + threadIdx.x) >> 5; vv < n; vv += nwarps) {
        const int v = (int)vv;
        const int64_t beg = row_ptr[v], end = row_ptr[v + 1];
        if (nhub > 0 && end - beg > kBfsHubDeg) continue;  // a hub block's vertex
        const uint32_t vis = visited[(int64_t)v * kBFSWords + lane];
        if (__all_sync(0xffffffffu, (vis & full) == full)) {
            fout[(int64_t)v * kBFSWords + lane] = 0u;
            continue;
        }
        const uint32_t acc = bfs_gather<HB>(col, fin, beg, end, 32, lane);
        my_bytes += (unsigned long long)(end - beg + 2) * 128ull;
        const uint32_t nw = acc & ~vis & full;
        fout[(int64_t)v * kBFSWords + lane] = nw;
        if (nw) {
            visited[(int64_t)v * kBFSWords + lane] = vis | nw;
            bfs_record<HB>(bbuf + (int64_t)v * bfs_row_bytes<HB>() + lane * (bfs_row_bytes<HB>() / 32), nw, level);
        }
        found |= __any_sync(0xffffffffu, nw != 0u);
    }
    if (lane == 0) {
        if (my_bytes) atomicAdd(&blk_bytes, my_bytes);
        if (found) blk_new = 1u;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (blk_bytes) atomicAdd(bytes, blk_bytes);
        if (blk_new) flags[level] = 1u;
    }
}

// After a batch's levels: the deepest level that found a vertex (running max
// over batches = the diameter) and whether level maxhop + 1 found one (the
// stored width cannot hold the hops: the host retries one width wider).
__global__ void k_bfs_batch_end(const unsigned int* flags, int nlevels, int maxhop, int* diam, int* overflow)
{
    int d = 0;
    for (int L = 1; L <= nlevels; ++L)
        if (flags[L]) d = L;
    if (d > maxhop) {
        *overflow = 1;
        d = maxhop;
    }
    if (d > *diam) *diam = d;
}

// Batch rows [s0, s0 + 1024) into the local triangle tiles: CTA per tile (I, J)
// of the batch's row blocks; thread (ty, tx) gathers the 8 x 8 cells of its
// sub-block (rows = batch sources, columns = vertices) from bbuf (8 or 16 bytes
// per column, contiguous) and stores its 16-byte chunks.
template <int HB>
__global__ void __launch_bounds__(256) k_bfs_retile(const uint8_t* __restrict__ bbuf, uint8_t* __restrict__ D, int n,
                                                    int s0, int nb, int64_t t0, int64_t t1, int I0, int nI)
{
    const int tid = threadIdx.x, ty = tid & 15, tx = tid >> 4;
    // tile index within the batch: row block I = I0 + bI, J = I .. nb-1
    int64_t q = blockIdx.x;
    int bI = 0;
    while (bI < nI && q >= nb - (I0 + bI)) {
        q -= nb - (I0 + bI);
        ++bI;
    }
    if (bI >= nI) return;
    const int I = I0 + bI, J = I + (int)q;
    const int64_t t = tri_index(I, J, nb);
    if (t < t0 || t >= t1) return;
    const int k0 = I * kT + ty * 8 - s0;  // first batch source (row) of the sub-block
    uint8_t* tile = D + (size_t)(t - t0) * (size_t)tile_bytes(HB);
    constexpr int RB = bfs_row_bytes<HB>();
    if (HB == 0) {
#pragma unroll
        for (int kc = 0; kc < 2; ++kc) {
            uint32_t w[4];
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                const int v = J * kT + tx * 8 + kc * 4 + cc;
                w[cc] = v < n ? *reinterpret_cast<const uint32_t*>(bbuf + (int64_t)v * RB + k0 / 2) : 0u;
            }
            *reinterpret_cast<uint4*>(tile + ((size_t)kc * 256 + tid) * 16) = make_uint4(w[0], w[1], w[2], w[3]);
        }
    } else if (HB == 1) {
#pragma unroll
        for (int kc = 0; kc < 4; ++kc) {
            uint2 a = make_uint2(0u, 0u), b = make_uint2(0u, 0u);
            const int v0 = J * kT + tx * 8 + kc * 2;
            if (v0 < n) a = *reinterpret_cast<const uint2*>(bbuf + (int64_t)v0 * RB + k0);
            if (v0 + 1 < n) b = *reinterpret_cast<const uint2*>(bbuf + (int64_t)(v0 + 1) * RB + k0);
            *reinterpret_cast<uint4*>(tile + ((size_t)kc * 256 + tid) * 16) = make_uint4(a.x, a.y, b.x, b.y);
        }
    } else {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int v = J * kT + tx * 8 + c;
            uint4 a = make_uint4(0u, 0u, 0u, 0u);
            if (v < n) a = *reinterpret_cast<const uint4*>(bbuf + (int64_t)v * RB + 2 * k0);
            *reinterpret_cast<uint4*>(tile + ((size_t)c * 256 + tid) * 16) = a;
        }
    }
}

// Blocks of `threads` threads of `kernel` resident on the whole device at once: the
// grid of a grid-stride kernel, so it runs as one wave (a partial second wave leaves SMs
// idle at the tail of every launch: C5 MS-BFS 238 -> 156 ms, C4 405 -> 225 ms)
static int resident_blocks(const void* kernel, int threads)
{
    int dev = 0, sms = 0, per_sm = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0) != cudaSuccess) {
        cudaGetLastError();
        return 1 << 20;  // unknown: no cap
    }
    return std::max(1, per_sm * sms);
}

cudaError_t launch_bfs_level_sym(const int64_t* row_ptr, const int32_t* col, const uint32_t* fin, uint32_t* fout,
                                 uint32_t* visited, uint8_t* bbuf, int n, int nsrc, int level, int hb,
                                 unsigned int* flags, unsigned long long* bytes, const int* hubs, int nhub, int grid,
                                 cudaStream_t s)
{
    static int resident[3] = {0, 0, 0};  // per width (the instantiations' occupancy may differ)
    if (!resident[hb])
        resident[hb] = resident_blocks(hb == 0 ? (const void*)k_bfs_level_sym<0>
                                               : (hb == 1 ? (const void*)k_bfs_level_sym<1> : (const void*)k_bfs_level_sym<2>),
                                       256);
    // hub blocks come first; the grid-stride blocks fill the rest of one wave
    const int cap = std::max(resident[hb] - nhub, resident[hb] / 2);
    const unsigned g =
        (unsigned)nhub + (unsigned)std::max(1, std::min({grid, cap, (int)(((int64_t)n * 32 + 255) / 256)}));
    if (hb == 0)
        k_bfs_level_sym<0><<<g, 256, 0, s>>>(row_ptr, col, fin, fout, visited, bbuf, n, nsrc, level, flags, bytes,
                                             hubs, nhub);
    else if (hb == 1)
        k_bfs_level_sym<1><<<g, 256, 0, s>>>(row_ptr, col, fin, fout, visited, bbuf, n, nsrc, level, flags, bytes,
                                             hubs, nhub);
    else
        k_bfs_level_sym<2><<<g, 256, 0, s>>>(row_ptr, col, fin, fout, visited, bbuf, n, nsrc, level, flags, bytes,
                                             hubs, nhub);
    return cudaGetLastError();
}

// Clustered batches (high-diameter graphs): the batch's sources are an arbitrary list
// srcs[0..nsrc) (a compact graph neighbourhood, so the wavefronts travel together); frontier /
// visited bit of slot k at vertex srcs[k] (nw words per vertex), frontier flags set.
__global__ void k_bfs_init_list(uint32_t* frontier, uint32_t* visited, uint8_t* fl, const int* __restrict__ srcs,
                                int nsrc, int nw)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nsrc) return;
    const int v = srcs[k];
    frontier[(int64_t)v * nw + (k >> 5)] = 1u << (k & 31);  // one source per vertex: no conflict
    visited[(int64_t)v * nw + (k >> 5)] = 1u << (k & 31);
    fl[v] = 1;
}

cudaError_t launch_bfs_init_list(uint32_t* frontier, uint32_t* visited, uint8_t* fl, const int* srcs, int nsrc,
                                 int nw, cudaStream_t s)
{
    k_bfs_init_list<<<(nsrc + 255) / 256, 256, 0, s>>>(frontier, visited, fl, srcs, nsrc, nw);
    return cudaGetLastError();
}

// One level of a clustered batch of up to kBfsWideWords x 32 = 4096 sources: lane holds
// source words lane + 32 j (j < 4).  Four times the sources of k_bfs_level_sym per
// level pass: a compact batch's search needs about as many levels as a 1024-source one
// (the graph's eccentricity), so a quarter of the batches means a quarter of the levels,
// each of which costs a pass over every vertex's frontier flags.  Frontier flags, the
// all-visited skip, device level flags and the gather-byte count as k_bfs_level_sym.
template <int HB>
__global__ void __launch_bounds__(256) k_bfs_level_wide(const int64_t* __restrict__ row_ptr,
                                                        const int32_t* __restrict__ col,
                                                        const uint32_t* __restrict__ fin, uint32_t* __restrict__ fout,
                                                        uint32_t* __restrict__ visited, uint8_t* __restrict__ bbuf,
                                                        int n, int nsrc, int level, unsigned int* flags,
                                                        unsigned long long* bytes, const uint8_t* __restrict__ fl_in,
                                                        uint8_t* __restrict__ fl_out)
{
    constexpr int NW = kBfsWideWords;
    constexpr int J = NW / 32;
    constexpr int CB = bfs_row_bytes<HB>() / 32;  // cell bytes of one source word (32 sources)
    if (level > 1 && *(volatile unsigned int*)&flags[level - 1] == 0u) return;
    __shared__ unsigned long long blk_bytes;
    __shared__ unsigned int blk_new;
    if (threadIdx.x == 0) {
        blk_bytes = 0ull;
        blk_new = 0u;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    uint32_t full[J];
#pragma unroll
    for (int j = 0; j < J; ++j) {
        const int nl = min(max(nsrc - 32 * (32 * j + lane), 0), 32);
        full[j] = nl == 32 ? 0xffffffffu : ((1u << nl) - 1u);
    }
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    unsigned long long my_bytes = 0ull;
    bool found = false;
    for (int64_t vv = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; vv < n; vv += nwarps) {
        const int v = (int)vv;
        const int64_t beg = row_ptr[v], end = row_ptr[v + 1];
        bool nf = false;
        for (int64_t e = beg + lane; e < end && !nf; e += 32) nf = fl_in[col[e]] != 0;
        if (!__any_sync(0xffffffffu, nf)) {
            if (lane == 0) fl_out[v] = 0;
            continue;
        }
        uint32_t vis[J];
        bool done = true;
#pragma unroll
        for (int j = 0; j < J; ++j) {
            vis[j] = visited[(int64_t)v * NW + 32 * j + lane];
            done &= (vis[j] & full[j]) == full[j];
        }
        if (__all_sync(0xffffffffu, done)) {
            if (lane == 0) fl_out[v] = 0;
            continue;
        }
        uint32_t acc[J];
#pragma unroll
        for (int j = 0; j < J; ++j) acc[j] = 0u;
        for (int64_t e0 = beg; e0 < end; e0 += 32) {
            const int myu = (e0 + lane < end) ? col[e0 + lane] : 0;
            const int cnt = (int)min((int64_t)32, end - e0);
            for (int k0 = 0; k0 < cnt; k0 += 4) {
                uint32_t t[4][J];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int u = __shfl_sync(0xffffffffu, myu, (k0 + k) & 31);
                    const bool ok = k0 + k < cnt && fl_in[u];
#pragma unroll
                    for (int j = 0; j < J; ++j) t[k][j] = ok ? __ldcg(&fin[(int64_t)u * NW + 32 * j + lane]) : 0u;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k)
#pragma unroll
                    for (int j = 0; j < J; ++j) acc[j] |= t[k][j];
            }
        }
        my_bytes += (unsigned long long)(end - beg + 2) * (128ull * J);
        bool anyw = false;
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const uint32_t nw = acc[j] & ~vis[j] & full[j];
            fout[(int64_t)v * NW + 32 * j + lane] = nw;
            if (nw) {
                visited[(int64_t)v * NW + 32 * j + lane] = vis[j] | nw;
                bfs_record<HB>(bbuf + ((int64_t)v * NW + 32 * j + lane) * CB, nw, level);
                anyw = true;
            }
        }
        const bool anyn = __any_sync(0xffffffffu, anyw);
        if (lane == 0) fl_out[v] = anyn ? 1 : 0;
        found |= anyn;
    }
    if (lane == 0) {
        if (my_bytes) atomicAdd(&blk_bytes, my_bytes);
        if (found) blk_new = 1u;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (blk_bytes) atomicAdd(bytes, blk_bytes);
        if (blk_new) flags[level] = 1u;
    }
}

cudaError_t launch_bfs_level_wide(const int64_t* row_ptr, const int32_t* col, const uint32_t* fin, uint32_t* fout,
                                  uint32_t* visited, uint8_t* bbuf, int n, int nsrc, int level, int hb,
                                  unsigned int* flags, unsigned long long* bytes, int grid, const uint8_t* fl_in,
                                  uint8_t* fl_out, cudaStream_t s)
{
    static int resident[3] = {0, 0, 0};
    if (!resident[hb])
        resident[hb] = resident_blocks(hb == 0 ? (const void*)k_bfs_level_wide<0>
                                               : (hb == 1 ? (const void*)k_bfs_level_wide<1> : (const void*)k_bfs_level_wide<2>),
                                       256);
    const unsigned g = (unsigned)std::max(1, std::min({grid, resident[hb], (int)(((int64_t)n * 32 + 255) / 256)}));
    if (hb == 0)
        k_bfs_level_wide<0><<<g, 256, 0, s>>>(row_ptr, col, fin, fout, visited, bbuf, n, nsrc, level, flags, bytes,
                                              fl_in, fl_out);
    else if (hb == 1)
        k_bfs_level_wide<1><<<g, 256, 0, s>>>(row_ptr, col, fin, fout, visited, bbuf, n, nsrc, level, flags, bytes,
                                              fl_in, fl_out);
    else
        k_bfs_level_wide<2><<<g, 256, 0, s>>>(row_ptr, col, fin, fout, visited, bbuf, n, nsrc, level, flags, bytes,
                                              fl_in, fl_out);
    return cudaGetLastError();
}

// Clustered batches: hop(srcs[k], v) from the batch buffer (rb bytes per vertex: the
// cells of slot k at k/2 (4-bit), k (8-bit), 2k (16-bit)) into the local upper-triangle
// tiles, one thread per (v, k) (k fastest: coalesced bbuf reads), scattered stores; 4-bit
// cells share a byte between rows 2p and 2p+1 (possibly of other batches): atomicOr of
// the nibble into its zero-initialised word (raw layout, nib_encode runs after all batches).
template <int HB>
__global__ void k_bfs_scatter(const uint8_t* __restrict__ bbuf, uint8_t* D, const int* __restrict__ srcs, int nsrc,
                              int n, int nb, int64_t t0, int64_t t1, int64_t rb)
{
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)n * nsrc) return;
    const int v = (int)(idx / nsrc), k = (int)(idx % nsrc);
    const int src = srcs[k];
    const int I = src / kT, J = v / kT;
    if (I > J) return;
    const int64_t t = tri_index(I, J, nb);
    if (t < t0 || t >= t1) return;
    const uint8_t* cells = bbuf + (int64_t)v * rb;
    uint32_t h;
    if (HB == 0)
        h = (cells[k >> 1] >> (4 * (k & 1))) & 15u;
    else if (HB == 1)
        h = cells[k];
    else
        h = reinterpret_cast<const uint16_t*>(cells)[k];
    if (!h) return;  // the diagonal (src == v); the tiles are zeroed
    const int rl = src % kT, cl = v % kT;
    const size_t off = sym_offset(t - t0, rl, cl, HB);
    FDL_DCHECK(off < (size_t)(t1 - t0) * tile_bytes(HB) && k < nsrc && v < n);
    if (HB == 0) {
        const size_t w = off & ~(size_t)3;
        atomicOr(reinterpret_cast<unsigned int*>(D + w), h << (8 * (off & 3) + 4 * (rl & 1)));
    } else if (HB == 1) {
        D[off] = (uint8_t)h;
    } else {
        *reinterpret_cast<uint16_t*>(D + off) = (uint16_t)h;
    }
}

cudaError_t launch_bfs_scatter(const uint8_t* bbuf, uint8_t* D, const int* srcs, int nsrc, int n, int nb, int64_t t0,
                               int64_t t1, int hb, int64_t rb, cudaStream_t s)
{
    const int64_t total = (int64_t)n * nsrc;
    const unsigned g = (unsigned)((total + 255) / 256);
    if (hb == 0)
        k_bfs_scatter<0><<<g, 256, 0, s>>>(bbuf, D, srcs, nsrc, n, nb, t0, t1, rb);
    else if (hb == 1)
        k_bfs_scatter<1><<<g, 256, 0, s>>>(bbuf, D, srcs, nsrc, n, nb, t0, t1, rb);
    else
        k_bfs_scatter<2><<<g, 256, 0, s>>>(bbuf, D, srcs, nsrc, n, nb, t0, t1, rb);
    return cudaGetLastError();
}

cudaError_t launch_bfs_batch_end(const unsigned int* flags, int nlevels, int maxhop, int* diam, int* overflow,
                                 cudaStream_t s)
{
    k_bfs_batch_end<<<1, 1, 0, s>>>(flags, nlevels, maxhop, diam, overflow);
    return cudaGetLastError();
}

cudaError_t launch_bfs_retile(const uint8_t* bbuf, uint8_t* D, int n, int s0, int nsrc, int nb, int64_t t0,
                              int64_t t1, int hb, cudaStream_t s)
{
    const int I0 = s0 / kT, nI = (nsrc + kT - 1) / kT;
    int64_t ntile = 0;
    for (int b = 0; b < nI; ++b) ntile += nb - (I0 + b);
    if (ntile <= 0) return cudaSuccess;
    if (hb == 0)
        k_bfs_retile<0><<<(unsigned)ntile, 256, 0, s>>>(bbuf, D, n, s0, nb, t0, t1, I0, nI);
    else if (hb == 1)
        k_bfs_retile<1><<<(unsigned)ntile, 256, 0, s>>>(bbuf, D, n, s0, nb, t0, t1, I0, nI);
    else
        k_bfs_retile<2><<<(unsigned)ntile, 256, 0, s>>>(bbuf, D, n, s0, nb, t0, t1, I0, nI);
    return cudaGetLastError();
}

int bfs_row_bytes_host(int hb) { return hb == 0 ? bfs_row_bytes<0>() : (hb == 1 ? bfs_row_bytes<1>() : bfs_row_bytes<2>()); }

// ------------------------------------------------ weighted APSP (NEXT-3 setup)
// Multi-source Bellman-Ford in fp64: dist[v * S + s] = shortest path length
// from source s0 + s to v.  Pull relaxation, warp per vertex, lanes over the
// sources; iterated until no value changes.  Each stored value is the fp64
// sum along a shortest path, so the result does not depend on the iteration
// order; the tiles get its correctly rounded fp32 value.
__global__ void k_bf_init(double* dist, int n, const int* __restrict__ srcs, int nsrc, int S)
{
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)n * S) return;
    const int v = (int)(idx / S), k = (int)(idx % S);
    dist[idx] = (k < nsrc && v == srcs[k]) ? 0.0 : INFINITY;
}

cudaError_t launch_bf_init(double* dist, int n, const int* srcs, int nsrc, int S, cudaStream_t s)
{
    const int64_t total = (int64_t)n * S;
    k_bf_init<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(dist, n, srcs, nsrc, S);
    return cudaGetLastError();
}

// Work-efficient sweep: per (vertex, source) change bits instead of a per-vertex
// stamp.  chg_in[u] holds S bits (W = S/32 words): which of u's distances
// improved in the previous sweep.  Vertex v ORs its neighbours' words (like the
// MS-BFS gather) and re-relaxes only the sources whose bit is set somewhere in
// its neighbourhood: dist[v][k] = min(dist[v][k], dist[u][k] + len(u, v)).
// In place (Gauss-Seidel order); a value read before its neighbour improved in
// the same sweep is re-checked in the next one, so the fixed point is the
// shortest-path distance (each value an fp64 sum along a shortest path).  A
// sweep whose predecessor changed nothing returns at once (flags[it - 1] = 0).
__global__ void __launch_bounds__(256, 4) k_bf_sweep(const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                                  const double* __restrict__ len, double* dist,
                                                  const uint32_t* __restrict__ chg_in, uint32_t* __restrict__ chg_out,
                                                  const uint16_t* __restrict__ pend_in, uint16_t* __restrict__ pend_out,
                                                  int n, int S, int nsrc, int it, double delta, unsigned int* flags)
{
    if (it > 0 && *(volatile unsigned int*)&flags[it - 1] == 0u) return;
    __shared__ uint32_t outw[8 * 32 * kBfWordsPerLane];  // per warp: the vertex's new change words
    const int lane = threadIdx.x & 31;
    const int W = S >> 5;
    const double T = delta * (double)(it + 1);  // this sweep's threshold (Delta-stepping buckets)
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    bool found = false;
    // weak L2 loads (ld.global.cg): a value another warp improves during this sweep may be
    // read stale, and is then re-relaxed in the next sweep through the change bits, as
    // with any Gauss-Seidel order (volatile's system-scope loads were slower)
    double* dv = dist;
    for (int64_t vv = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; vv < n; vv += nwarps) {
        const int v = (int)vv;
        const int64_t beg = row_ptr[v], end = row_ptr[v + 1];
        const int nu = (int)min((int64_t)32, end - beg);
        const int myu = lane < nu ? col[beg + lane] : 0;
        // pending chunks (bit c: some source of chunk c changed at that vertex in the last
        // sweep).  A vertex with nothing pending in its neighbourhood (the usual case away
        // from the wavefront band) costs its neighbours' 2-byte masks only
        const uint32_t smask = pend_in[v];
        const uint32_t lmask = lane < nu ? pend_in[myu] : 0u;
        uint32_t xmask = 0u;  // neighbours past the first 32 (rare)
        for (int64_t e = beg + 32 + lane; e < end; e += 32) xmask |= pend_in[col[e]];
        const uint32_t cmask = __reduce_or_sync(0xffffffffu, lmask | xmask) | smask;
        if (!cmask) {
            if (lane == 0) pend_out[v] = 0;
            continue;
        }
        uint32_t outmask = 0u;
        for (uint32_t cm = cmask; cm; cm &= cm - 1) {
            const int ch = __ffs(cm) - 1;  // chunk: sources [4096 ch, 4096 ch + 4096), words [128 ch, ...)
            const unsigned pm = __ballot_sync(0xffffffffu, (lmask >> ch) & 1u);
            const bool selfp = (smask >> ch) & 1u;
            const int wofs = ch * 32 * kBfWordsPerLane, WC = min(W - wofs, 32 * kBfWordsPerLane);
            // candidate sources: pending bits of the neighbours that have any; lane holds words
            // lane, lane + 32, ... of the W = S/32 source words (S <= 4096: up to 4 per lane)
            uint32_t act[kBfWordsPerLane], own[kBfWordsPerLane];
#pragma unroll
            for (int j = 0; j < kBfWordsPerLane; ++j) act[j] = own[j] = 0u;
            {
                unsigned m = pm & (nu == 32 ? 0xffffffffu : ((1u << nu) - 1u));  // warp-uniform (a ballot)
                while (m) {  // four neighbours' words in flight at once
                    uint32_t t[4][kBfWordsPerLane];
#pragma unroll
                    for (int a = 0; a < 4; ++a) {
                        const int q = m ? __ffs(m) - 1 : -1;
                        m &= m - 1;
                        const int u = __shfl_sync(0xffffffffu, myu, q < 0 ? 0 : q);
#pragma unroll
                        for (int j = 0; j < kBfWordsPerLane; ++j)
                            t[a][j] = (q >= 0 && 32 * j + lane < WC) ? __ldcg(&chg_in[(int64_t)u * W + wofs + 32 * j + lane]) : 0u;
                    }
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int j = 0; j < kBfWordsPerLane; ++j) act[j] |= t[a][j];
                }
            }
            if (end - beg > 32)  // long lists: the rest in order (rare)
                for (int64_t e = beg + 32; e < end; ++e) {
                    const int u = col[e];
                    if ((pend_in[u] >> ch) & 1u)
#pragma unroll
                        for (int j = 0; j < kBfWordsPerLane; ++j)
                            if (32 * j + lane < WC) act[j] |= __ldcg(&chg_in[(int64_t)u * W + wofs + 32 * j + lane]);
                }
            if (selfp)
#pragma unroll
                for (int j = 0; j < kBfWordsPerLane; ++j)
                    if (32 * j + lane < WC) own[j] = chg_in[(int64_t)v * W + wofs + 32 * j + lane];
            const double myl = lane < nu ? len[beg + lane] : 0.0;
            // The candidates (set bits of act | own) compacted over the lanes: round b gives
            // lane L the (32 b + L)-th candidate in (owner lane, word, bit) order, so a round
            // relaxes 32 (vertex, source) values whatever the words' bit density (one word at
            // a time used 8.7 of 32 lanes on W4).  The new change bits collect in the warp's
            // shared word buffer.
            uint32_t* ob = outw + (threadIdx.x >> 5) * (32 * kBfWordsPerLane);
            int cnt = 0;
#pragma unroll
            for (int j = 0; j < kBfWordsPerLane; ++j) {
                if (32 * j + lane < WC) ob[32 * j + lane] = 0u;
                cnt += __popc(act[j] | own[j]);
            }
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            __syncwarp();
            for (int base = 0; base < total; base += 32) {
                const int r = base + lane;
                int ol = 0;  // owner lane: the first with an inclusive count above r
#pragma unroll
                for (int step = 16; step > 0; step >>= 1) {
                    const int t = __shfl_sync(0xffffffffu, incl, ol + step - 1);
                    if (t <= r) ol += step;
                }
                int rr = r - (__shfl_sync(0xffffffffu, incl, ol) - __shfl_sync(0xffffffffu, cnt, ol));
                uint32_t aw = 0u, owd = 0u;
                int wj = 0;
                bool picked = false;
#pragma unroll
                for (int j = 0; j < kBfWordsPerLane; ++j) {
                    const uint32_t a = __shfl_sync(0xffffffffu, act[j], ol), o = __shfl_sync(0xffffffffu, own[j], ol);
                    const int c = __popc(a | o);
                    if (!picked && rr < c) {
                        aw = a;
                        owd = o;
                        wj = j;
                        picked = true;
                    } else if (!picked) {
                        rr -= c;
                    }
                }
                const bool valid = r < total && picked;
                const int bit = valid ? (int)__fns(aw | owd, 0u, rr + 1) : 0;
                const int word = 32 * wj + ol;
                const int k = 32 * (wofs + word) + bit;
                const bool on = valid && ((aw >> bit) & 1u) && k < nsrc;
                const bool mine = valid && ((owd >> bit) & 1u);
                FDL_DCHECK(!valid || (k < nsrc && k < S && word < WC));
                const double old = (on || mine) ? __ldcg(&dv[(int64_t)v * S + k]) : 0.0;
                double best = old;
                for (int q0 = 0; q0 < nu; q0 += 8) {
                    double c[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const int u = __shfl_sync(0xffffffffu, myu, (q0 + q) & 31);
                        const double l = __shfl_sync(0xffffffffu, myl, (q0 + q) & 31);
                        const double du = (on && q0 + q < nu) ? __ldcg(&dv[(int64_t)u * S + k]) : INFINITY;
                        c[q] = du <= T ? du + l : INFINITY;  // a distance above the threshold waits
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q) best = c[q] < best ? c[q] : best;
                }
                if (on)
                    for (int64_t e = beg + 32; e < end; ++e) {  // lists longer than 32 (rare)
                        const double du = __ldcg(&dv[(int64_t)col[e] * S + k]);
                        const double c = du <= T ? du + len[e] : INFINITY;
                        best = c < best ? c : best;
                    }
                bool imp = false;
                if (on && best < old) {
                    dv[(int64_t)v * S + k] = best;
                    imp = true;
                }
                // pending after this sweep: a new value, or an own pending value above the
                // threshold (its neighbours did not take it yet); own values <= T were pulled
                // by every neighbour in this sweep
                if (imp || (mine && old > T)) atomicOr(&ob[word], 1u << bit);
            }
            __syncwarp();
            bool anyw = false;
#pragma unroll
            for (int j = 0; j < kBfWordsPerLane; ++j)
                if (32 * j + lane < WC) {
                    const uint32_t wv = ob[32 * j + lane];
                    chg_out[(int64_t)v * W + wofs + 32 * j + lane] = wv;
                    anyw |= wv != 0u;
                }
            __syncwarp();
            if (__any_sync(0xffffffffu, anyw)) outmask |= 1u << ch;
        }
        if (lane == 0) pend_out[v] = (uint16_t)outmask;
        found |= outmask != 0u;
    }
    // per warp, no block barrier (a block's warps finish their vertex lists at
    // different times; a barrier here held 25% of the stall samples, W4)
    if (found && lane == 0) flags[it] = 1u;
}

// change bits of the batch's sources: vertex s0 + k has source k's bit (its
// distance 0 is the only finite value at the start)
__global__ void k_bf_seed(uint32_t* chg, uint16_t* pend, const int* __restrict__ srcs, int nsrc, int S)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nsrc) return;
    chg[(int64_t)srcs[k] * (S >> 5) + (k >> 5)] = 1u << (k & 31);
    pend[srcs[k]] = (uint16_t)(1u << (k / kBfChunk));  // a vertex is one source of the batch
}

cudaError_t launch_bf_sweep(const int64_t* row_ptr, const int32_t* col, const double* len, double* dist,
                            const uint32_t* chg_in, uint32_t* chg_out, const uint16_t* pend_in, uint16_t* pend_out,
                            int n, int S, int nsrc, int it, double delta, unsigned int* flags, int grid,
                            cudaStream_t s)
{
    // grid-stride warps: one wave of resident blocks (a second partial wave idled SMs)
    static const int resident = resident_blocks((const void*)k_bf_sweep, 256);
    const unsigned g = (unsigned)std::max(1, std::min({grid, resident, (int)(((int64_t)n * 32 + 255) / 256)}));
    k_bf_sweep<<<g, 256, 0, s>>>(row_ptr, col, len, dist, chg_in, chg_out, pend_in, pend_out, n, S, nsrc, it, delta,
                                 flags);
    return cudaGetLastError();
}

cudaError_t launch_bf_seed(uint32_t* chg, uint16_t* pend, const int* srcs, int nsrc, int S, cudaStream_t s)
{
    k_bf_seed<<<(nsrc + 255) / 256, 256, 0, s>>>(chg, pend, srcs, nsrc, S);
    return cudaGetLastError();
}

// rows srcs[0..nsrc) of the upper-triangle tiles of the local range <- fp32(dist)
__global__ void __launch_bounds__(256) k_bf_store(const double* __restrict__ dist, int n,
                                                  const int* __restrict__ srcs, int nsrc, int S, int nb, int64_t t0,
                                                  int64_t t1, float* D, double* dmax)
{
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // max distance as the max of the positive doubles' bit patterns (they order alike):
    // per block, one atomic (one per element serialised on the address: 67 ms per W4 batch)
    unsigned long long mb = 0ull;
    if (idx < (int64_t)n * nsrc) {
        const int v = (int)(idx / nsrc), k = (int)(idx % nsrc);
        const int src = srcs[k];
        const int I = src / kT, J = v / kT;
        const int64_t t = tri_index(I, J, nb);
        if (I <= J && t >= t0 && t < t1) {
            const double d = dist[(int64_t)v * S + k];
            FDL_DCHECK(sym_offset(t - t0, src % kT, v % kT, kHbDist) < (size_t)(t1 - t0) * tile_bytes(kHbDist));
            D[sym_offset(t - t0, src % kT, v % kT, kHbDist) / 4] = (float)d;
            if (d > 0.0) mb = (unsigned long long)__double_as_longlong(d);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xffffffffu, mb, o);
        mb = x > mb ? x : mb;
    }
    __shared__ unsigned long long wmax[8];
    if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = mb;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) mb = wmax[w] > mb ? wmax[w] : mb;
        if (mb) atomicMax(reinterpret_cast<unsigned long long*>(dmax), mb);
    }
}

cudaError_t launch_bf_store(const double* dist, int n, const int* srcs, int nsrc, int S, int nb, int64_t t0,
                            int64_t t1, uint8_t* D, double* dmax, cudaStream_t s)
{
    const int64_t total = (int64_t)n * nsrc;
    k_bf_store<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(dist, n, srcs, nsrc, S, nb, t0, t1,
                                                             reinterpret_cast<float*>(D), dmax);
    return cudaGetLastError();
}

// Dense rows of the stored distances (any width) as fp32: out[r][j] = d'(rows[r], j)
__global__ void k_dist_rows(const uint8_t* __restrict__ D, int hb, int nb, int64_t t0, int64_t t1,
                            const int* __restrict__ rows, int nrows, int n, float* out, int* missing)
{
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)nrows * n) return;
    const int r = (int)(idx / n), j = (int)(idx % n);
    int a = rows[r], b = j;
    if (a / kT > b / kT) {
        const int tmp = a;
        a = b;
        b = tmp;
    }
    const int64_t t = tri_index(a / kT, b / kT, nb);
    if (t < t0 || t >= t1) {
        *missing = 1;
        out[idx] = 0.0f;
        return;
    }
    const size_t off = sym_offset(t - t0, a % kT, b % kT, hb);
    float v;
    if (hb == kHbDist)
        v = *reinterpret_cast<const float*>(D + off);
    else if (hb == 0)
        v = (float)((a & 1) ? nib_decode_hi(D[off]) : nib_decode_lo(D[off]));
    else if (hb == 1)
        v = (float)D[off];
    else
        v = (float)(D[off] | (D[off + 1] << 8));
    out[idx] = (rows[r] == j) ? 0.0f : v;
}

cudaError_t launch_dist_rows(const uint8_t* D, int hb, int nb, int64_t t0, int64_t t1, const int* rows, int nrows,
                             int n, float* out, int* missing, cudaStream_t s)
{
    const int64_t total = (int64_t)nrows * n;
    k_dist_rows<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(D, hb, nb, t0, t1, rows, nrows, n, out, missing);
    return cudaGetLastError();
}

// raw (lo | hi << 4) -> nib_encode, four bytes per 32-bit word at once (no
// carries cross a byte: lo + 4 hi <= 75)
__global__ void k_nib_encode(uint32_t* __restrict__ D, size_t words)
{
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += (size_t)gridDim.x * blockDim.x) {
        const uint32_t w = D[i];
        const uint32_t lo = w & 0x0F0F0F0Fu, hi = (w >> 4) & 0x0F0F0F0Fu;
        D[i] = ((lo + (hi << 2)) & 0x0F0F0F0Fu) | (hi << 4);
    }
}

cudaError_t launch_nib_encode(uint8_t* D, size_t bytes, cudaStream_t s)
{
    const size_t words = bytes / 4;  // tiles are 8 KB: always whole words
    if (words == 0) return cudaSuccess;
    const unsigned grid = (unsigned)std::min<size_t>((words + 255) / 256, 148 * 16);
    k_nib_encode<<<grid, 256, 0, s>>>(reinterpret_cast<uint32_t*>(D), words);
    return cudaGetLastError();
}

}  // namespace fdl
