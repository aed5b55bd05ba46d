// Per-instruction throughput on sm_100a (SMSP cycles per warp instruction).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_rates pipe_rates.cu
// Results: profiles/r01_pipe_rates.md
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) { u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ u64 fadd2(u64 a, u64 b) { u64 d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ float ffma(float a, float b, float c) { float d; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
__device__ __forceinline__ float rsq(float x) { float y; asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

template <int K>
__global__ void k(float* out, int iters, float p)
{
    float a[8], b[8], c[8];
    u64 A[8], B[8], Cc[8];
    for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3f + i; b[i] = p + i * 1e-3f; c[i] = 1e-3f * i; A[i] = __float_as_uint(a[i]) | ((u64)__float_as_uint(b[i]) << 32); B[i] = A[i] ^ 0x100000001ull; Cc[i] = A[i] ^ 0x200000002ull; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (K == 0) a[i] = ffma(a[i], b[i], c[i]);           // FFMA, 3 distinct regs
            if (K == 1) A[i] = ffma2(A[i], B[i], Cc[i]);         // FFMA2, 3 distinct reg pairs
            if (K == 2) A[i] = fadd2(A[i], B[i]);                // FADD2
            if (K == 3) a[i] = rsq(a[i]);                        // MUFU.RSQ
            if (K == 4) { a[i] = ffma(a[i], b[i], c[i]); A[i] = ffma2(A[i], B[i], Cc[i]); }
            if (K == 5) { A[i] = ffma2(A[i], B[i], Cc[i]); if (i < 2) a[i] = rsq(a[i]); }   // 8 FFMA2 : 2 MUFU
            if (K == 6) { a[i] = ffma(a[i], b[0], c[i]); }       // FFMA with one shared operand
        }
    }
    float s = 0; for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float((unsigned)A[i]);
    if (s == 1.2345f) out[threadIdx.x] = s;
}
template <int K>
void run(const char* name, int per_it, float* out)
{
    const int iters = 20000, blocks = 148 * 4, threads = 256;
    k<K><<<blocks, threads>>>(out, 10, 1.f);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); k<K><<<blocks, threads>>>(out, iters, 1.f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double winstr = (double)blocks * threads / 32 * iters * 8 * per_it;  // warp instructions (per_it per i)
    printf("%-34s %.3f SMSP-cycles per warp instruction group\n", name, ms * 1e-3 * 1.965e9 * 148 * 4 / (winstr / per_it));
}
int main()
{
    float* out; cudaMalloc(&out, 4096 * 4);
    run<0>("FFMA r,r,r", 1, out);
    run<1>("FFMA2 rr,rr,rr", 1, out);
    run<2>("FADD2 rr,rr", 1, out);
    run<3>("MUFU.RSQ", 1, out);
    run<4>("FFMA + FFMA2 (per pair of instrs)", 2, out);
    run<5>("FFMA2 x8 + MUFU x2 (per FFMA2)", 1, out);
    run<6>("FFMA r,rshared,r", 1, out);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
