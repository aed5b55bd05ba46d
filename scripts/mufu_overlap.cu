// How MUFU ops overlap with FP32 FFMA work on sm_100a (SMSP cycles per group).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_overlap mufu_overlap.cu
// Results: profiles/r01_pipe_rates.md
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ffma(float a, float b, float c) { float d; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
__device__ __forceinline__ float fadd(float a, float b) { float d; asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b)); return d; }
__device__ __forceinline__ float rsq(float x) { float y; asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float sq(float x) { float y; asm volatile("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float lg2(float x) { float y; asm volatile("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float rcp(float x) { float y; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float rsq2(float x) { return ex2(-0.5f * lg2(x)); }

// NF scalar FFMA + NM MUFU per group, 8 independent chains each
template <int NF, int NM, int KIND>
__global__ void k(float* out, int iters, float p)
{
    float a[16], m[4];
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
    for (int i = 0; i < 4; ++i) m[i] = 1.f + i + threadIdx.x;
    const float b = p, c = p * 0.5f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int f = 0; f < NF; ++f) {
            a[f % 16] = ffma(a[f % 16], b, a[(f + 5) % 16]);
            constexpr int step = NM ? NF / NM : 1;
            if (NM && f % step == 0) {
                const int j = (f / step) % 4;
                m[j] = KIND == 0 ? rsq(m[j] + c) : (KIND == 1 ? sq(m[j] + c) : (KIND == 2 ? ex2(m[j]) : (KIND == 3 ? lg2(m[j] + c) : (KIND == 4 ? rcp(m[j] + c) : rsq2(m[j] + c)))));
            }
        }
    }
    float s = 0; for (int i = 0; i < 16; ++i) s += a[i]; for (int i = 0; i < 4; ++i) s += m[i];
    if (s == 1.2345f) out[threadIdx.x] = s;
}
template <int NF, int NM, int KIND = 0>
void run(const char* name, float* out)
{
    const int iters = 4000, blocks = 148 * 4, threads = 256;
    k<NF, NM, KIND><<<blocks, threads>>>(out, 10, 1.f);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); k<NF, NM, KIND><<<blocks, threads>>>(out, iters, 1.f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double groups = (double)blocks * threads / 32 * iters;
    printf("%-30s %.2f SMSP-cycles per group (NF=%d NM=%d)\n", name, ms * 1e-3 * 1.965e9 * 148 * 4 / groups, NF, NM);
}
int main()
{
    float* out; cudaMalloc(&out, 4096 * 4);
    run<16, 0>("16 FFMA", out);
    run<16, 2>("16 FFMA + 2 RSQ", out);
    run<16, 2, 2>("16 FFMA + 2 EX2", out);
    run<16, 2, 3>("16 FFMA + 2 LG2", out);
    run<16, 2, 4>("16 FFMA + 2 RCP", out);
    run<16, 2, 5>("16 FFMA + 2 (LG2,FMUL,EX2)", out);
    run<2, 2, 2>("2 FFMA + 2 EX2", out);
    run<2, 2, 3>("2 FFMA + 2 LG2", out);
    run<2, 2, 5>("2 FFMA + 2 (LG2,FMUL,EX2)", out);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
