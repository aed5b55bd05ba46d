// Is MUFU rcp.approx.ftz.f32(h^2) the correctly rounded fp32(1/h^2) for the hop
// values the 4-bit (1..15) and 8-bit (1..255) tables hold?  Prints the mismatches.
#include <cstdio>
__global__ void k(int hmax, int* bad, int* nbad)
{
    const int h = blockIdx.x * blockDim.x + threadIdx.x + 1;
    if (h > hmax) return;
    const float h2 = (float)h * (float)h;
    float a;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(a) : "f"(h2));
    const float b = __frcp_rn(h2);
    if (a != b) {
        const int i = atomicAdd(nbad, 1);
        if (i < 64) bad[i] = h;
    }
}
int main()
{
    int *bad, *nbad;
    cudaMallocManaged(&bad, 64 * sizeof(int));
    cudaMallocManaged(&nbad, sizeof(int));
    for (int hmax : {15, 255, 4095}) {
        *nbad = 0;
        k<<<(hmax + 255) / 256, 256>>>(hmax, bad, nbad);
        cudaDeviceSynchronize();
        printf("hmax %d: %d mismatches:", hmax, *nbad);
        for (int i = 0; i < *nbad && i < 64; ++i) printf(" %d", bad[i]);
        printf("\n");
    }
    return 0;
}
