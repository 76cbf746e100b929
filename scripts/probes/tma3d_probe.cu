// Probe: 3-D float32 TMA tile copy (box {bx, by, 4}) at given start coords.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
struct Params { CUtensorMap m; int x, y, bx, by; float *out; };
__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ Params P) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(sa(&bar)), "r"(P.bx * P.by * 4 * 4) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(sa(smem)), "l"((uint64_t)&P.m), "r"(P.x), "r"(P.y), "r"(0), "r"(sa(&bar)) : "memory");
    }
    asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(sa(&bar)), "r"(0) : "memory");
    const float *f = (const float *)smem;
    for (int i = threadIdx.x; i < P.bx * P.by * 4; i += blockDim.x) P.out[i] = f[i];
}
int main(int argc, char **argv) {
    const int DW = 64, DH = 24;
    Params P; memset(&P, 0, sizeof(P));
    P.x = atoi(argv[1]); P.y = atoi(argv[2]); P.bx = atoi(argv[3]); P.by = atoi(argv[4]);
    float *d, *o; cudaMalloc(&d, DW * DH * 4 * 4); cudaMalloc(&o, P.bx * P.by * 16);
    float *h = (float *)malloc(DW * DH * 16);
    for (int i = 0; i < DW * DH * 4; ++i) h[i] = (float)i + 1;
    cudaMemcpy(d, h, DW * DH * 16, cudaMemcpyHostToDevice);
    void *fnp; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
    cuuint64_t dims[3] = {DW, DH, 4}, str[2] = {DW * 4, DW * DH * 4};
    cuuint32_t box[3] = {(cuuint32_t)P.bx, (cuuint32_t)P.by, 4}, es[3] = {1, 1, 1};
    CUresult r = enc(&P.m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    P.out = o;
    k<<<1, 128, P.bx * P.by * 16 + 128>>>(P);
    cudaError_t e = cudaDeviceSynchronize();
    int bad = 0;
    if (e == cudaSuccess) {
        float *ho = (float *)malloc(P.bx * P.by * 16);
        cudaMemcpy(ho, o, P.bx * P.by * 16, cudaMemcpyDeviceToHost);
        for (int z = 0; z < 4; ++z) for (int y = 0; y < P.by; ++y) for (int x = 0; x < P.bx; ++x) {
            int gx = P.x + x, gy = P.y + y;
            float want = (gx >= 0 && gy >= 0 && gx < DW && gy < DH) ? h[(z * DH + gy) * DW + gx] : 0.f;
            if (ho[(z * P.by + y) * P.bx + x] != want) ++bad;
        }
    }
    printf("x=%d y=%d box=%dx%d encode=%d kernel=%s bad=%d\n", P.x, P.y, P.bx, P.by, (int)r, cudaGetErrorString(e), bad);
    return 0;
}
