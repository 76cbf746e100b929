// Standalone probe of the TMA staging pattern used by lpa_fast_kernel.
// variant 0: tensor map in __grid_constant__ param struct (as in the kernel)
// variant 1: same, dynamic smem base manually aligned to 128 B
// variant 2: tensor map copied to global memory
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>

struct Params {
    CUtensorMap tmap[2];
    int ox, oy, rw, rh;
    uint16_t *out;
    const CUtensorMap *gmap;
};

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int V>
__global__ void k(const __grid_constant__ Params P, int flags) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    unsigned char *buf = smem;
    if (V == 1) buf = (unsigned char *)(((uintptr_t)smem + 127) & ~(uintptr_t)127);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar)), "r"(1));
        if (!(flags & 1)) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        else asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const CUtensorMap *m = (V == 2) ? P.gmap : &P.tmap[0];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(sa(&bar)), "r"(P.rw * P.rh * 2) : "memory");
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(sa(buf)), "l"((uint64_t)m), "r"(P.ox), "r"(P.oy), "r"(sa(&bar)) : "memory");
    }
    asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(sa(&bar)), "r"(0) : "memory");
    const uint16_t *b16 = (const uint16_t *)buf;
    for (int i = threadIdx.x; i < P.rw * P.rh; i += blockDim.x) P.out[i] = b16[i];
}

int main(int argc, char **argv) {
    int V = argc > 1 ? atoi(argv[1]) : 0;
    int flags = argc > 2 ? atoi(argv[2]) : 0;
    const int W = 160, H = 112, pitch = 160;
    uint16_t *d_raw, *d_out;
    cudaMalloc(&d_raw, W * H * 2);
    uint16_t *h = (uint16_t *)malloc(W * H * 2);
    for (int i = 0; i < W * H; ++i) h[i] = (uint16_t)(i * 7 + 3);
    cudaMemcpy(d_raw, h, W * H * 2, cudaMemcpyHostToDevice);
    Params P;
    memset(&P, 0, sizeof(P));
    P.ox = (flags & 4) ? 8 : -4; if (argc > 3) P.ox = atoi(argv[3]); P.oy = 10; P.rw = 48; P.rh = 22;
    cudaMalloc(&d_out, P.rw * P.rh * 2);
    void *fnp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
    cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H}, str[1] = {(cuuint64_t)pitch * 2};
    cuuint32_t box[2] = {(cuuint32_t)P.rw, (cuuint32_t)P.rh}, es[2] = {1, 1};
    CUresult r = enc(&P.tmap[0], CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, d_raw, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("variant %d encode=%d sizeof(Params)=%zu\n", V, (int)r, sizeof(Params));
    CUtensorMap *gm;
    cudaMalloc(&gm, sizeof(CUtensorMap));
    cudaMemcpy(gm, &P.tmap[0], sizeof(CUtensorMap), cudaMemcpyHostToDevice);
    P.gmap = gm;
    P.out = d_out;
    int smem = P.rw * P.rh * 2 + 256;
    if (flags & 2) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(1); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        cudaError_t le = cudaLaunchKernelEx(&cfg, k<0>, P, flags);
        printf("launchEx: %s\n", cudaGetErrorString(le));
    } else {
        if (V == 0) k<0><<<1, 128, smem>>>(P, flags);
        if (V == 1) k<1><<<1, 128, smem>>>(P, flags);
        if (V == 2) k<2><<<1, 128, smem>>>(P, flags);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d flags %d kernel: %s\n", V, flags, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    uint16_t *o = (uint16_t *)malloc(P.rw * P.rh * 2);
    cudaMemcpy(o, d_out, P.rw * P.rh * 2, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int y = 0; y < P.rh; ++y)
        for (int x = 0; x < P.rw; ++x) {
            int gx = P.ox + x, gy = P.oy + y;
            uint16_t want = (gx >= 0 && gy >= 0 && gx < W && gy < H) ? h[gy * pitch + gx] : 0;
            if (o[y * P.rw + x] != want) ++bad;
        }
    printf("variant %d mismatches %d\n", V, bad);
    return 0;
}
