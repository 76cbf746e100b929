// FP64 throughput on this GPU: DFMA (CUDA cores) vs mma.sync m8n8k4 f64 (tensor cores).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double *out, int iters, double a, double b) {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    double s = 0;
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.0) out[0] = s;
}

__global__ void dmma_kernel(double *out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[4][2];
    for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(c[i][0]), "+d"(c[i][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.0) out[0] = s;
}

__global__ void mixed_kernel(double *out, int iters, double a2, double b2) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[4][2];
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(c[i][0]), "+d"(c[i][1])
                         : "d"(a), "d"(b));
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a2, b2);
    }
    double s = 0;
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 12345.0) out[0] = s;
}

int main() {
    double *out;
    cudaMalloc(&out, 8);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 1 << 14;
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(e0);
        dfma_kernel<<<nsm * 8, 256>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * iters * (double)nsm * 8 * 256;
        printf("DFMA: %.1f TFLOP/s\n", flops / (ms * 1e-3) / 1e12);
        for (int blocks_per_sm : {4, 8, 16}) {
            cudaEventRecord(e0);
            dmma_kernel<<<nsm * blocks_per_sm, 128>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            double mflops = 2.0 * 256 * 4 * iters * (double)nsm * blocks_per_sm * 4;  // per warp 256 FMA per mma
            printf("DMMA m8n8k4 (%d blocks/SM x 4 warps): %.1f TFLOP/s\n", blocks_per_sm,
                   mflops / (ms * 1e-3) / 1e12);
        }
    }
    {
        float ms;
        cudaEventRecord(e0);
        mixed_kernel<<<nsm * 8, 128>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double warps = (double)nsm * 8 * 4;
        double f = (2.0 * 256 * 4 + 2.0 * 8 * 32) * iters * warps;
        printf("mixed DMMA+DFMA: %.1f TFLOP/s total (%.3f ms)\n", f / (ms * 1e-3) / 1e12, ms);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
