// frame_kernels.cuh -- per-frame radiometric kernels (LUT, phase-plane
// pre-pass, float64 sample planes, saturation masks) and the DFMA probe.
#pragma once

#include "config.cuh"

namespace hdrlpa {

// Exact radiometry LUT (scalar calibration): entry v = radiance_exact of a
// raw value v below saturation, for the slow path's float64 sweeps.
__global__ void radiance_lut_kernel(const __grid_constant__ DevParams P) {
    const DevSensor &S = P.s[blockIdx.y];
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (S.planes || v >= S.sat) return;
    double f, iv;
    radiometry_exact(S, v, S.bias, S.nonuni, S.readvar, P.use_sigma, f, iv);
    S.lut[v] = make_double2(f, iv);
}

// Per-frame radiometric pre-pass: every raw pixel converted once into the
// de-interleaved phase planes (radiometry.py:303-336 for the whole frame);
// out-of-frame padding gets 1/den = 0 (no sample).  HBM-bound.
// One thread per (sensor, phase row j, group of 4 phase columns): raw rows
// 2j and 2j+1, columns 8g..8g+7 read as 16-B vectors (when the frame's pitch
// and base allow), the four phase planes written as 2 x 16-B per plane.
__global__ void __launch_bounds__(128) radiance_phase_kernel(const __grid_constant__ DevParams P) {
    const DevSensor &S = P.s[blockIdx.z];
    const int j = blockIdx.y * blockDim.y + threadIdx.y;
    const int i0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (i0 >= S.pwg || j >= S.phg) return;
    const int x0 = 2 * i0;
    const bool vec = S.vec_raw && x0 + 8 <= S.pitch;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const int y = 2 * j + r;
        uint16_t v[8];
        if (y < S.height && vec) {
            const uint4 q = __ldg((const uint4 *)(S.raw + (size_t)y * S.pitch + x0));
            const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                v[2 * k] = (uint16_t)(w[k] & 0xffffu);
                v[2 * k + 1] = (uint16_t)(w[k] >> 16);
            }
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k)
                v[k] = (y < S.height && x0 + k < S.width) ? __ldg(S.raw + (size_t)y * S.pitch + x0 + k)
                                                          : (uint16_t)0;
        }
        float2 o[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
            o[k] = (y < S.height && x0 + k < S.width)
                       ? radiance_from_raw(S, (int)v[k], x0 + k, y, P.use_sigma)
                       : make_float2(0.f, 0.f);  // padding: no sample
#pragma unroll
        for (int px = 0; px < 2; ++px) {
            float4 *dst = (float4 *)(S.phase + ((size_t)(2 * r + px) * S.phg + j) * S.pwg + i0);
            dst[0] = make_float4(o[px].x, o[px].y, o[px + 2].x, o[px + 2].y);
            dst[1] = make_float4(o[px + 4].x, o[px + 4].y, o[px + 6].x, o[px + 6].y);
        }
    }
}

// Co-sited pre-pass (PAT 3/4: every sensor has the same transform, frame size
// and Bayer phase, so the samples of all sensors at a sensor pixel share one
// position, offset and window weight): the sensors' samples of a pixel merged
// into one float4 (sum 1/den, sum f_hat/den, sum |f_hat|/den, count) in the
// phase-plane layout [4][phg][pwg] (sensor 0's geometry; the planes occupy
// the workspace of sensors 0 and 1).  Sensors are summed in index order.
__device__ __forceinline__ void load_raw8(const DevSensor &S, int x0, int y, uint16_t (&v)[8]) {
    if (S.vec_raw && x0 + 8 <= S.pitch) {
        const uint4 q = __ldg((const uint4 *)(S.raw + (size_t)y * S.pitch + x0));
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[2 * k] = (uint16_t)(w[k] & 0xffffu);
            v[2 * k + 1] = (uint16_t)(w[k] >> 16);
        }
    } else {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            v[k] = x0 + k < S.width ? __ldg(S.raw + (size_t)y * S.pitch + x0 + k) : (uint16_t)0;
    }
}

// Scalar-calibration radiometry of a raw value for the merged planes, branch
// free: (f_hat, 1/den) as radiance_from_raw (same fp32 operations; the
// reciprocal is MUFU + one Newton step, within 1 ulp of the rounded one),
// 1/den = 0 at or above saturation.
__device__ __forceinline__ void merge_scalar(const DevSensor &S, uint32_t raw, int use_sigma,
                                             float4 &o) {
    const float f = ((float)raw - S.bias_f) * S.inv_denom_f;
    const float shot = S.c_shot_f * fmaxf(f, 0.f);
    const float var = fmaxf((shot + S.readvar_f) * S.inv_denom2_f, S.qv_f);
    float iv;
    if (use_sigma) {
        iv = rsqrtf(var);
    } else {
        float r;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(var));
        iv = fmaf(r, fmaf(-var, r, 1.f), r);
    }
    iv = (int)raw < S.sat ? iv : 0.f;
    o.x += iv;
    o.y = fmaf(f, iv, o.y);
    o.z = fmaf(fabsf(f), iv, o.z);
    o.w += iv > 0.f ? 1.f : 0.f;
}

// One thread per (phase row j, raw row 2j + r) and 4 phase columns i spaced
// by a warp (i = base + lane + 32k): every store of a warp is 32 consecutive
// float4 (512 B) and every raw load 32 consecutive 4-B pixel pairs.  The raw
// pairs of all sensors and columns are loaded before any conversion (the loads
// overlap).  Sensors with scalar calibration, no defect map and 16-B rows take
// a branch-free path.  (HDR_MERGE_COALESCED 0: the previous mapping, 4
// adjacent phase columns per thread -- each warp store then touched 32
// half-sectors 64 B apart.)
#ifndef HDR_MERGE_COALESCED
#define HDR_MERGE_COALESCED 1
#endif
__global__ void __launch_bounds__(128) radiance_merge_kernel(const __grid_constant__ DevParams P) {
#if HDR_MERGE_COALESCED
    const DevSensor &S0 = P.s[0];
    const int jr = blockIdx.y * blockDim.y + threadIdx.y;
    const int j = jr >> 1, r = jr & 1;
    if (j >= S0.phg) return;
    const int y = 2 * j + r;
    const int ib = blockIdx.x * 128 + (int)threadIdx.x;
    float4 *planes = (float4 *)S0.phase;
    float4 *dst0 = planes + ((size_t)(2 * r) * S0.phg + j) * S0.pwg;
    float4 *dst1 = planes + ((size_t)(2 * r + 1) * S0.phg + j) * S0.pwg;
    bool simple = y < S0.height;
#pragma unroll
    for (int s = 0; s < PAT_MAXS; ++s)
        if (s < P.n_sensors) simple &= !P.s[s].planes && !P.s[s].defective && P.s[s].vec_raw;
    // the scalar path per aligned group of 8 raw columns inside the width (the
    // previous mapping's rule, so every pixel takes the same path as before)
    if (simple && ((2 * (ib + 96)) & ~7) + 8 <= S0.width) {
        uint32_t w[4][PAT_MAXS];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int s = 0; s < PAT_MAXS; ++s)
                if (s < P.n_sensors)
                    w[k][s] = __ldg((const uint32_t *)(P.s[s].raw + (size_t)y * P.s[s].pitch +
                                                       2 * (ib + 32 * k)));
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            float4 o0 = make_float4(0.f, 0.f, 0.f, 0.f), o1 = o0;
#pragma unroll
            for (int s = 0; s < PAT_MAXS; ++s) {
                if (s >= P.n_sensors) break;
                merge_scalar(P.s[s], w[k][s] & 0xffffu, P.use_sigma, o0);
                merge_scalar(P.s[s], w[k][s] >> 16, P.use_sigma, o1);
            }
            dst0[ib + 32 * k] = o0;
            dst1[ib + 32 * k] = o1;
        }
        return;
    }
    // the frame's right edge, odd widths, per-pixel calibration planes, defects
    for (int k = 0; k < 4; ++k) {
        const int i = ib + 32 * k;
        if (i >= S0.pwg) break;
        float4 o[2] = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
        if (y < S0.height) {
            for (int s = 0; s < PAT_MAXS; ++s) {
                if (s >= P.n_sensors) break;
                const DevSensor &S = P.s[s];
                for (int d = 0; d < 2; ++d) {
                    const int x = 2 * i + d;
                    if (x >= S.width) continue;
                    const int v = (int)__ldg(S.raw + (size_t)y * S.pitch + x);
                    if (simple && (x & ~7) + 8 <= S0.width) {
                        merge_scalar(S, (uint32_t)v, P.use_sigma, o[d]);
                    } else {
                        const float2 e = radiance_from_raw(S, v, x, y, P.use_sigma);
                        o[d].x += e.y;
                        o[d].y = fmaf(e.x, e.y, o[d].y);
                        o[d].z = fmaf(fabsf(e.x), e.y, o[d].z);
                        o[d].w += e.y > 0.f ? 1.f : 0.f;
                    }
                }
            }
        }
        dst0[i] = o[0];
        dst1[i] = o[1];
    }
#else
    const DevSensor &S0 = P.s[0];
    const int jr = blockIdx.y * blockDim.y + threadIdx.y;
    const int j = jr >> 1, r = jr & 1;
    const int i0 = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (i0 >= S0.pwg || j >= S0.phg) return;
    const int x0 = 2 * i0;
    const int y = 2 * j + r;
    float4 o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (y < S0.height) {
        bool simple = x0 + 8 <= S0.width;
#pragma unroll
        for (int s = 0; s < PAT_MAXS; ++s)
            if (s < P.n_sensors)
                simple &= !P.s[s].planes && !P.s[s].defective && P.s[s].vec_raw;
        if (simple) {
            uint4 q[PAT_MAXS];
#pragma unroll
            for (int s = 0; s < PAT_MAXS; ++s)
                if (s < P.n_sensors)
                    q[s] = __ldg((const uint4 *)(P.s[s].raw + (size_t)y * P.s[s].pitch + x0));
#pragma unroll
            for (int s = 0; s < PAT_MAXS; ++s) {
                if (s >= P.n_sensors) break;
                const uint32_t w[4] = {q[s].x, q[s].y, q[s].z, q[s].w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    merge_scalar(P.s[s], w[k] & 0xffffu, P.use_sigma, o[2 * k]);
                    merge_scalar(P.s[s], w[k] >> 16, P.use_sigma, o[2 * k + 1]);
                }
            }
        } else {
            uint16_t v[PAT_MAXS][8];
#pragma unroll
            for (int s = 0; s < PAT_MAXS; ++s)
                if (s < P.n_sensors) load_raw8(P.s[s], x0, y, v[s]);
#pragma unroll
            for (int s = 0; s < PAT_MAXS; ++s) {
                if (s >= P.n_sensors) break;
                const DevSensor &S = P.s[s];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (x0 + k >= S.width) continue;
                    const float2 e = radiance_from_raw(S, (int)v[s][k], x0 + k, y, P.use_sigma);
                    o[k].x += e.y;
                    o[k].y = fmaf(e.x, e.y, o[k].y);
                    o[k].z = fmaf(fabsf(e.x), e.y, o[k].z);
                    o[k].w += e.y > 0.f ? 1.f : 0.f;
                }
            }
        }
    }
    float4 *planes = (float4 *)S0.phase;
#pragma unroll
    for (int px = 0; px < 2; ++px) {
        float4 *dst = planes + ((size_t)(2 * r + px) * S0.phg + j) * S0.pwg + i0;
#pragma unroll
        for (int k = 0; k < 4; ++k) dst[k] = o[px + 2 * k];
    }
#endif
}

// ---------------------------------------------------------------------------
// Saturation mask bit-planes (radiometry.py:298-300, :316-317)
// ---------------------------------------------------------------------------
__global__ void saturation_mask_kernel(const DevSensor S, uint32_t *bits, int wpr) {
    const int y = blockIdx.y;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    bool m = false;
    if (x < S.width) {
        const int raw = (int)__ldg(S.raw + (size_t)y * S.pitch + x);
        m = raw >= S.sat || (S.defective && __ldg(S.defective + (size_t)y * S.width + x));
    }
    const uint32_t word = __ballot_sync(0xffffffffu, m);
    if ((threadIdx.x & 31) == 0 && x < S.width) bits[(size_t)y * wpr + (x >> 5)] = word;
}

__global__ void radiance_planes_kernel(const DevSensor S, int use_sigma, float *value,
                                       float *inv_den) {
    const int y = blockIdx.y;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= S.width) return;
    const float2 e = radiance_sample(S, x, y, use_sigma);
    value[(size_t)y * S.width + x] = e.x;
    inv_den[(size_t)y * S.width + x] = e.y;
}

// The reference's sample columns as float64 planes (radiometry.py:303-336):
// value = f_hat, sigma = sqrt(max(var, quantisation floor)); sigma = 0 marks
// "no sample" (saturated / defective).
__global__ void sample_planes_kernel(const DevSensor S, double *value, double *sigma) {
    const int y = blockIdx.y;
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= S.width) return;
    const size_t i = (size_t)y * S.width + x;
    const int raw = (int)__ldg(S.raw + (size_t)y * S.pitch + x);
    double f = 0.0, sg = 0.0;
    if (raw < S.sat && !(S.defective && __ldg(S.defective + i))) {
        const double b = S.bias_p ? __ldg(S.bias_p + i) : S.bias;
        const double a = S.nonuni_p ? __ldg(S.nonuni_p + i) : S.nonuni;
        const double vr = S.readvar_p ? __ldg(S.readvar_p + i) : S.readvar;
        radiometry_sigma(S, raw, b, a, vr, f, sg);
    }
    value[i] = f;
    sigma[i] = sg;
}

// DFMA throughput probe: 8 independent chains per thread, full occupancy.
__global__ void __launch_bounds__(256) fp64_probe_kernel(double *sink, int iters, double a,
                                                         double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
        x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
        x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
    const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 1234.5) sink[threadIdx.x] = s;  // keep the chains alive
}

}  // namespace hdrlpa
