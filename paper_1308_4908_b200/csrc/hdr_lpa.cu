// hdr_lpa.cu -- sm_100a kernels and the C ABI (include/hdr_lpa.h) of the
// unified HDR LPA operator.
//
// Pipeline per frame (one stream, no host synchronisation):
//   1. memset of the slow-path work counter
//   2. lpa_fast_kernel<ORDER, ICI>: one CTA per 32x8 output tile.  The raw
//      uint16 footprint of the tile plus its window halo is staged per sensor
//      into shared memory, converted once per pixel into (f_hat, 1/den) fp32
//      pairs and de-interleaved into the four Bayer phase planes.  One thread
//      per output pixel then fits R, G and B: exact float64 support test,
//      fp32 window weight, float64 moment accumulation, in-register Cholesky,
//      condition bounds and (optionally) ICI scale selection.  Any pixel-
//      channel whose decision the fast path cannot take exactly (too few
//      samples, ill-conditioned, condition number near the threshold) is
//      appended to a work list.
//   3. lpa_slow_kernel<ORDER>: grid-stride over the work list; re-evaluates
//      those items from global memory with the reference's complete semantics
//      (radius ladder x1.5 up to max_radius, order fallback, exact eigenvalue
//      range) -- _kernels.py:257-300.
#include <cuda_runtime.h>
#include <climits>
#include <math.h>
#include <stdio.h>
#include <string.h>

#include "hdr_lpa.h"
#include "lpa_device.cuh"

namespace hdrlpa {

constexpr int TW = 32, TH = 8, NT = TW * TH;

template <int ORDER>
struct NC {
    static constexpr int P = (ORDER + 1) * (ORDER + 2) / 2;
};

// ---------------------------------------------------------------------------
// Window sweeps.  The iteration order (sensor, Bayer phase, row, column over
// the window's sensor bbox) depends only on (q, r, sensor), never on the tile,
// so a pixel's result is identical whichever path or band computes it.
// ---------------------------------------------------------------------------
template <class Fetch, class Body>
__device__ __forceinline__ void sweep(const DevParams &P, int c, double qx, double qy, double r,
                                      double r2, Fetch fetch, Body body) {
    for (int s = 0; s < P.n_sensors; ++s) {
        const DevSensor &S = P.s[s];
        const int pm = S.phmask[c];
        if (!pm) continue;
        int xlo, xhi, ylo, yhi;
        window_bbox(S, qx, qy, r, xlo, xhi, ylo, yhi);
        const double T0 = S.T[0], T1 = S.T[1], T2 = S.T[2];
        const double T3 = S.T[3], T4 = S.T[4], T5 = S.T[5];
        for (int ph = 0; ph < 4; ++ph) {
            if (!((pm >> ph) & 1)) continue;
            const int py = ph >> 1, px = ph & 1;
            const int ys = ylo + ((py - ylo) & 1), xs = xlo + ((px - xlo) & 1);
            for (int y = ys; y <= yhi; y += 2) {
                const double yd = (double)y;
                const double t1y = __dmul_rn(T1, yd), t4y = __dmul_rn(T4, yd);
                for (int x = xs; x <= xhi; x += 2) {
                    const float2 e = fetch(s, x, y);
                    if (!(e.y > 0.f)) continue;  // saturated / defective / off-frame
                    const double xd = (double)x;
                    // apply_transform (radiometry.py:84): T00*x + T01*y + T02
                    const double X = __dadd_rn(__dadd_rn(__dmul_rn(T0, xd), t1y), T2);
                    const double Y = __dadd_rn(__dadd_rn(__dmul_rn(T3, xd), t4y), T5);
                    const double dx = __dsub_rn(X, qx), dy = __dsub_rn(Y, qy);
                    const double dxx = __dmul_rn(dx, dx), dyy = __dmul_rn(dy, dy);
                    if (__dadd_rn(dxx, dyy) > r2) continue;  // _kernels.py:162
                    body(e, dx, dy, dxx, dyy);
                }
            }
        }
    }
}

// Window weight W = exp(-dX^T Hinv dX) (_kernels.py:164-168) with isotropic
// Hinv = I/h.  Fast path: fp32 MUFU ex2 (q <= 9 at the base/ICI radii).  Exact
// path: float64 exp in the reference's operation order, because the radius
// ladder reaches q ~ 1e2 where fp32 would underflow.
template <bool EXACT>
__device__ __forceinline__ double window_w(const DevParams &P, int c, int k, double dx, double dy,
                                           double dxx, double dyy) {
    if constexpr (EXACT) {
        const double hi = P.hinv[c][k];
        const double q = __dadd_rn(__dmul_rn(__dmul_rn(hi, dx), dx), __dmul_rn(__dmul_rn(hi, dy), dy));
        return exp(-q);
    } else {
        return (double)ex2_approx(-P.hl[c][k] * (float)(dxx + dyy));
    }
}

template <int ORDER, bool EXACT>
using AccFor = Acc<NC<ORDER>::P, (!EXACT && ORDER == 0)>;

template <int ORDER, bool EXACT, class Fetch>
__device__ __forceinline__ void accumulate(const DevParams &P, int c, int k, double qx, double qy,
                                           double r, double r2, Fetch fetch,
                                           AccFor<ORDER, EXACT> &acc) {
    acc.zero();
    sweep(P, c, qx, qy, r, r2, fetch, [&](float2 e, double dx, double dy, double dxx, double dyy) {
        if constexpr (!EXACT && ORDER == 0) {
            const float W = ex2_approx(-P.hl[c][k] * (float)(dxx + dyy));
            acc.add(W * e.y, e.x, dx, dy, dxx, dyy);
        } else {
            const double W = window_w<EXACT>(P, c, k, dx, dy, dxx, dyy);
            acc.add(W * (double)e.y, e.x, dx, dy, dxx, dyy);
        }
    });
}

// Variance of the constant term (ICI spec): v = sum w^2 var (phi . g)^2,
// with w^2 var = W^2/den for variance weights and W^2 for sigma weights.
template <int ORDER, bool EXACT, class Fetch>
__device__ __forceinline__ double fit_variance(const DevParams &P, int c, int k, double qx,
                                               double qy, Fetch fetch, const double *g) {
    const bool sig = P.use_sigma;
    double v = 0.0;
    sweep(P, c, qx, qy, P.r[c][k], P.r2[c][k], fetch,
          [&](float2 e, double dx, double dy, double dxx, double dyy) {
              const double W = window_w<EXACT>(P, c, k, dx, dy, dxx, dyy);
              const double t = sig ? W * W : W * W * (double)e.y;
              double pg = g[0];
              if (ORDER >= 1) pg += dx * g[1] + dy * g[2];
              if (ORDER >= 2) pg += dxx * g[3] + __dmul_rn(dx, dy) * g[4] + dyy * g[5];
              v = fma(t, pg * pg, v);
          });
    return v;
}

struct PixelResult {
    double val, gx, gy;
    int outcome;  // order*16 + radius step, or HDR_OUTCOME_NAN
    int sidx;
    int count;    // samples in the accepted window
};

__device__ __forceinline__ void write_result(const DevParams &P, int pix, int c,
                                             const PixelResult &R) {
    const double v = R.val;
    // np.maximum(val, 0).astype(float32) (lpa.py:428) keeps NaN
    const float o = (v != v) ? __int_as_float(0x7fc00000) : __double2float_rn(fmax(v, 0.0));
    P.rgb[(size_t)pix * 3 + c] = o;
    const size_t plane = (size_t)P.out_w * P.out_h;
    if (P.grad) {
        P.grad[(size_t)(2 * c) * plane + pix] = (float)R.gx;
        P.grad[(size_t)(2 * c + 1) * plane + pix] = (float)R.gy;
    }
    if (P.sidx) P.sidx[(size_t)c * plane + pix] = (uint8_t)R.sidx;
    if (P.outcome) P.outcome[(size_t)c * plane + pix] = (uint8_t)R.outcome;
    if (P.value) P.value[(size_t)c * plane + pix] = (float)v;
    if (P.count) P.count[(size_t)c * plane + pix] = (uint16_t)min(R.count, 65535);
}

// ---------------------------------------------------------------------------
// Exact evaluation (slow path): lpa_evaluate's ladder (_kernels.py:257-300)
// and the ICI rule, from global memory.
// ---------------------------------------------------------------------------
template <int ORDER, class Fetch>
__device__ bool ladder_order(const DevParams &P, int c, double qx, double qy, Fetch fetch,
                             PixelResult &R) {
    constexpr int PN = NC<ORDER>::P;
    double r = P.r[c][0];  // already min(r0, max_radius)
    int step = 0;
    AccFor<ORDER, true> acc;
    for (;;) {
        accumulate<ORDER, true>(P, c, 0, qx, qy, r, __dmul_rn(r, r), fetch, acc);
        Fit fit;
        if (solve_exact<PN>(acc, P.cond, fit) == FIT_OK) {
            R.count = acc.count;
            R.val = fit.c0;
            R.gx = ORDER >= 1 ? fit.c1 : __longlong_as_double(0x7ff8000000000000ll);
            R.gy = ORDER >= 1 ? fit.c2 : __longlong_as_double(0x7ff8000000000000ll);
            R.outcome = ORDER * 16 + (step < 15 ? step : 15);
            return true;
        }
        if (r >= P.max_radius * (1.0 - 1e-12)) return false;
        r = fmin(r * 1.5, P.max_radius);
        ++step;
    }
}

template <int ORDER, class Fetch>
__device__ void ladder(const DevParams &P, int c, double qx, double qy, Fetch fetch,
                       PixelResult &R) {
    R.sidx = 0;
    if (ladder_order<ORDER>(P, c, qx, qy, fetch, R)) return;
    if constexpr (ORDER >= 1) {
        if (ladder_order<ORDER - 1>(P, c, qx, qy, fetch, R)) return;
    }
    if constexpr (ORDER >= 2) {
        if (ladder_order<0>(P, c, qx, qy, fetch, R)) return;
    }
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    R.val = R.gx = R.gy = nan;
    R.outcome = HDR_OUTCOME_NAN;
    R.count = 0;
}

// ICI with a pluggable decision (fast: bounds, may return AMBIG; exact).
// Returns FIT_OK with R filled, FIT_FAIL if scale 0 fails (caller runs the
// ladder), FIT_AMBIG if a decision needs the exact path.
template <int ORDER, bool EXACT, class Fetch>
__device__ int ici(const DevParams &P, int c, double qx, double qy, Fetch fetch, PixelResult &R) {
    constexpr int PN = NC<ORDER>::P;
    AccFor<ORDER, EXACT> acc;
    Fit fit;
    double L = 0.0, U = 0.0;
    for (int k = 0; k < P.n_scales; ++k) {
        accumulate<ORDER, EXACT>(P, c, k, qx, qy, P.r[c][k], P.r2[c][k], fetch, acc);
        const int st = EXACT ? solve_exact<PN>(acc, P.cond, fit) : solve_fast<PN>(acc, P.cond, fit);
        if (st == FIT_AMBIG) return FIT_AMBIG;
        if (st != FIT_OK) {
            if (k == 0) return FIT_FAIL;
            break;  // invalid scale ends the search at k-1
        }
        const double sd = sqrt(fit_variance<ORDER, EXACT>(P, c, k, qx, qy, fetch, fit.g));
        const double lo = fit.c0 - P.gamma * sd, hi = fit.c0 + P.gamma * sd;
        if (k == 0) {
            L = lo;
            U = hi;
        } else {
            L = fmax(L, lo);
            U = fmin(U, hi);
            if (L > U) break;
        }
        R.val = fit.c0;
        R.gx = fit.c1;
        R.gy = fit.c2;
        R.sidx = k;
        R.count = acc.count;
    }
    if (ORDER == 0) R.gx = R.gy = __longlong_as_double(0x7ff8000000000000ll);
    R.outcome = ORDER * 16;
    return FIT_OK;
}

template <int ORDER>
__global__ void __launch_bounds__(128) lpa_slow_kernel(const __grid_constant__ DevParams P) {
    const uint32_t n = *P.work_count;
    auto fetch = [&](int s, int x, int y) { return radiance_sample(P.s[s], x, y, P.use_sigma); };
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t item = P.work_items[i];
        const int pix = (int)(item >> 2), c = (int)(item & 3);
        const int ox = pix % P.out_w, oy = pix / P.out_w;
        const double qx = qcoord(ox, P.sx), qy = qcoord(oy, P.sy);
        PixelResult R;
        if (P.n_scales > 1) {
            if (ici<ORDER, true>(P, c, qx, qy, fetch, R) != FIT_OK) ladder<ORDER>(P, c, qx, qy, fetch, R);
        } else {
            ladder<ORDER>(P, c, qx, qy, fetch, R);
        }
        write_result(P, pix, c, R);
    }
}

// ---------------------------------------------------------------------------
// Fast path
// ---------------------------------------------------------------------------
__device__ __forceinline__ void region_origin(const DevSensor &S, const DevParams &P, int tx0,
                                              int ty0, int tx1, int ty1, int &ox, int &oy) {
    // union of the window bboxes of the tile's corner queries at radius fast_R;
    // the bbox is affine in q, so its minimum is attained at a corner.
    int xmin = INT_MAX, ymin = INT_MAX;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double qx = qcoord((k & 1) ? tx1 : tx0, P.sx);
        const double qy = qcoord((k & 2) ? ty1 : ty0, P.sy);
        int xlo, xhi, ylo, yhi;
        window_bbox(S, qx, qy, P.fast_R, xlo, xhi, ylo, yhi);
        xmin = min(xmin, xlo);
        ymin = min(ymin, ylo);
    }
    ox = xmin & ~1;  // even, so phase = coordinate parity
    oy = ymin & ~1;
}

template <int ORDER, bool ICI>
__global__ void __launch_bounds__(NT, 2) lpa_fast_kernel(const __grid_constant__ DevParams P) {
    extern __shared__ float2 smem[];
    __shared__ int s_org[MAXS][2];
    constexpr int PN = NC<ORDER>::P;

    const int tile = blockIdx.x;
    const int tx0 = (tile % P.tiles_x) * TW;
    const int ty0 = P.row_begin + (tile / P.tiles_x) * TH;
    const int tx1 = min(tx0 + TW, P.out_w) - 1;
    const int ty1 = min(ty0 + TH, P.row_end) - 1;

    if (threadIdx.x < P.n_sensors) {
        int ox, oy;
        region_origin(P.s[threadIdx.x], P, tx0, ty0, tx1, ty1, ox, oy);
        s_org[threadIdx.x][0] = ox;
        s_org[threadIdx.x][1] = oy;
    }
    __syncthreads();

    // Stage raw footprint -> (f_hat, 1/den) in Bayer phase planes.
    for (int s = 0; s < P.n_sensors; ++s) {
        const DevSensor &S = P.s[s];
        const int ox = s_org[s][0], oy = s_org[s][1];
        const int rw = S.rw, rh = S.rh, pw = rw >> 1, plane = pw * (rh >> 1);
        float2 *base = smem + S.smem_off;
        for (int idx = threadIdx.x; idx < rw * rh; idx += NT) {
            const int ly = idx / rw, lx = idx - ly * rw;
            const float2 e = radiance_sample(S, ox + lx, oy + ly, P.use_sigma);
            base[((ly & 1) * 2 + (lx & 1)) * plane + (ly >> 1) * pw + (lx >> 1)] = e;
        }
    }
    __syncthreads();

    const int px = tx0 + (int)(threadIdx.x % TW);
    const int py = ty0 + (int)(threadIdx.x / TW);
    if (px >= P.out_w || py >= P.row_end) return;
    const int pix = py * P.out_w + px;
    const double qx = qcoord(px, P.sx), qy = qcoord(py, P.sy);

    // every window of this pixel must lie inside the staged region
    bool covered = true;
    for (int s = 0; s < P.n_sensors; ++s) {
        const DevSensor &S = P.s[s];
        int xlo, xhi, ylo, yhi;
        window_bbox(S, qx, qy, P.fast_R, xlo, xhi, ylo, yhi);
        covered &= xlo >= s_org[s][0] && ylo >= s_org[s][1] && xhi < s_org[s][0] + S.rw &&
                   yhi < s_org[s][1] + S.rh;
    }

    auto fetch = [&](int s, int x, int y) {
        const DevSensor &S = P.s[s];
        const int lx = x - s_org[s][0], ly = y - s_org[s][1];
        const int pw = S.rw >> 1;
        return smem[S.smem_off + ((y & 1) * 2 + (x & 1)) * (pw * (S.rh >> 1)) + (ly >> 1) * pw +
                    (lx >> 1)];
    };

    for (int c = 0; c < 3; ++c) {
        PixelResult R;
        R.sidx = 0;
        int st = FIT_AMBIG;
        if (covered) {
            if constexpr (ICI) {
                st = ici<ORDER, false>(P, c, qx, qy, fetch, R);
            } else {
                AccFor<ORDER, false> acc;
                accumulate<ORDER, false>(P, c, 0, qx, qy, P.r[c][0], P.r2[c][0], fetch, acc);
                Fit fit;
                st = solve_fast<PN>(acc, P.cond, fit);
                if (st == FIT_OK) {
                    R.count = acc.count;
                    R.val = fit.c0;
                    const double nan = __longlong_as_double(0x7ff8000000000000ll);
                    R.gx = ORDER >= 1 ? fit.c1 : nan;
                    R.gy = ORDER >= 1 ? fit.c2 : nan;
                    R.outcome = ORDER * 16;
                }
            }
        }
        if (st == FIT_OK) {
            write_result(P, pix, c, R);
        } else {
            const uint32_t slot = atomicAdd(P.work_count, 1u);
            P.work_items[slot] = ((uint32_t)pix << 2) | (uint32_t)c;
        }
    }
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

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
static int fill_sensor(const HdrSensor &h, DevSensor &d) {
    memset(&d, 0, sizeof(d));
    if (!h.raw || h.width <= 0 || h.height <= 0 || h.pitch < h.width) return HDR_ERR_ARG;
    if (!(h.exposure_time > 0) || !(h.gain > 0) || !isfinite(h.exposure_time) || !isfinite(h.gain))
        return HDR_ERR_ARG;  // check_positive (radiometry.py:55-56)
    if (!(h.exposure_scaling > 0 && h.exposure_scaling <= 1)) return HDR_ERR_CONFIG;
    const double *T = h.transform;
    const double det = T[0] * T[4] - T[1] * T[3];
    if (!(fabs(det) > 1e-9)) return HDR_ERR_CONFIG;  // radiometry.py:64-66
    if (h.saturation_level <= 0 || h.saturation_level > 65535) return HDR_ERR_CONFIG;
    for (int k = 0; k < 4; ++k)
        if (h.tile[k] < 0 || h.tile[k] > 2) return HDR_ERR_ARG;
    d.raw = h.raw;
    d.width = h.width;
    d.height = h.height;
    d.pitch = h.pitch;
    d.sat = h.saturation_level;
    for (int c = 0; c < 3; ++c) {
        d.phmask[c] = 0;
        for (int ph = 0; ph < 4; ++ph)
            if (h.tile[ph] == c) d.phmask[c] |= 1 << ph;
    }
    for (int k = 0; k < 6; ++k) d.T[k] = T[k];
    d.separable = (T[1] == 0.0 && T[3] == 0.0);
    d.N[0] = T[4] / det;
    d.N[1] = -T[1] / det;
    d.N[2] = -T[3] / det;
    d.N[3] = T[0] / det;
    d.nrow0 = sqrt(d.N[0] * d.N[0] + d.N[1] * d.N[1]);
    d.nrow1 = sqrt(d.N[2] * d.N[2] + d.N[3] * d.N[3]);
    d.bias = h.bias;
    d.readvar = h.readout_variance;
    d.nonuni = h.nonuniformity;
    d.bias_p = h.bias_plane;
    d.readvar_p = h.readvar_plane;
    d.nonuni_p = h.nonuni_plane;
    d.defective = h.defective;
    d.planes = (h.bias_plane || h.readvar_plane || h.nonuni_plane) ? 1 : 0;
    d.g = h.gain;
    d.t = h.exposure_time;
    d.n = h.exposure_scaling;
    if (!d.nonuni_p && !(h.nonuniformity > 0)) return HDR_ERR_CONFIG;
    if (!d.readvar_p && h.readout_variance < 0) return HDR_ERR_ARG;
    const double denom = h.gain * h.exposure_time * h.exposure_scaling * h.nonuniformity;
    if (!d.nonuni_p && (!(denom > 0) || !isfinite(denom))) return HDR_ERR_CONFIG;
    d.inv_denom = 1.0 / denom;
    d.inv_denom2 = 1.0 / (denom * denom);
    d.c_shot = h.gain * h.gain * h.exposure_time * h.nonuniformity * h.exposure_scaling;
    d.qv = (1.0 / 12.0) / (denom * denom);
    return HDR_OK;
}

static int set_smem_attr(const void *fn, int bytes) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    return e == cudaSuccess ? HDR_OK : HDR_ERR_CUDA;
}

template <int ORDER>
static int launch_all(const DevParams &P, int tiles, int smem_bytes, cudaStream_t st) {
    const void *fn = P.n_scales > 1 ? (const void *)lpa_fast_kernel<ORDER, true>
                                    : (const void *)lpa_fast_kernel<ORDER, false>;
    if (set_smem_attr(fn, smem_bytes) != HDR_OK) return HDR_ERR_CUDA;
    if (P.n_scales > 1)
        lpa_fast_kernel<ORDER, true><<<tiles, NT, smem_bytes, st>>>(P);
    else
        lpa_fast_kernel<ORDER, false><<<tiles, NT, smem_bytes, st>>>(P);
    if (cudaPeekAtLastError() != cudaSuccess) return HDR_ERR_CUDA;
    if (P.flags & HDR_FLAG_FAST_ONLY) return HDR_OK;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    lpa_slow_kernel<ORDER><<<nsm * 4, 128, 0, st>>>(P);
    if (cudaPeekAtLastError() != cudaSuccess) return HDR_ERR_CUDA;
    return HDR_OK;
}

}  // namespace hdrlpa

using namespace hdrlpa;

extern "C" {

static const size_t WS_HEADER = 256;

int hdr_lpa_abi_version(void) { return HDR_LPA_ABI_VERSION; }

const char *hdr_lpa_status_string(int status) {
    switch (status) {
        case HDR_OK: return "ok";
        case HDR_ERR_ARG: return "invalid argument";
        case HDR_ERR_CONFIG: return "invalid sensor configuration";
        case HDR_ERR_SHAPE: return "dimension mismatch";
        case HDR_ERR_WORKSPACE: return "workspace too small";
        case HDR_ERR_CUDA: return "CUDA error";
        default: return "unknown status";
    }
}

int hdr_lpa_workspace_bytes(int out_w, int out_h, size_t *bytes) {
    if (out_w <= 0 || out_h <= 0 || !bytes) return HDR_ERR_ARG;
    const size_t items = (size_t)out_w * out_h * 3;
    if ((size_t)out_w * out_h >= (1ull << 30)) return HDR_ERR_ARG;  // item packing
    *bytes = WS_HEADER + items * sizeof(uint32_t);
    return HDR_OK;
}

int hdr_lpa_reconstruct(const HdrSensor *sensors, int n_sensors, const HdrParams *params,
                        int out_w, int out_h, double ref_w, double ref_h, int row_begin,
                        int row_end, const HdrOutputs *out, void *workspace,
                        size_t workspace_bytes, void *stream) {
    if (!sensors || !params || !out || !out->rgb || !workspace) return HDR_ERR_ARG;
    if (n_sensors < 1 || n_sensors > MAXS) return HDR_ERR_ARG;
    if (out_w <= 0 || out_h <= 0 || !(ref_w > 0) || !(ref_h > 0)) return HDR_ERR_ARG;
    if (params->order < 0 || params->order > 2) return HDR_ERR_ARG;
    if (params->n_scales < 1 || params->n_scales > MAXJ) return HDR_ERR_ARG;
    if (params->weight_mode != HDR_WEIGHT_VARIANCE && params->weight_mode != HDR_WEIGHT_SIGMA)
        return HDR_ERR_ARG;
    if (!(params->max_radius > 0) || !(params->cond_threshold > 0)) return HDR_ERR_ARG;
    if (row_end <= 0 || row_end > out_h) row_end = out_h;
    if (row_begin < 0 || row_begin >= row_end) return HDR_ERR_ARG;
    size_t need = 0;
    if (hdr_lpa_workspace_bytes(out_w, out_h, &need) != HDR_OK) return HDR_ERR_ARG;
    if (workspace_bytes < need) return HDR_ERR_WORKSPACE;

    DevParams P;
    memset(&P, 0, sizeof(P));
    for (int s = 0; s < n_sensors; ++s) {
        const int rc = fill_sensor(sensors[s], P.s[s]);
        if (rc != HDR_OK) return rc;
    }
    P.n_sensors = n_sensors;
    P.order = params->order;
    P.n_scales = params->n_scales;
    P.use_sigma = params->weight_mode == HDR_WEIGHT_SIGMA;
    P.out_w = out_w;
    P.out_h = out_h;
    P.row_begin = row_begin;
    P.row_end = row_end;
    P.sx = ref_w / (double)out_w;
    P.sy = ref_h / (double)out_h;
    P.max_radius = params->max_radius;
    P.cond = params->cond_threshold;
    P.gamma = params->ici_gamma;
    double fastR = 0.0;
    for (int c = 0; c < 3; ++c)
        for (int k = 0; k < P.n_scales; ++k) {
            const double h = params->scale[c][k];
            if (!(h > 0) || !isfinite(h)) return HDR_ERR_ARG;
            double r = 3.0 * sqrt(h);  // SUPPORT_SIGMAS * sqrt(scale), lpa.py:37, :353
            if (r > P.max_radius) r = P.max_radius;
            P.r[c][k] = r;
            P.r2[c][k] = r * r;
            P.hl[c][k] = (float)(1.4426950408889634 / h);
            P.hinv[c][k] = 1.0 / h;  // iso Hinv = 1/scale (lpa.py:351)
            fastR = fmax(fastR, r);
        }
    P.fast_R = fastR;
    P.rgb = out->rgb;
    P.grad = out->grad;
    P.sidx = out->scale_idx;
    P.outcome = out->outcome;
    P.value = out->value;
    P.count = out->count;
    P.flags = params->flags;
    P.work_count = (uint32_t *)workspace;
    P.work_items = (uint32_t *)((char *)workspace + WS_HEADER);

    // staged region per sensor: tile extent in sensor space + 2 x window half-width
    int smem_f2 = 0;
    for (int s = 0; s < n_sensors; ++s) {
        DevSensor &d = P.s[s];
        const double ex = (TW - 1) * P.sx, ey = (TH - 1) * P.sy;
        const double wx = fabs(d.N[0]) * ex + fabs(d.N[1]) * ey + 2.0 * fastR * d.nrow0;
        const double wy = fabs(d.N[2]) * ex + fabs(d.N[3]) * ey + 2.0 * fastR * d.nrow1;
        int rw = (int)ceil(wx) + 8, rh = (int)ceil(wy) + 8;
        rw += rw & 1;
        rh += rh & 1;
        d.rw = rw;
        d.rh = rh;
        d.smem_off = smem_f2;
        smem_f2 += rw * rh;
    }
    const int smem_bytes = smem_f2 * (int)sizeof(float2);
    if (smem_bytes > 200 * 1024) return HDR_ERR_ARG;  // window too large for the staged path

    cudaStream_t st = (cudaStream_t)stream;
    const int tiles_y = (row_end - row_begin + TH - 1) / TH;
    P.tiles_x = (out_w + TW - 1) / TW;
    const int tiles = P.tiles_x * tiles_y;
    if (cudaMemsetAsync(workspace, 0, sizeof(uint32_t), st) != cudaSuccess) return HDR_ERR_CUDA;
    int rc;
    switch (P.order) {
        case 0: rc = launch_all<0>(P, tiles, smem_bytes, st); break;
        case 1: rc = launch_all<1>(P, tiles, smem_bytes, st); break;
        default: rc = launch_all<2>(P, tiles, smem_bytes, st); break;
    }
    return rc;
}

int hdr_saturation_mask(const HdrSensor *sensor, uint32_t *out_bits, int words_per_row,
                        void *stream) {
    if (!sensor || !out_bits) return HDR_ERR_ARG;
    DevSensor d;
    const int rc = fill_sensor(*sensor, d);
    if (rc != HDR_OK) return rc;
    if (words_per_row < (d.width + 31) / 32) return HDR_ERR_SHAPE;
    dim3 grid((d.width + 255) / 256, d.height);
    saturation_mask_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(d, out_bits, words_per_row);
    return cudaPeekAtLastError() == cudaSuccess ? HDR_OK : HDR_ERR_CUDA;
}

int hdr_radiance_planes(const HdrSensor *sensor, int weight_mode, float *value, float *inv_den,
                        void *stream) {
    if (!sensor || !value || !inv_den) return HDR_ERR_ARG;
    if (weight_mode != HDR_WEIGHT_VARIANCE && weight_mode != HDR_WEIGHT_SIGMA) return HDR_ERR_ARG;
    DevSensor d;
    const int rc = fill_sensor(*sensor, d);
    if (rc != HDR_OK) return rc;
    dim3 grid((d.width + 255) / 256, d.height);
    radiance_planes_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
        d, weight_mode == HDR_WEIGHT_SIGMA, value, inv_den);
    return cudaPeekAtLastError() == cudaSuccess ? HDR_OK : HDR_ERR_CUDA;
}

int hdr_fp64_peak_probe(double *flops_per_s, void *stream) {
    if (!flops_per_s) return HDR_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    double *sink = nullptr;
    if (cudaMalloc(&sink, 256 * sizeof(double)) != cudaSuccess) return HDR_ERR_CUDA;
    const int blocks = nsm * 8, iters = 1 << 15;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    fp64_probe_kernel<<<blocks, 256, 0, st>>>(sink, iters / 8, 0.999999, 1e-7);  // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0, st);
        fp64_probe_kernel<<<blocks, 256, 0, st>>>(sink, iters, 0.999999, 1e-7);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        best = fminf(best, ms);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    if (cudaGetLastError() != cudaSuccess) return HDR_ERR_CUDA;
    *flops_per_s = (double)blocks * 256 * iters * 8 * 2 / (best * 1e-3);
    return HDR_OK;
}

int hdr_lpa_slow_items(const void *workspace, uint32_t *count, void *stream) {
    if (!workspace || !count) return HDR_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemcpyAsync(count, workspace, sizeof(uint32_t), cudaMemcpyDeviceToHost, st) !=
        cudaSuccess)
        return HDR_ERR_CUDA;
    return cudaStreamSynchronize(st) == cudaSuccess ? HDR_OK : HDR_ERR_CUDA;
}

}  // extern "C"
