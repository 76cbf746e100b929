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
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <atomic>
#include <climits>
#include <type_traits>
#include <math.h>
#include <vector>
#include <stdio.h>
#include <string.h>

#include "hdr_lpa.h"
#include "lpa_device.cuh"

namespace hdrlpa {

constexpr int TW = 32, TH = 8, NT = TW * TH;  // NT consumer threads, one per tile pixel

// workspace layout: [header: work counter][pre-computed taps][work items]
static const size_t WS_HEADER = 256;
// Order-2 tile sweeps: skip samples outside the disk with branches (1) or
// accumulate them with zero weight (0; the row-factored moments make a
// sample cheap enough that divergent branches cost more than they save)
#ifndef HDR_BRANCHY_O2
#define HDR_BRANCHY_O2 1
#endif
static_assert(sizeof(DevParams) + TAP_PARAM_BYTES <= 32764, "kernel parameter space");
// plane buffers per CTA of the fast kernel's staging pipeline (measured: 3
// buffers gain nothing on cfg2 and cost cfg3 5% through occupancy)
#ifndef HDR_NBUF
#define HDR_NBUF 2
#endif
constexpr int NBUF = HDR_NBUF;
static const size_t LUT_BYTES = 65536 * sizeof(double2);
static const size_t RT_TABLE_BYTES = 64 * 1024;  // row-tap table (workspace, then shared memory)

template <int ORDER>
struct NC {
    static constexpr int P = (ORDER + 1) * (ORDER + 2) / 2;
};

// ---------------------------------------------------------------------------
// Window sweeps.  A sweep enumerates the samples of one channel inside the
// support disk |X - q| <= r, in the order (sensor, Bayer phase, row, column),
// and calls body(value, 1/den, dx, dy, dx^2, dy^2, |d|^2 as fp32) for each
// (value and 1/den: fp32 in the tile sweeps, float64 in the global sweep).
// Offsets and the membership test are float64 in the reference's exact
// operation order (radiometry.py:84, _kernels.py:160-163), so both sweeps
// below select exactly the reference's sample set in the same order.
// ---------------------------------------------------------------------------

// Slow path: straight from the raw frames in global memory, float64 radiometry.
// LANES > 1: the candidates of every window are split over an aligned group
// of LANES lanes of a warp (candidate j -> group lane j % LANES) and the sums
// are combined by a butterfly reduction, after which every lane of the group
// holds bitwise-identical totals.  Groups of one warp may diverge.
template <int LANES>
struct GlobalSweep {
    const DevParams &P;
    double qx, qy;
    __device__ __forceinline__ static unsigned group_mask() {
        if constexpr (LANES >= 32)
            return 0xffffffffu;
        else
            return ((1u << LANES) - 1u) << ((threadIdx.x & 31) & ~(LANES - 1));
    }
    template <int PN>
    __device__ __forceinline__ void reduce(Acc<PN> &acc) const {
        if constexpr (LANES > 1) {
            const unsigned mask = group_mask();
#pragma unroll
            for (int m = LANES / 2; m >= 1; m >>= 1) {
#pragma unroll
                for (int i = 0; i < Acc<PN>::NS; ++i) acc.A[i] += __shfl_xor_sync(mask, acc.A[i], m);
#pragma unroll
                for (int i = 0; i < PN; ++i) acc.b[i] += __shfl_xor_sync(mask, acc.b[i], m);
                acc.count += __shfl_xor_sync(mask, acc.count, m);
            }
        }
    }
    __device__ __forceinline__ double reduce(double v) const {
        if constexpr (LANES > 1) {
            const unsigned mask = group_mask();
#pragma unroll
            for (int m = LANES / 2; m >= 1; m >>= 1) v += __shfl_xor_sync(mask, v, m);
        }
        return v;
    }
    template <class Body>
    __device__ __forceinline__ void operator()(int c, int /*k*/, double r, double r2,
                                               Body body) const {
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
                const int nrow = yhi >= ys ? ((yhi - ys) >> 1) + 1 : 0;
                const int ncol = xhi >= xs ? ((xhi - xs) >> 1) + 1 : 0;
                const int lane = LANES > 1 ? (int)(threadIdx.x & (LANES - 1)) : 0;
                for (int j = lane; j < nrow * ncol; j += LANES) {
                    const int y = ys + 2 * (j / ncol), x = xs + 2 * (j % ncol);
                    const double yd = (double)y;
                    const double t1y = __dmul_rn(T1, yd), t4y = __dmul_rn(T4, yd);
                    double f, iv;  // float64 radiometry straight from the raw frame
                    if (!radiance_exact(S, x, y, P.use_sigma, f, iv)) continue;
                    const double xd = (double)x;
                    const double X = __dadd_rn(__dadd_rn(__dmul_rn(T0, xd), t1y), T2);
                    const double Y = __dadd_rn(__dadd_rn(__dmul_rn(T3, xd), t4y), T5);
                    const double dx = __dsub_rn(X, qx), dy = __dsub_rn(Y, qy);
                    const double dxx = __dmul_rn(dx, dx), dyy = __dmul_rn(dy, dy);
                    const double d2 = __dadd_rn(dxx, dyy);
                    if (d2 > r2) continue;  // _kernels.py:162
                    body(true, f, iv, dx, dy, dxx, dyy, (float)d2);
                }
            }
        }
    }
};

// Adapter: a per-sample body as a traversal policy (no row hooks).
template <class Body>
struct PerSample {
    Body &body;
    __device__ __forceinline__ void begin_row(double, double) {}
    __device__ __forceinline__ void end_row(double, double) {}
    __device__ __forceinline__ void sample(bool ok, double v, float iv, double dx, double dy,
                                           double dxx, double dyy, float d2f) {
        body(ok, v, iv, dx, dy, dxx, dyy, d2f);
    }
    __device__ __forceinline__ void general(bool ok, double v, float iv, double dx, double dy,
                                            double dxx, double dyy, float d2f) {
        body(ok, v, iv, dx, dy, dxx, dyy, d2f);
    }
};

template <int MAXC, bool BRANCHY, bool RT = false>
struct TileSweep {
    const DevParams &P;
    const unsigned char *sm;
    const int (*org)[2];
    double qx, qy;
    int px, py;                 // the output pixel (RT: parity class, phase-plane base)
    const unsigned char *rt;    // RT: row-tap table in shared memory (rows, then taps)
    template <int PN>
    __device__ __forceinline__ void reduce(Acc<PN> &) const {}
    __device__ __forceinline__ double reduce(double v) const { return v; }
    // Per-sample traversal (same interface as GlobalSweep).
    template <class Body>
    __device__ __forceinline__ void operator()(int c, int k, double r, double r2, Body body) const {
        PerSample<Body> pol{body};
        rows(c, k, r, r2, pol);
    }

    // RT: the pre-computed rows of a translation-only sensor at scale k (all
    // taps inside r_k by construction; masked samples contribute weight 0).
    template <class Pol>
    __device__ __forceinline__ void tap_rows(int s, int c, int k, Pol &pol) const {
        const DevSensor &S = P.s[s];
        const int pm = P.rt_period - 1;
        const int cls = (py & pm) * P.rt_period + (px & pm);
        const RtHeader &hd = *(const RtHeader *)rt;
        const int r0 = hd.row0[s][c][cls], nr = hd.nrow[s][c][cls];
        const TapRow *rows = (const TapRow *)(rt + sizeof(RtHeader));
        const RowTap *taps =
            (const RowTap *)(rt + sizeof(RtHeader) + (size_t)hd.n_rows * sizeof(TapRow));
        const int pw = S.rw >> 1;
        // the pixel's anchor: its own sensor pixel (sx = 1) or cell (sx = 1/2)
        const int ax = px >> P.rt_shift, ay = py >> P.rt_shift;
        const unsigned char *vb = sm + S.off_vi +
                                  8 * (((ay - org[s][1]) >> 1) * pw + ((ax - org[s][0]) >> 1));
        for (int ri = r0; ri < r0 + nr; ++ri) {
            const TapRow &R = rows[ri];
            const int lo = R.lo[k], hi = R.hi[k];
            if (lo >= hi) continue;
            const double dy = R.dy, dyy = dy * dy;
            pol.begin_row(dy, dyy);
            for (int t = R.first + lo; t < R.first + hi; ++t) {
                const RowTap T = taps[t];
                const float2 e = *(const float2 *)(vb + T.off);
                pol.sample(e.y > 0.f, (double)e.x, e.y, T.dx, dy, T.dx * T.dx, dyy, T.d2f);
            }
            pol.end_row(dy, dyy);
        }
    }

    // Traversal with row hooks: for separable sensors every sample of a row
    // shares dy, so a policy can accumulate per-row sums (begin_row / sample /
    // end_row); rotated sensors go through pol.general() per sample.
    template <class Pol>
    __device__ __forceinline__ void rows(int c, int k, double r, double r2, Pol &pol) const {
        for (int s = 0; s < P.n_sensors; ++s) {
            const DevSensor &S = P.s[s];
            const int pm = S.phmask[c];
            if (!pm) continue;
            if constexpr (RT) {
                // RT mode: every separable sensor is translation-only and tapped
                if (S.separable) {
                    tap_rows(s, c, k, pol);
                    continue;
                }
            }
            const int ox = org[s][0], oy = org[s][1];
            const float2 *vi = (const float2 *)(sm + S.off_vi);
            const double *tx0 = (const double *)(sm + S.off_tx0);
            const double *ty4 = (const double *)(sm + S.off_ty4);
            const int pw = S.rw >> 1, plane = pw * (S.rh >> 1);
            int xlo, xhi, ylo, yhi;
            window_bbox(S, qx, qy, r, xlo, xhi, ylo, yhi);
            if (!RT && S.separable) {
                for (int ph = 0; ph < 4; ++ph) {
                    if (!((pm >> ph) & 1)) continue;
                    const int py = ph >> 1, px = ph & 1;
                    const int ys = ylo + ((py - ylo) & 1);
                    const int xs0 = xlo + ((px - xlo) & 1);
                    const int nc = xhi >= xs0 ? ((xhi - xs0) >> 1) + 1 : 0;
                    for (int c0 = 0; c0 < nc; c0 += MAXC) {
                        const int xs = xs0 + 2 * c0;
                        double cdx[MAXC], cdxx[MAXC];
#pragma unroll
                        for (int i = 0; i < MAXC; ++i) {
                            if (c0 + i < nc) {
                                cdx[i] = __dsub_rn(tx0[xs + 2 * i - ox], qx);  // X(x) - qx
                                cdxx[i] = __dmul_rn(cdx[i], cdx[i]);
                            } else {
                                // finite sentinel: never inside, and 0 * phi stays 0
                                cdx[i] = 0.0;
                                cdxx[i] = 1e150;  // (1e150)^2 stays finite: 0 * dx^4 = 0
                            }
                        }
                        const int colbase = ph * plane + ((xs - ox) >> 1);
                        for (int y = ys; y <= yhi; y += 2) {
                            const int ly = y - oy;
                            const double dy = __dsub_rn(ty4[ly], qy);  // Y(y) - qy
                            const double dyy = __dmul_rn(dy, dy);
                            if (dyy > r2) continue;
                            const int rb = colbase + (ly >> 1) * pw;
                            pol.begin_row(dy, dyy);
                            // orders 0-1: branch-free over the row (candidates outside the
                            // disk or without a sample contribute with weight 0); order 2
                            // (27 DFMA per sample) only visits the samples inside.
#pragma unroll
                            for (int i = 0; i < MAXC; ++i) {
                                const double d2 = __dadd_rn(cdxx[i], dyy);
                                if constexpr (BRANCHY) {
                                    if (d2 <= r2) {
                                        const float2 e = vi[rb + i];
                                        if (e.y > 0.f)
                                            pol.sample(true, (double)e.x, e.y, cdx[i], dy, cdxx[i],
                                                       dyy, (float)d2);
                                    }
                                } else {
                                    const float2 e = vi[rb + i];
                                    const bool ok = (d2 <= r2) && (e.y > 0.f);
                                    pol.sample(ok, (double)e.x, e.y, cdx[i], dy, cdxx[i], dyy,
                                               (float)d2);
                                }
                            }
                            pol.end_row(dy, dyy);
                        }
                    }
                }
            } else {
                const double *tx3 = (const double *)(sm + S.off_tx3);
                const double *ty1 = (const double *)(sm + S.off_ty1);
                const double T2 = S.T[2], T5 = S.T[5];
                // sensor-space position of q relative to the bbox corner (fp32 pre-test)
                const double u = qx - T2, v = qy - T5;
                const float fcx = (float)(S.N[0] * u + S.N[1] * v - (double)xlo);
                const float fcy = (float)(S.N[2] * u + S.N[3] * v - (double)ylo);
                const float r2hi = (float)r2 + 1e-3f;
                const float a0 = S.Tf[0], a1 = S.Tf[1], a3 = S.Tf[2], a4 = S.Tf[3];
                for (int ph = 0; ph < 4; ++ph) {
                    if (!((pm >> ph) & 1)) continue;
                    const int py = ph >> 1, px = ph & 1;
                    const int ys = ylo + ((py - ylo) & 1), xs = xlo + ((px - xlo) & 1);
                    float ey = (float)(ys - ylo) - fcy;
                    for (int y = ys; y <= yhi; y += 2, ey += 2.f) {
                        const int ly = y - oy;
                        const double t1y = ty1[ly], t4y = ty4[ly];
                        const int rb = ph * plane + (ly >> 1) * pw - (ox >> 1);
                        float ex = (float)(xs - xlo) - fcx;
                        for (int x = xs; x <= xhi; x += 2, ex += 2.f) {
                            const float fx = fmaf(a0, ex, a1 * ey), fy = fmaf(a3, ex, a4 * ey);
                            if (fmaf(fx, fx, fy * fy) > r2hi) continue;
                            const int k = rb + (x >> 1);
                            const float2 e = vi[k];
                            if (!(e.y > 0.f)) continue;
                            const int lx = x - ox;
                            const double X = __dadd_rn(__dadd_rn(tx0[lx], t1y), T2);
                            const double Y = __dadd_rn(__dadd_rn(tx3[lx], t4y), T5);
                            const double dx = __dsub_rn(X, qx), dy = __dsub_rn(Y, qy);
                            const double dxx = __dmul_rn(dx, dx), dyy = __dmul_rn(dy, dy);
                            const double d2 = __dadd_rn(dxx, dyy);
                            if (d2 > r2) continue;
                            pol.general(true, (double)e.x, e.y, dx, dy, dxx, dyy, (float)d2);
                        }
                    }
                }
            }
        }
    }
};

// Window weight (_kernels.py:164-168) W = exp(-dX^T Hinv dX), Hinv = I/h.
// Fast path: fp32 MUFU ex2 (q <= 9 at the base/ICI radii).  Exact path:
// float64 exp in the reference's operation order, because the radius ladder
// reaches q ~ 1e2 where fp32 would underflow.
template <bool EXACT>
__device__ __forceinline__ double window_w(const DevParams &P, int c, int k, double dx, double dy,
                                           float d2f) {
    if constexpr (EXACT) {
        const double hi = P.hinv[c][k];
        const double q = __dadd_rn(__dmul_rn(__dmul_rn(hi, dx), dx), __dmul_rn(__dmul_rn(hi, dy), dy));
        return exp(-q);
    } else {
        return (double)ex2_approx(-P.hl[c][k] * d2f);
    }
}

// Row-factored moments (fast path, separable sensors).  Along a sensor row
// dy is constant, so with phi_a = dx^i_a dy^j_a the row contributes
//   A_ab += dy^(j_a+j_b) * S_(i_a+i_b),  b_a += dy^j_a * T_i_a,
//   S_n = sum w dx^n (n <= 2*ORDER),  T_n = sum w y dx^n (n <= ORDER),
// i.e. 2*ORDER+1 + ORDER+1 sums per sample instead of P(P+1)/2 + P.
// Rotated sensors accumulate per sample.
template <int ORDER>
struct RowMoments {
    static constexpr int PN = NC<ORDER>::P;
    Acc<PN> &acc;
    float hl;
    double S[2 * ORDER + 1], T[ORDER + 1];
    int cnt;
    __device__ __forceinline__ void begin_row(double, double) {
#pragma unroll
        for (int n = 0; n <= 2 * ORDER; ++n) S[n] = 0.0;
#pragma unroll
        for (int n = 0; n <= ORDER; ++n) T[n] = 0.0;
        cnt = 0;
    }
    __device__ __forceinline__ void sample(bool ok, double v, float iv, double dx, double,
                                           double dxx, double, float d2f) {
        const float w32 = ok ? ex2_approx(-hl * d2f) * iv : 0.f;
        const double w = (double)w32, y = ok ? v : 0.0;
        acc.sabs = fmaf(w32, fabsf((float)y), acc.sabs);
        // w dx^n from independent products (dx^2 is the cached column square):
        // dependency depth 2 instead of a 2*ORDER-long multiply chain
        double p[5];
        p[0] = w;
        if (ORDER >= 1) {
            p[1] = w * dx;
            p[2] = w * dxx;
        }
        if (ORDER >= 2) {
            p[3] = w * (dx * dxx);
            p[4] = w * (dxx * dxx);
        }
#pragma unroll
        for (int n = 0; n <= 2 * ORDER; ++n) {
            S[n] += p[n];
            if (n <= ORDER) T[n] = fma(p[n], y, T[n]);
        }
        cnt += ok ? 1 : 0;
    }
    __device__ __forceinline__ void end_row(double dy, double dyy) {
        double dp[5];
        dp[0] = 1.0;
        dp[1] = dy;
        dp[2] = dyy;
        dp[3] = dyy * dy;
        dp[4] = dyy * dyy;
#pragma unroll
        for (int a = 0; a < PN; ++a) {
            const int ia = basis_i(a), ja = basis_j(a);
            acc.b[a] = (ja == 0) ? acc.b[a] + T[ia] : fma(T[ia], dp[ja], acc.b[a]);
        }
        if constexpr (Acc<PN>::MOM) {
            // moments M_ij += S_i dy^j, i + j <= 2 ORDER
#pragma unroll
            for (int d = 0; d <= 2 * ORDER; ++d)
#pragma unroll
                for (int j = 0; j <= d; ++j) {
                    const int k = midx(d - j, j);
                    acc.A[k] = j == 0 ? acc.A[k] + S[d - j] : fma(S[d - j], dp[j], acc.A[k]);
                }
        } else {
            int k = 0;
#pragma unroll
            for (int a = 0; a < PN; ++a) {
#pragma unroll
                for (int bb = a; bb < PN; ++bb) {
                    const int ii = basis_i(a) + basis_i(bb), jj = basis_j(a) + basis_j(bb);
                    acc.A[k] = jj == 0 ? acc.A[k] + S[ii] : fma(S[ii], dp[jj], acc.A[k]);
                    ++k;
                }
            }
        }
        acc.count += cnt;
    }
    __device__ __forceinline__ void general(bool ok, double v, float iv, double dx, double dy,
                                            double dxx, double dyy, float d2f) {
        const float w = ok ? ex2_approx(-hl * d2f) * iv : 0.f;
        const double y = ok ? v : 0.0;
        acc.sabs = fmaf(w, fabsf((float)y), acc.sabs);
        acc.add((double)w, y, dx, dy, dxx, dyy, ok ? 1 : 0);
    }
};

// Row-factored variance sweep (ICI, fast path): phi.g = c0(dy) + dx (c1(dy) + g3 dx).
// Also accumulates T = sum w |phi.g| |y| (fp32): the sharp precision bound of
// c0 (fit_precise_sharp).
template <int ORDER>
struct RowVariance {
    const double *g;
    float hl;
    bool sig;
    double v, c0, c1;
    float T;
    __device__ __forceinline__ void begin_row(double dy, double dyy) {
        c0 = g[0];
        c1 = 0.0;
        if (ORDER >= 1) {
            c0 += g[2] * dy;
            c1 = g[1];
        }
        if (ORDER >= 2) {
            c0 += g[5] * dyy;
            c1 += g[4] * dy;
        }
    }
    __device__ __forceinline__ void end_row(double, double) {}
    __device__ __forceinline__ void sample(bool ok, double y, float iv, double dx, double, double,
                                           double, float d2f) {
        const float W = ok ? ex2_approx(-hl * d2f) : 0.f;
        const double t = (double)(sig ? W * W : W * W * iv);
        double pg = c0;
        if (ORDER == 1) pg = fma(dx, c1, c0);
        if (ORDER == 2) pg = fma(dx, fma(g[3], dx, c1), c0);
        if (ok) {
            v = fma(t, pg * pg, v);
            T = fmaf(W * iv, fabsf((float)pg) * fabsf((float)y), T);
        }
    }
    __device__ __forceinline__ void general(bool ok, double y, float iv, double dx, double dy,
                                            double dxx, double dyy, float d2f) {
        const float W = ok ? ex2_approx(-hl * d2f) : 0.f;
        const double t = (double)(sig ? W * W : W * W * iv);
        double pg = g[0];
        if (ORDER >= 1) pg += dx * g[1] + dy * g[2];
        if (ORDER >= 2) pg += dxx * g[3] + __dmul_rn(dx, dy) * g[4] + dyy * g[5];
        if (ok) {
            v = fma(t, pg * pg, v);
            T = fmaf(W * iv, fabsf((float)pg) * fabsf((float)y), T);
        }
    }
};

template <class Sweep>
struct HasRows {
    static constexpr bool value = false;
};
template <int MAXC, bool BRANCHY, bool RT>
struct HasRows<TileSweep<MAXC, BRANCHY, RT>> {
    static constexpr bool value = true;
};

template <int ORDER, bool EXACT, class Sweep>
__device__ __forceinline__ void accumulate(const DevParams &P, int c, int k, double r, double r2,
                                           const Sweep &sweep, Acc<NC<ORDER>::P> &acc) {
    if constexpr (!EXACT && ORDER >= 1 && HasRows<Sweep>::value) {
        acc.zero();
        RowMoments<ORDER> pol{acc, P.hl[c][k]};
        sweep.rows(c, k, r, r2, pol);
        return;
    }
    acc.zero();
    if constexpr (EXACT) {
        const double hi = P.hinv[c][k];
        sweep(c, k, r, r2, [&](bool, double v, auto iv, double dx, double dy, double dxx, double dyy,
                            float) {
            const double q =
                __dadd_rn(__dmul_rn(__dmul_rn(hi, dx), dx), __dmul_rn(__dmul_rn(hi, dy), dy));
            acc.add(exp(-q) * (double)iv, v, dx, dy, dxx, dyy);
        });
        sweep.reduce(acc);
    } else {
        const float hl = P.hl[c][k];
        sweep(c, k, r, r2, [&](bool ok, double v, float iv, double dx, double dy, double dxx,
                            double dyy, float d2f) {
            const float w = ok ? ex2_approx(-hl * d2f) * iv : 0.f;  // w = W / den
            const double y = ok ? v : 0.0;
            acc.sabs = fmaf(w, fabsf((float)y), acc.sabs);
            acc.add((double)w, y, dx, dy, dxx, dyy, ok ? 1 : 0);
        });
    }
}

// Variance of the constant term (ICI spec): v = sum w^2 var (phi . g)^2,
// with w^2 var = W^2/den for variance weights and W^2 for sigma weights.
template <int ORDER, bool EXACT, class Sweep>
__device__ __forceinline__ double fit_variance(const DevParams &P, int c, int k, const Sweep &sweep,
                                               const double *g, float *tsum = nullptr) {
    if constexpr (!EXACT && ORDER >= 1 && HasRows<Sweep>::value) {
        RowVariance<ORDER> pol{g, P.hl[c][k], (bool)P.use_sigma, 0.0, 0.0, 0.0, 0.f};
        sweep.rows(c, k, P.r[c][k], P.r2[c][k], pol);
        if (tsum) *tsum = pol.T;
        return pol.v;
    }
    const bool sig = P.use_sigma;
    const double hi = P.hinv[c][k];
    const float hl = P.hl[c][k];
    const double g0 = g[0], g1 = g[1], g2 = g[2], g3 = g[3], g4 = g[4], g5 = g[5];
    double v = 0.0;
    float T = 0.f;
    sweep(c, k, P.r[c][k], P.r2[c][k],
          [&](bool ok, double y, auto iv, double dx, double dy, double dxx, double dyy, float d2f) {
              double t;
              if constexpr (EXACT) {
                  const double q = __dadd_rn(__dmul_rn(__dmul_rn(hi, dx), dx),
                                             __dmul_rn(__dmul_rn(hi, dy), dy));
                  const double W = exp(-q);
                  t = sig ? W * W : W * W * (double)iv;
              } else {
                  const float W = ok ? ex2_approx(-hl * d2f) : 0.f;
                  t = (double)(sig ? W * W : W * W * iv);
              }
              double pg = g0;
              if (ORDER >= 1) pg += dx * g1 + dy * g2;
              if (ORDER >= 2) pg += dxx * g3 + __dmul_rn(dx, dy) * g4 + dyy * g5;
              if (ok) v = fma(t, pg * pg, v);  // select: unused columns carry sentinels
              if constexpr (!EXACT) {
                  const float W = ok ? ex2_approx(-hl * d2f) : 0.f;
                  if (ok) T = fmaf(W * (float)iv, fabsf((float)pg) * fabsf((float)y), T);
              }
          });
    if (tsum) *tsum = T;
    return sweep.reduce(v);
}

struct PixelResult {
    double val, gx, gy;
    int outcome;  // order*16 + radius step, or HDR_OUTCOME_NAN
    int sidx;
    int count;     // samples in the accepted window
    int work = 0;  // inside-window samples over every moment sweep evaluated
};

__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000ll); }

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
    if (P.work) P.work[(size_t)c * plane + pix] = (uint32_t)R.work;
}

// ---------------------------------------------------------------------------
// Exact evaluation (slow path): lpa_evaluate's ladder (_kernels.py:257-300)
// and the ICI rule.
// ---------------------------------------------------------------------------
template <int ORDER, class Sweep>
__device__ bool ladder_order(const DevParams &P, int c, const Sweep &sweep, PixelResult &R) {
    constexpr int PN = NC<ORDER>::P;
    double r = P.r[c][0];  // already min(r0, max_radius)
    int step = 0;
    Acc<PN> acc;
    for (;;) {
        accumulate<ORDER, true>(P, c, 0, r, __dmul_rn(r, r), sweep, acc);
        R.work += acc.count;
        Fit fit;
        if (solve_exact<PN>(acc, P.cond, fit) == FIT_OK) {
            R.count = acc.count;
            R.val = fit.c0;
            R.gx = ORDER >= 1 ? fit.c1 : qnan();
            R.gy = ORDER >= 1 ? fit.c2 : qnan();
            R.outcome = ORDER * 16 + (step < 15 ? step : 15);
            return true;
        }
        if (r >= P.max_radius * (1.0 - 1e-12)) return false;
        r = fmin(r * 1.5, P.max_radius);
        ++step;
    }
}

template <int ORDER, class Sweep>
__device__ void ladder(const DevParams &P, int c, const Sweep &sweep, PixelResult &R) {
    R.sidx = 0;
    if (ladder_order<ORDER>(P, c, sweep, R)) return;
    if constexpr (ORDER >= 1) {
        if (ladder_order<ORDER - 1>(P, c, sweep, R)) return;
    }
    if constexpr (ORDER >= 2) {
        if (ladder_order<0>(P, c, sweep, R)) return;
    }
    R.val = R.gx = R.gy = qnan();
    R.outcome = HDR_OUTCOME_NAN;
    R.count = 0;
}

// ICI with a pluggable decision: fast (condition
// bounds; may return AMBIG) or exact.  Returns FIT_OK with R filled, FIT_FAIL
// if scale 0 fails (the caller runs the ladder), FIT_AMBIG if a decision
// needs the exact path.
template <int ORDER, bool EXACT, class Sweep>
__device__ int ici(const DevParams &P, int c, const Sweep &sweep, PixelResult &R) {
    constexpr int PN = NC<ORDER>::P;
    Acc<PN> acc;
    Fit fit;
    double L = 0.0, U = 0.0, eL = 0.0, eU = 0.0;  // running bounds and their error bounds
    bool precise = true;
    for (int k = 0; k < P.n_scales; ++k) {
        accumulate<ORDER, EXACT>(P, c, k, P.r[c][k], P.r2[c][k], sweep, acc);
        R.work += acc.count;
        const int st = EXACT ? solve_exact<PN>(acc, P.cond, fit) : solve_fast<PN>(acc, P.cond, fit);
        if (st == FIT_AMBIG) return FIT_AMBIG;
        if (st != FIT_OK) {
            if (k == 0) return FIT_FAIL;
            break;  // an invalid scale ends the search at k-1
        }
        float tk = 0.f;
        const double sd = sqrt(fit_variance<ORDER, EXACT>(P, c, k, sweep, fit.g, &tk));
        const double lo = fit.c0 - P.gamma * sd, hi = fit.c0 + P.gamma * sd;
        // fast path: error bound of lo/hi (fp32 rounding of c0: fit_precise_sharp;
        // of sd: ICI_SD_EPS relative) -- an intersection test closer than the
        // bounds is decided by the exact path, so scale indices stay exact
        const double ek = EXACT ? 0.0 : 2.0 * FAST_EPS * (double)tk + P.gamma * sd * ICI_SD_EPS;
        if (k == 0) {
            L = lo;
            U = hi;
            eL = eU = ek;
        } else {
            if (lo >= L) eL = lo > L ? ek : fmax(eL, ek);
            if (hi <= U) eU = hi < U ? ek : fmax(eU, ek);
            L = fmax(L, lo);
            U = fmin(U, hi);
            if (!EXACT && fabs(L - U) <= eL + eU) return FIT_AMBIG;
            if (L > U) break;
        }
        R.val = fit.c0;
        R.gx = fit.c1;
        R.gy = fit.c2;
        R.sidx = k;
        R.count = acc.count;
        if constexpr (!EXACT) precise = fit_precise_sharp(fit.c0, tk, P.prec_floor);
    }
    if (!precise) return FIT_PREC;  // selected estimate too close to fp32 rounding limits
    if (ORDER == 0) R.gx = R.gy = qnan();
    R.outcome = ORDER * 16;
    return FIT_OK;
}

// Float64 recomputation of a fit whose fast-path decisions (validity, ICI
// scale) were sound but whose value failed fit_precise: exact weights and
// values at scale k.  False if the exact solve disagrees (then the caller
// runs the full exact evaluation).
template <int ORDER, class Sweep>
__device__ bool precise_fit(const DevParams &P, int c, int k, const Sweep &sweep, PixelResult &R) {
    constexpr int PN = NC<ORDER>::P;
    Acc<PN> acc;
    accumulate<ORDER, true>(P, c, k, P.r[c][k], P.r2[c][k], sweep, acc);
    R.work += acc.count;
    Fit fit;
    if (solve_fast<PN>(acc, P.cond, fit) != FIT_OK) return false;
    R.val = fit.c0;
    R.gx = ORDER >= 1 ? fit.c1 : qnan();
    R.gy = ORDER >= 1 ? fit.c2 : qnan();
    R.sidx = k;
    R.outcome = ORDER * 16;
    R.count = acc.count;
    return true;
}

// One group of SLOW_LANES lanes per work item: they share every window's
// candidates.
#ifndef SLOW_LANES
#define SLOW_LANES 8
#endif
template <int ORDER>
__global__ void __launch_bounds__(128) lpa_slow_kernel(const __grid_constant__ DevParams P) {
    constexpr int G = SLOW_LANES;  // lanes per work item
    const uint32_t n = *P.work_count;
    const uint32_t grp = (blockIdx.x * blockDim.x + threadIdx.x) / G;
    const uint32_t ngrp = (gridDim.x * blockDim.x) / G;
    for (uint32_t i = grp; i < n; i += ngrp) {
        const uint32_t item = P.work_items[i];
        const int pix = P.row_begin * P.out_w + (int)(item >> 6), c = (int)(item & 3);
        const int kk = (int)((item >> 2) & 15);
        const int ox = pix % P.out_w, oy = pix / P.out_w;
        const GlobalSweep<G> sweep{P, qcoord(ox, P.sx), qcoord(oy, P.sy)};
        PixelResult R;
        if (kk && precise_fit<ORDER>(P, c, kk - 1, sweep, R)) {
            // the fast path's decisions stand; only the value was recomputed
        } else if (P.n_scales > 1) {
            if (ici<ORDER, true>(P, c, sweep, R) != FIT_OK) ladder<ORDER>(P, c, sweep, R);
        } else {
            ladder<ORDER>(P, c, sweep, R);
        }
        if ((threadIdx.x & (G - 1)) == 0) write_result(P, pix, c, R);
    }
}

// ---------------------------------------------------------------------------
// Fast path: persistent CTAs, double-buffered TMA staging of the raw tiles.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile(
        "{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}" ::"r"(
            smem_addr(bar)),
        "r"(bytes)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}" ::"r"(
                     smem_addr(bar))
                 : "memory");
}
// Bounded wait: a barrier that never completes (a lost TMA transaction)
// traps -- the launch fails with an error -- instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    for (uint32_t spin = 0;; ++spin) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
        if (done) return;
        if (spin > (1u << 24)) __trap();
    }
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int x, int y,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_addr(dst)),
        "l"((uint64_t)map), "r"(x), "r"(y), "r"(smem_addr(bar))
        : "memory");
}

__device__ __forceinline__ bool region_origin(const DevSensor &S, const DevParams &P, int tx0,
                                              int ty0, int tx1, int ty1, int &ox, int &oy) {
    // union of the window bboxes of the tile's corner queries at radius fast_R;
    // every bbox bound is a floor/ceil of a correctly rounded affine function
    // of (qx, qy), monotone in each, so its extremes over the tile are
    // attained at the corners.
    int xmin = INT_MAX, ymin = INT_MAX, xmax = INT_MIN, ymax = INT_MIN;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double qx = qcoord((k & 1) ? tx1 : tx0, P.sx);
        const double qy = qcoord((k & 2) ? ty1 : ty0, P.sy);
        int xlo, xhi, ylo, yhi;
        window_bbox(S, qx, qy, P.fast_R, xlo, xhi, ylo, yhi);
        xmin = min(xmin, xlo);
        ymin = min(ymin, ylo);
        xmax = max(xmax, xhi);
        ymax = max(ymax, yhi);
    }
    // x: multiple of 8 elements -- a TMA tile copy must start on a 16-byte
    // boundary of the row (measured: unaligned starts raise an illegal-
    // instruction fault; scripts/probes/tma_probe.cu).  Both even, so the
    // Bayer phase of a staged pixel equals the parity of its coordinates.
    ox = xmin & ~7;
    oy = ymin & ~1;
    // true: every window of every pixel of the tile lies inside the region
    return xmax < ox + S.rw && ymax < oy + S.rh;
}

__device__ __forceinline__ void tile_bounds(const DevParams &P, int t, int &tx0, int &ty0, int &tx1,
                                            int &ty1) {
    tx0 = (t % P.tiles_x) * TW;
    ty0 = P.row_begin + (t / P.tiles_x) * TH;
    tx1 = min(tx0 + TW, P.out_w) - 1;
    ty1 = min(ty0 + TH, P.row_end) - 1;
}

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int x, int y, int z,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_addr(dst)),
        "l"((uint64_t)map), "r"(x), "r"(y), "r"(z), "r"(smem_addr(bar))
        : "memory");
}

// One warp stages tile t into plane buffer `pb`: region origins + tile
// coverage (lane s: sensor s), the f64 coordinate tables (rotated path), then
// lane 0 issues one 3-D TMA copy per sensor of the four (f_hat, 1/den) phase
// planes' staged regions, completing on `full` (arrive + expect_tx; the
// arrive releases the origins and tables to the consumers).
template <bool TABLES>
__device__ __forceinline__ void stage_tile(const DevParams &P, unsigned char *pb, int t,
                                           int (*org)[2], int *cov, uint64_t *full) {
    const int lane = threadIdx.x & 31;
    int tx0, ty0, tx1, ty1;
    tile_bounds(P, t, tx0, ty0, tx1, ty1);
    bool in = true;
    if (lane < P.n_sensors)
        in = region_origin(P.s[lane], P, tx0, ty0, tx1, ty1, org[lane][0], org[lane][1]);
    const bool all_in = __all_sync(0xffffffffu, in);
    if (lane == 0) *cov = all_in ? 1 : 0;
    __syncwarp();
    if constexpr (TABLES) {
        for (int s = 0; s < P.n_sensors; ++s) {
            const DevSensor &S = P.s[s];
            const int ox = org[s][0], oy = org[s][1];
            // separable sensors: tx0 = X(x) = fl(fl(T00*x) + T02), ty4 = Y(y)
            // (exact, since fl(T01*y) = fl(T10*x) = 0); otherwise the four
            // partial products.
            double *tx0t = (double *)(pb + S.off_tx0), *tx3t = (double *)(pb + S.off_tx3);
            double *ty1t = (double *)(pb + S.off_ty1), *ty4t = (double *)(pb + S.off_ty4);
            for (int i = lane; i < S.rw; i += 32) {
                const double xd = (double)(ox + i);
                const double a = __dmul_rn(S.T[0], xd);
                tx0t[i] = S.separable ? __dadd_rn(a, S.T[2]) : a;
                tx3t[i] = __dmul_rn(S.T[3], xd);
            }
            for (int i = lane; i < S.rh; i += 32) {
                const double yd = (double)(oy + i);
                const double bb = __dmul_rn(S.T[4], yd);
                ty1t[i] = __dmul_rn(S.T[1], yd);
                ty4t[i] = S.separable ? __dadd_rn(bb, S.T[5]) : bb;
            }
        }
        __syncwarp();
    }
    if (lane == 0) {
        // the buffer's previous contents were read through the generic proxy
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        uint32_t bytes = 0;
        for (int s = 0; s < P.n_sensors; ++s) bytes += (uint32_t)(P.s[s].rw * P.s[s].rh * 8);
        mbar_expect_tx(full, bytes);
        for (int s = 0; s < P.n_sensors; ++s)  // phase-plane coords: ox/2 float2 = ox floats, oy/2
            tma_load_3d(pb + P.s[s].off_vi, &P.tmap[s], org[s][0], org[s][1] >> 1, 0, full);
    }
}

// Fixed-scale accumulation from the pre-computed taps: the window of every
// output pixel of a parity class visits the same sensor offsets with the same
// weights, so there is no membership test, no exp and no loop control beyond
// the tap list (the samples and weights are the reference's: DESIGN.md s3).
__device__ __forceinline__ double2 lds_d2(uint32_t a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ uint2 lds_u2(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ float2 lds_f2(uint32_t a) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
    return v;
}

template <int ORDER>
__device__ __forceinline__ void accumulate_taps(const DevParams &P, const unsigned char *sm,
                                                const unsigned char *taps, const int (*org)[2],
                                                int c, int px, int py, Acc<NC<ORDER>::P> &acc) {
    acc.zero();
    const int cls = ((py & 1) << 1) | (px & 1);
    // shared-window addresses: one LDS.128 (dx, dy), one LDS.64 (W, byte
    // offset) and one LDS.64 (f_hat, 1/den) per tap
    const uint32_t txy = smem_addr(taps);
    const uint32_t tw = txy + (uint32_t)P.n_taps * (uint32_t)sizeof(TapXY);
    int count = 0;
    float sabs = 0.f;
    for (int s = 0; s < P.n_sensors; ++s) {
        const int n = P.pat_cnt[s][c][py & 1];
        if (!n) continue;
        const DevSensor &S = P.s[s];
        const int o = P.pat_off[s][c][cls];
        const int pw = S.rw >> 1;
        // the pixel's own position in its phase plane (origins are even)
        const uint32_t vb = smem_addr(sm + S.off_vi) +
                            8u * (uint32_t)(((py - org[s][1]) >> 1) * pw + ((px - org[s][0]) >> 1));
        for (int t = o; t < o + n; ++t) {
            const double2 X = lds_d2(txy + 16u * (uint32_t)t);
            const uint2 Q = lds_u2(tw + 8u * (uint32_t)t);
            // masked samples carry (0, 0) and padding taps W = 0, so w and the
            // value are already zero exactly when the tap must not count
            const float2 e = lds_f2(vb + Q.y);
            const float w = __uint_as_float(Q.x) * e.y;
            sabs = fmaf(w, fabsf(e.x), sabs);
            const double dxx = ORDER >= 2 ? __dmul_rn(X.x, X.x) : 0.0;
            const double dyy = ORDER >= 2 ? __dmul_rn(X.y, X.y) : 0.0;
            acc.add((double)w, (double)e.x, X.x, X.y, dxx, dyy, 0);
            // predicated increment (setp + @p add): one instruction less than a select
            asm("{\n .reg .pred p;\n setp.gt.f32 p, %1, 0f00000000;\n @p add.s32 %0, %0, 1;\n}"
                : "+r"(count)
                : "f"(w));
        }
    }
    acc.count = count;
    acc.sabs = sabs;
}

// ---------------------------------------------------------------------------
// CALPA steered pass, fast path (lpa_evaluate two_phase, _kernels.py:257-300):
// the phase-0 step-0 fit (anisotropic window of the steering field at
// r = min(r0, max_radius)) from the staged planes with fp32 weights; any
// other outcome, and fits failing fit_precise, go to lpa_steered_slow_kernel.
// ---------------------------------------------------------------------------
// Per-pixel kernel inputs (SteeringField.kernel_inputs, steering.py:80-107),
// float64 in the reference's operation order; an = (h11, h12, h22, r0).
__device__ __forceinline__ void steer_inputs(const DevParams &P, int pix, int c, double *an) {
    const double th = P.st_theta[pix], s = P.st_sigma[pix], g = P.st_gamma[pix];
    const double ct = cos(th), st = sin(th);
    const double h = P.h[c][0];  // channel scale
    const double c11 = g * (s * ct * ct + st * st / s);
    const double c12 = g * (ct * st) * (1.0 / s - s);
    const double c22 = g * (s * st * st + ct * ct / s);
    an[0] = c11 / h;
    an[1] = c12 / h;
    an[2] = c22 / h;
    an[3] = 3.0 * sqrt(h * s / g);
}

// Row-factored moments with the anisotropic window
// W = exp(-(h11 dx^2 + 2 h12 dx dy + h22 dy^2)) (_kernels.py:164-168): along a
// row dy is constant, so q = h11 dx^2 + (2 h12 dy) dx + h22 dy^2.
template <int ORDER>
struct RowAniso {
    static constexpr int PN = NC<ORDER>::P;
    RowMoments<ORDER> m;
    float h11, h12x2, h22;  // pre-scaled by log2(e)
    float a, b;             // per row: h22 dy^2, 2 h12 dy
    __device__ __forceinline__ void begin_row(double dy, double dyy) {
        m.begin_row(dy, dyy);
        a = h22 * (float)dyy;
        b = h12x2 * (float)dy;
    }
    __device__ __forceinline__ void end_row(double dy, double dyy) { m.end_row(dy, dyy); }
    __device__ __forceinline__ void sample(bool ok, double v, float iv, double dx, double dy,
                                           double dxx, double dyy, float) {
        const float q2 = fmaf(h11, (float)dxx, fmaf(b, (float)dx, a));
        // RowMoments' weight is ex2(-hl * d2f) * iv: feed it q2 with hl = 1
        m.sample(ok, v, iv, dx, dy, dxx, dyy, q2);
    }
    __device__ __forceinline__ void general(bool ok, double v, float iv, double dx, double dy,
                                            double dxx, double dyy, float) {
        const float q2 = fmaf(h11, (float)dxx, fmaf(h12x2, (float)(dx * dy), h22 * (float)dyy));
        m.general(ok, v, iv, dx, dy, dxx, dyy, q2);
    }
};

template <int ORDER, class Sweep>
__device__ __forceinline__ void accumulate_aniso(const Sweep &sweep, int c, const double *an,
                                                 double r, double r2, Acc<NC<ORDER>::P> &acc) {
    constexpr float L2E = 1.4426950408889634f;
    acc.zero();
    const float h11 = (float)an[0] * L2E, h12x2 = 2.f * (float)an[1] * L2E, h22 = (float)an[2] * L2E;
    if constexpr (ORDER >= 1) {
        RowAniso<ORDER> pol{RowMoments<ORDER>{acc, 1.0f}, h11, h12x2, h22, 0.f, 0.f};
        sweep.rows(c, -1, r, r2, pol);
    } else {
        sweep(c, -1, r, r2, [&](bool ok, double v, float iv, double dx, double dy, double dxx,
                                double dyy, float) {
            const float q2 = fmaf(h11, (float)dxx, fmaf(h12x2, (float)(dx * dy), h22 * (float)dyy));
            const float w = ok ? ex2_approx(-q2) * iv : 0.f;
            const double y = ok ? v : 0.0;
            acc.sabs = fmaf(w, fabsf((float)y), acc.sabs);
            acc.add((double)w, y, dx, dy, dxx, dyy, ok ? 1 : 0);
        });
    }
}

template <int ORDER, bool ICI, int MAXC, bool PAT, bool RT, bool STEER>
__device__ __forceinline__ void tile_compute(const DevParams &P, const unsigned char *sm,
                                             const unsigned char *taps, int t,
                                             const int (*org)[2], bool tile_covered) {
    constexpr int PN = NC<ORDER>::P;
    int tx0, ty0, tx1, ty1;
    tile_bounds(P, t, tx0, ty0, tx1, ty1);
    const int px = tx0 + (int)(threadIdx.x % TW);
    const int py = ty0 + (int)(threadIdx.x / TW);
    if (px > tx1 || py > ty1) return;
    const int pix = py * P.out_w + px;
    const double qx = qcoord(px, P.sx), qy = qcoord(py, P.sy);

    // every window of this pixel must lie inside the staged region (checked
    // per pixel only when the tile as a whole is not covered)
    bool covered = true;
    for (int s = 0; !tile_covered && s < P.n_sensors; ++s) {
        const DevSensor &S = P.s[s];
        int xlo, xhi, ylo, yhi;
        window_bbox(S, qx, qy, P.fast_R, xlo, xhi, ylo, yhi);
        covered &= xlo >= org[s][0] && ylo >= org[s][1] && xhi < org[s][0] + S.rw &&
                   yhi < org[s][1] + S.rh;
    }
    const TileSweep<MAXC, HDR_BRANCHY_O2 && (ORDER >= 2), RT> sweep{P, sm, org, qx, qy,
                                                                   px, py, taps};

    for (int c = 0; c < 3; ++c) {
        PixelResult R;
        R.sidx = 0;
        int st = FIT_AMBIG;
        if (covered) {
            if constexpr (STEER) {
                double an[4];
                steer_inputs(P, pix, c, an);
                const double r = fmin(an[3], P.max_radius);
                Acc<PN> acc;
                accumulate_aniso<ORDER>(sweep, c, an, r, __dmul_rn(r, r), acc);
                R.work = acc.count;
                Fit fit;
                st = solve_fast<PN>(acc, P.cond, fit);
                if (st == FIT_OK && !fit_precise<PN>(fit, acc.sabs, r, P.prec_floor)) st = FIT_AMBIG;
                if (st == FIT_OK) {
                    R.count = acc.count;
                    R.val = fit.c0;
                    R.gx = ORDER >= 1 ? fit.c1 : qnan();
                    R.gy = ORDER >= 1 ? fit.c2 : qnan();
                    R.outcome = ORDER * 16;  // phase 0 (anisotropic), radius step 0
                }
            } else if constexpr (ICI) {
                st = ici<ORDER, false>(P, c, sweep, R);
            } else {
                Acc<PN> acc;
                if constexpr (PAT)
                    accumulate_taps<ORDER>(P, sm, taps, org, c, px, py, acc);
                else
                    accumulate<ORDER, false>(P, c, 0, P.r[c][0], P.r2[c][0], sweep, acc);
                R.work = acc.count;
                Fit fit;
                st = solve_fast<PN>(acc, P.cond, fit);
                if (st == FIT_OK && !fit_precise<PN>(fit, acc.sabs, P.r[c][0], P.prec_floor)) {
                    // loose bound failed: the sharp one needs a sweep with g (not
                    // for the tap path, where this is rare); else the exact path
                    float tk = 0.f;
                    if constexpr (!PAT && ORDER >= 1)
                        fit_variance<ORDER, false>(P, c, 0, sweep, fit.g, &tk);
                    if (PAT || ORDER == 0 || !fit_precise_sharp(fit.c0, tk, P.prec_floor))
                        st = FIT_PREC;
                }
                if (st == FIT_OK) {
                    R.count = acc.count;
                    R.val = fit.c0;
                    R.gx = ORDER >= 1 ? fit.c1 : qnan();
                    R.gy = ORDER >= 1 ? fit.c2 : qnan();
                    R.outcome = ORDER * 16;
                }
            }
        }
        if (st == FIT_OK) {
            write_result(P, pix, c, R);
        } else {
            // work item: band-relative pixel | kk | channel, kk = 0: full exact
            // evaluation, kk = k + 1: float64 recomputation of the fit at scale k
            const uint32_t kk = st == FIT_PREC ? (uint32_t)R.sidx + 1u : 0u;
            const uint32_t slot = atomicAdd(P.work_count, 1u);
            P.work_items[slot] =
                ((uint32_t)(pix - P.row_begin * P.out_w) << 6) | (kk << 2) | (uint32_t)c;
        }
    }
}

// Persistent kernel.  The raw frames were converted once per frame into
// (f_hat, 1/den) phase planes by radiance_phase_kernel; each tile's staged
// regions are TMA-loaded from them, double-buffered: while tile t is fitted
// from buffer b, the copies for tile t+1 land in buffer b^1.
#ifndef HDR_O2_MINBLOCKS
#define HDR_O2_MINBLOCKS 2
#endif
#ifndef HDR_PAT_MINBLOCKS
#define HDR_PAT_MINBLOCKS 3
#endif
template <int ORDER, bool ICI, int MAXC, bool PAT, bool RT = false, bool STEER = false>
// Tap-table order<=1 kernels are held to 80 registers: 3 CTAs per SM beat 2
// by ~8% on cfg2; 4 (64 registers, no spills) measured ~2% slower than 3.
__global__ void __launch_bounds__(NT, (ORDER >= 2 ? HDR_O2_MINBLOCKS : (PAT ? HDR_PAT_MINBLOCKS : 2)))
    lpa_fast_kernel(const __grid_constant__ DevParams P,
                    const __grid_constant__
                    typename std::conditional<PAT, TapParam, NoTaps>::type T) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ int s_org[NBUF][MAXS][2];
    __shared__ int s_cov[NBUF];
    __shared__ unsigned s_done[NBUF];
    __shared__ __align__(8) uint64_t bar_full[NBUF];
    const int ntiles = P.tiles_x * P.tiles_y;
    const unsigned char *taps = smem + P.off_taps;
    unsigned char *planes = smem + P.plane_base;
    if constexpr (PAT) {  // the kernel-parameter tap table into shared memory
        const uint4 *src = (const uint4 *)T.bytes;
        uint4 *dst = (uint4 *)(smem + P.off_taps);
        const int n16 = (P.tab_bytes + 15) / 16;
        for (int i = threadIdx.x; i < n16; i += NT) dst[i] = src[i];
    } else if constexpr (RT) {  // the row-tap table from the workspace
        const uint4 *src = (const uint4 *)P.rt_global;
        uint4 *dst = (uint4 *)(smem + P.off_taps);
        const int n16 = (P.tab_bytes + 15) / 16;
        for (int i = threadIdx.x; i < n16; i += NT) dst[i] = __ldg(src + i);
    }
    int t = blockIdx.x;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&bar_full[b], 1);
            s_done[b] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();  // barriers initialised, taps staged
    // prologue: warp 0 stages this CTA's first NBUF tiles
    if (threadIdx.x < 32) {
#pragma unroll
        for (int b = 0; b < NBUF; ++b)
            if (t + b * (int)gridDim.x < ntiles)
                stage_tile<!PAT>(P, planes + b * P.buf_stride, t + b * gridDim.x, s_org[b],
                                 &s_cov[b], &bar_full[b]);
    }
    // No CTA-wide barrier in the loop: a warp waits only for its tile's data.
    // The LAST warp to finish tile t (buffer b) refills b with tile t + NBUF*G,
    // so warps that finish early run up to NBUF-1 tiles ahead instead of idling
    // at a __syncthreads while the slowest warp of the tile completes.
    constexpr int NWARPS = NT / 32;
    for (int i = 0; t < ntiles; ++i, t += gridDim.x) {
        const int b = i % NBUF;
        unsigned char *pb = planes + b * P.buf_stride;
        mbar_wait(&bar_full[b], (uint32_t)((i / NBUF) & 1));
        tile_compute<ORDER, ICI, MAXC, PAT, RT, STEER>(P, pb, taps, t, s_org[b], s_cov[b] != 0);
        const int tn = t + NBUF * (int)gridDim.x;
        if (tn < ntiles) {  // CTA-uniform
            __syncwarp();
            unsigned last = 0;
            if ((threadIdx.x & 31) == 0) {
                __threadfence_block();  // this warp's reads of buffer b precede the count
                last = atomicAdd(&s_done[b], 1u) == NWARPS - 1;
                if (last) {
                    s_done[b] = 0;
                    __threadfence_block();
                }
            }
            if (__shfl_sync(0xffffffffu, last, 0))
                stage_tile<!PAT>(P, pb, tn, s_org[b], &s_cov[b], &bar_full[b]);
        }
    }
}

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

// ---------------------------------------------------------------------------
// CALPA: steering field and steered (anisotropic, two-phase) pass
// (reference steering.py:72-248, _kernels.py:262-275, :303-392)
// ---------------------------------------------------------------------------
struct SteerConsts {
    int half;
    double wstd, lam1, lam2, alpha, sigma_max, inv_scale;
};

// steering_field_kernel (_kernels.py:310-392), float64, one thread per pixel.
__global__ void steering_field_kernel(const float *gx, const float *gy, int w, int h,
                                      SteerConsts K, double *theta, double *sigma,
                                      double *gamma) {
    const int xx = blockIdx.x * blockDim.x + threadIdx.x, yy = blockIdx.y;
    if (xx >= w) return;
    double s11 = 0.0, s12 = 0.0, s22 = 0.0;
    int n = 0;
    const double den = 2.0 * K.wstd * K.wstd;
    for (int dy = -K.half; dy <= K.half; ++dy) {
        const int iy = yy + dy;
        if (iy < 0 || iy >= h) continue;
        for (int dx = -K.half; dx <= K.half; ++dx) {
            const int ix = xx + dx;
            if (ix < 0 || ix >= w) continue;
            const double g1 = (double)gx[(size_t)iy * w + ix] * K.inv_scale;
            const double g2 = (double)gy[(size_t)iy * w + ix] * K.inv_scale;
            if (!(isfinite(g1) && isfinite(g2))) continue;
            const double wgt = exp(-(double)(dx * dx + dy * dy) / den);
            s11 += wgt * g1 * g1;
            s12 += wgt * g1 * g2;
            s22 += wgt * g2 * g2;
            ++n;
        }
    }
    const size_t o = (size_t)yy * w + xx;
    if (n == 0) {
        theta[o] = 0.0;
        sigma[o] = 1.0;
        gamma[o] = 1.0;
        return;
    }
    const double m = 0.5 * (s11 + s22), dd = hypot(0.5 * (s11 - s22), s12);
    const double lmax = m + dd, lmin = fmax(m - dd, 0.0);
    const double s1 = sqrt(lmax), s2 = sqrt(lmin);
    double v1, v2;
    if (fabs(s12) > 1e-300) {
        v1 = s12;
        v2 = lmin - s11;
        if (v1 == 0.0 && v2 == 0.0) v1 = 1.0;
    } else if (s11 <= s22) {
        v1 = 1.0;
        v2 = 0.0;
    } else {
        v1 = 0.0;
        v2 = 1.0;
    }
    double th = atan2(v1, v2);
    if (th <= -0.5 * M_PI)
        th += M_PI;
    else if (th > 0.5 * M_PI)
        th -= M_PI;
    const double dn = s2 + K.lam1;
    double sg = dn == 0.0 ? ((s1 + K.lam1 == 0.0) ? 1.0 : K.sigma_max) : (s1 + K.lam1) / dn;
    if (sg > K.sigma_max) sg = K.sigma_max;
    theta[o] = th;
    sigma[o] = sg;
    gamma[o] = pow((s1 * s2 + K.lam2) / n, K.alpha);
}

// Exact accumulation with an arbitrary SPD window Hinv (two-phase CALPA).
template <int ORDER, class Sweep>
__device__ __forceinline__ void accumulate_hinv(const Sweep &sweep, int c, double h11, double h12,
                                                double h22, double r, double r2,
                                                Acc<NC<ORDER>::P> &acc) {
    acc.zero();
    const double h12x2 = 2.0 * h12;
    sweep(c, -1, r, r2, [&](bool, double v, auto iv, double dx, double dy, double dxx, double dyy,
                        float) {
        // q = h11*dx*dx + 2.0*h12*dx*dy + h22*dy*dy (_kernels.py:164)
        const double q = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(h11, dx), dx),
                                             __dmul_rn(__dmul_rn(h12x2, dx), dy)),
                                   __dmul_rn(__dmul_rn(h22, dy), dy));
        acc.add(exp(-q) * (double)iv, v, dx, dy, dxx, dyy);
    });
    sweep.reduce(acc);
}

template <int ORDER, class Sweep>
__device__ bool steered_order(const DevParams &P, int c, const Sweep &sweep, const double *an,
                              PixelResult &R) {
    constexpr int PN = NC<ORDER>::P;
    Acc<PN> acc;
    for (int phase = 0; phase < 2; ++phase) {
        const double h11 = phase ? P.hinv[c][0] : an[0];
        const double h12 = phase ? 0.0 : an[1];
        const double h22 = phase ? P.hinv[c][0] : an[2];
        double r = phase ? P.r[c][0] : fmin(an[3], P.max_radius);
        int step = 0;
        for (;;) {
            accumulate_hinv<ORDER>(sweep, c, h11, h12, h22, r, __dmul_rn(r, r), acc);
            R.work += acc.count;
            Fit fit;
            if (solve_exact<PN>(acc, P.cond, fit) == FIT_OK) {
                R.count = acc.count;
                R.val = fit.c0;
                R.gx = ORDER >= 1 ? fit.c1 : qnan();
                R.gy = ORDER >= 1 ? fit.c2 : qnan();
                R.outcome = ORDER * 16 + phase * 8 + (step < 7 ? step : 7);
                return true;
            }
            if (r >= P.max_radius * (1.0 - 1e-12)) break;
            r = fmin(r * 1.5, P.max_radius);
            ++step;
        }
    }
    return false;
}

// Steered pass (lpa_evaluate two_phase, _kernels.py:257-300): per pixel and
// channel, Hinv = C/h and r0 = 3 sqrt(h sigma/gamma) from the steering field
// (SteeringField.kernel_inputs, steering.py:94-107).
template <int ORDER>
__global__ void __launch_bounds__(128) lpa_steered_kernel(const __grid_constant__ DevParams P) {
    const int n = P.out_w * (P.row_end - P.row_begin) * 3;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int it = warp; it < n; it += nwarps) {  // one warp per pixel-channel
        const int c = it % 3, pl = it / 3;
        const int ox = pl % P.out_w, oy = P.row_begin + pl / P.out_w;
        const int pix = oy * P.out_w + ox;
        const GlobalSweep<32> sweep{P, qcoord(ox, P.sx), qcoord(oy, P.sy)};
        const double th = P.st_theta[pix], s = P.st_sigma[pix], g = P.st_gamma[pix];
        const double ct = cos(th), st = sin(th);
        const double h = P.h[c][0];  // channel scale
        // covariance_entries (steering.py:80-87), same operation order
        const double c11 = g * (s * ct * ct + st * st / s);
        const double c12 = g * (ct * st) * (1.0 / s - s);
        const double c22 = g * (s * st * st + ct * ct / s);
        const double an[4] = {c11 / h, c12 / h, c22 / h, 3.0 * sqrt(h * s / g)};
        PixelResult R;
        R.sidx = 0;
        bool ok = steered_order<ORDER>(P, c, sweep, an, R);
        if (!ok && ORDER >= 1) ok = steered_order<(ORDER >= 1 ? ORDER - 1 : 0)>(P, c, sweep, an, R);
        if (!ok && ORDER >= 2) ok = steered_order<0>(P, c, sweep, an, R);
        if (!ok) {
            R.val = R.gx = R.gy = qnan();
            R.outcome = HDR_OUTCOME_NAN;
            R.count = 0;
        }
        if ((threadIdx.x & 31) == 0) write_result(P, pix, c, R);
    }
}

// The steered pass's exact evaluation of the fast path's work items (all
// outcomes other than a sound phase-0 step-0 fit), one 8-lane group per item.
template <int ORDER>
__global__ void __launch_bounds__(128) lpa_steered_slow_kernel(const __grid_constant__ DevParams P) {
    constexpr int G = SLOW_LANES;
    const uint32_t n = *P.work_count;
    const uint32_t grp = (blockIdx.x * blockDim.x + threadIdx.x) / G;
    const uint32_t ngrp = (gridDim.x * blockDim.x) / G;
    for (uint32_t i = grp; i < n; i += ngrp) {
        const uint32_t item = P.work_items[i];
        const int pix = P.row_begin * P.out_w + (int)(item >> 6), c = (int)(item & 3);
        const int ox = pix % P.out_w, oy = pix / P.out_w;
        const GlobalSweep<G> sweep{P, qcoord(ox, P.sx), qcoord(oy, P.sy)};
        double an[4];
        steer_inputs(P, pix, c, an);
        PixelResult R;
        R.sidx = 0;
        bool ok = steered_order<ORDER>(P, c, sweep, an, R);
        if (!ok && ORDER >= 1) ok = steered_order<(ORDER >= 1 ? ORDER - 1 : 0)>(P, c, sweep, an, R);
        if (!ok && ORDER >= 2) ok = steered_order<0>(P, c, sweep, an, R);
        if (!ok) {
            R.val = R.gx = R.gy = qnan();
            R.outcome = HDR_OUTCOME_NAN;
            R.count = 0;
        }
        if ((threadIdx.x & (G - 1)) == 0) write_result(P, pix, c, R);
    }
}

// ---------------------------------------------------------------------------
// Scattered samples: the reference kernel boundary itself.  lpa_evaluate over
// a CSR unit-cell index of packed (x, y, value, variance) rows
// (_kernels.py:104-300, radiometry.py:208-242), in the reference's operation
// order: cells row-major, rows in storage order, no FMA contraction, the
// reference's Cholesky (_kernels.py:76-101).
// ---------------------------------------------------------------------------
struct CsrIndex {
    const double *packed;  // n x 4
    const int64_t *cell_start;
    int x0, y0, nx, ny;
};

struct CsrQuery {
    const double *qx, *qy;
    const double *an[4];   // nullable: anisotropic h11, h12, h22, r0 per query (two-phase)
    double iso_hinv, iso_r0, max_radius, cond;
    int order, use_sigma, m, pad;
    double *val, *gx, *gy;
};

template <int P>
__device__ bool chol_solve_ref(const double (&A)[6][6], const double *b, double *coef) {
    double L[6][6], work[6];
#pragma unroll
    for (int i = 0; i < P; ++i)
#pragma unroll
        for (int j = 0; j <= i; ++j) {
            double s = A[i][j];
#pragma unroll
            for (int k = 0; k < j; ++k) s = __dsub_rn(s, __dmul_rn(L[i][k], L[j][k]));
            if (i == j) {
                if (s <= 0.0) return false;
                L[i][i] = __dsqrt_rn(s);
            } else {
                L[i][j] = __ddiv_rn(s, L[j][j]);
            }
        }
#pragma unroll
    for (int i = 0; i < P; ++i) {
        double s = b[i];
#pragma unroll
        for (int k = 0; k < i; ++k) s = __dsub_rn(s, __dmul_rn(L[i][k], work[k]));
        work[i] = __ddiv_rn(s, L[i][i]);
    }
#pragma unroll
    for (int i = P - 1; i >= 0; --i) {
        double s = work[i];
#pragma unroll
        for (int k = i + 1; k < P; ++k) s = __dsub_rn(s, __dmul_rn(L[k][i], coef[k]));
        coef[i] = __ddiv_rn(s, L[i][i]);
    }
    return true;
}

// _fit_at (_kernels.py:104-200) over the CSR index
template <int ORDER>
__device__ int csr_fit_at(const CsrIndex &ix, double qx, double qy, double h11, double h12,
                          double h22, double radius, double cond, int use_sigma, double *coef) {
    constexpr int P = NC<ORDER>::P;
    double A[6][6], rhs[6];
#pragma unroll
    for (int a = 0; a < P; ++a) {
        rhs[a] = 0.0;
#pragma unroll
        for (int b = 0; b < P; ++b) A[a][b] = 0.0;
    }
    int count = 0;
    const double r2 = __dmul_rn(radius, radius);
    int cx_lo = (int)floor(qx - radius) - ix.x0, cx_hi = (int)floor(qx + radius) - ix.x0;
    int cy_lo = (int)floor(qy - radius) - ix.y0, cy_hi = (int)floor(qy + radius) - ix.y0;
    cx_lo = max(cx_lo, 0);
    cy_lo = max(cy_lo, 0);
    cx_hi = min(cx_hi, ix.nx - 1);
    cy_hi = min(cy_hi, ix.ny - 1);
    const double h12x2 = __dmul_rn(2.0, h12);
    for (int cy = cy_lo; cy <= cy_hi; ++cy) {
        const int64_t row = (int64_t)cy * ix.nx;
        for (int cx = cx_lo; cx <= cx_hi; ++cx) {
            const int64_t cell = row + cx;
            const int64_t k1 = ix.cell_start[cell + 1];
            for (int64_t k = ix.cell_start[cell]; k < k1; ++k) {
                const double4 R = *(const double4 *)(ix.packed + 4 * k);
                const double dx = __dsub_rn(R.x, qx), dy = __dsub_rn(R.y, qy);
                if (__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) > r2) continue;
                const double q = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(h11, dx), dx),
                                                     __dmul_rn(__dmul_rn(h12x2, dx), dy)),
                                           __dmul_rn(__dmul_rn(h22, dy), dy));
                const double den = use_sigma ? __dsqrt_rn(R.w) : R.w;
                const double w = __ddiv_rn(exp(-q), den);
                double phi[6];
                phi[0] = 1.0;
                if (ORDER >= 1) {
                    phi[1] = dx;
                    phi[2] = dy;
                }
                if (ORDER >= 2) {
                    phi[3] = __dmul_rn(dx, dx);
                    phi[4] = __dmul_rn(dx, dy);
                    phi[5] = __dmul_rn(dy, dy);
                }
#pragma unroll
                for (int a = 0; a < P; ++a) {
                    const double wa = __dmul_rn(w, phi[a]);
                    rhs[a] = __dadd_rn(rhs[a], __dmul_rn(wa, R.z));
#pragma unroll
                    for (int b = a; b < P; ++b) A[a][b] = __dadd_rn(A[a][b], __dmul_rn(wa, phi[b]));
                }
                ++count;
            }
        }
    }
    if (count < P) return FIT_FAIL;
#pragma unroll
    for (int a = 0; a < P; ++a)
#pragma unroll
        for (int b = a + 1; b < P; ++b) A[b][a] = A[a][b];
    if constexpr (P == 1) {
        if (A[0][0] <= 0.0) return FIT_FAIL;
        coef[0] = __ddiv_rn(rhs[0], A[0][0]);
        return FIT_OK;
    } else {
        double packedA[P * (P + 1) / 2], lmin, lmax;
        int k = 0;
#pragma unroll
        for (int a = 0; a < P; ++a)
#pragma unroll
            for (int b = a; b < P; ++b) packedA[k++] = A[a][b];
        if constexpr (P == 3)
            eig_range3(packedA, lmin, lmax);
        else
            eig_range6(packedA, lmin, lmax);
        if (lmin <= 0.0 || lmax > cond * lmin) return FIT_FAIL;
        return chol_solve_ref<P>(A, rhs, coef) ? FIT_OK : FIT_FAIL;
    }
}

template <int ORDER>
__device__ bool csr_order(const CsrIndex &ix, const CsrQuery &Q, int i, double *out) {
    const int nphase = Q.an[0] ? 2 : 1;
    double coef[6];
    for (int phase = 0; phase < nphase; ++phase) {
        double h11, h12, h22, r;
        if (phase == 0 && Q.an[0]) {
            h11 = Q.an[0][i];
            h12 = Q.an[1][i];
            h22 = Q.an[2][i];
            r = Q.an[3][i];
        } else {
            h11 = Q.iso_hinv;
            h12 = 0.0;
            h22 = Q.iso_hinv;
            r = Q.iso_r0;
        }
        if (r > Q.max_radius) r = Q.max_radius;
        for (;;) {
            if (csr_fit_at<ORDER>(ix, Q.qx[i], Q.qy[i], h11, h12, h22, r, Q.cond, Q.use_sigma,
                                  coef) == FIT_OK) {
                out[0] = coef[0];
                out[1] = ORDER >= 1 ? coef[1] : qnan();
                out[2] = ORDER >= 1 ? coef[2] : qnan();
                return true;
            }
            if (r >= Q.max_radius * (1.0 - 1e-12)) break;
            r = fmin(r * 1.5, Q.max_radius);
        }
    }
    return false;
}

template <int ORDER>
__global__ void __launch_bounds__(128) lpa_samples_kernel(const CsrIndex ix, const CsrQuery Q) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < Q.m; i += gridDim.x * blockDim.x) {
        double out[3];
        bool ok = csr_order<ORDER>(ix, Q, i, out);
        if (!ok && ORDER >= 1) ok = csr_order<(ORDER >= 1 ? ORDER - 1 : 0)>(ix, Q, i, out);
        if (!ok && ORDER >= 2) ok = csr_order<0>(ix, Q, i, out);
        if (!ok) out[0] = out[1] = out[2] = qnan();
        Q.val[i] = out[0];
        Q.gx[i] = out[1];
        Q.gy[i] = out[2];
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
    // 16-B vector loads of raw rows in the pre-pass
    d.vec_raw = ((uintptr_t)h.raw % 16 == 0) && (h.pitch % 8 == 0);
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
    d.bias_f = (float)d.bias;
    d.readvar_f = (float)d.readvar;
    d.inv_denom_f = (float)d.inv_denom;
    d.inv_denom2_f = (float)d.inv_denom2;
    d.c_shot_f = (float)d.c_shot;
    d.qv_f = (float)d.qv;
    d.Tf[0] = (float)T[0];
    d.Tf[1] = (float)T[1];
    d.Tf[2] = (float)T[3];
    d.Tf[3] = (float)T[4];
    return HDR_OK;
}

static thread_local char g_last_error[256] = "";
// kernel launches issued by this library since load (hdr_lpa_launch_count)
static std::atomic<unsigned long long> g_launches{0};
#define COUNT_LAUNCH() g_launches.fetch_add(1, std::memory_order_relaxed)

static int cuda_fail(const char *where) {
    const cudaError_t e = cudaGetLastError();
    snprintf(g_last_error, sizeof(g_last_error), "%s: %s", where, cudaGetErrorString(e));
    return HDR_ERR_CUDA;
}

static int set_smem_attr(const void *fn, int bytes) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    return e == cudaSuccess ? HDR_OK : cuda_fail("cudaFuncSetAttribute(smem)");
}

template <int ORDER, bool ICI, int MAXC, bool PAT = false, bool RT = false, bool STEER = false>
static int launch_fast(const DevParams &P, const TapParam &T, int tiles, int smem_bytes,
                       cudaStream_t st) {
    const void *fn = (const void *)lpa_fast_kernel<ORDER, ICI, MAXC, PAT, RT, STEER>;
    if (set_smem_attr(fn, smem_bytes) != HDR_OK) return HDR_ERR_CUDA;
    int dev = 0, nsm = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT, smem_bytes) != cudaSuccess ||
        per_sm < 1)
        return cuda_fail("occupancy query");
    const int grid = min(tiles, nsm * per_sm);  // persistent: every CTA loops over tiles
    COUNT_LAUNCH();
    if constexpr (PAT)
        lpa_fast_kernel<ORDER, ICI, MAXC, PAT, RT, STEER><<<grid, NT, smem_bytes, st>>>(P, T);
    else
        lpa_fast_kernel<ORDER, ICI, MAXC, PAT, RT, STEER><<<grid, NT, smem_bytes, st>>>(P, NoTaps{});
    return cudaPeekAtLastError() == cudaSuccess ? HDR_OK : cuda_fail("lpa_fast_kernel launch");
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

// 3-D float32 tensor map over one sensor's phase planes [4][phg][2*pwg]
// (float2 = 2 floats); the box is the staged region (rw floats = rw/2 float2,
// rh/2 rows, 4 phases).  The planes live in the workspace, 16-B aligned with
// 16-B row pitch, so TMA is always applicable.
static bool encode_phase_map(const DevSensor &d, CUtensorMap *map) {
    auto enc = tensor_map_encoder();
    if (!enc || d.rw > 256 || (d.rh >> 1) > 256) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)d.pwg * 2, (cuuint64_t)d.phg, 4};
    const cuuint64_t strides[2] = {(cuuint64_t)d.pwg * 8, (cuuint64_t)d.pwg * 8 * d.phg};
    const cuuint32_t box[3] = {(cuuint32_t)d.rw, (cuuint32_t)(d.rh >> 1), 4};
    const cuuint32_t estr[3] = {1, 1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void *)d.phase, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int ORDER>
static int launch_all(const DevParams &P, const TapParam &T, int tiles, int smem_bytes, int maxc,
                      cudaStream_t st) {
    int rc;
    if (P.pat)
        rc = launch_fast<ORDER, false, 4, true>(P, T, tiles, smem_bytes, st);
    else if (P.rt && P.n_scales > 1)
        rc = maxc <= 6 ? launch_fast<ORDER, true, 6, false, true>(P, T, tiles, smem_bytes, st)
                       : launch_fast<ORDER, true, 8, false, true>(P, T, tiles, smem_bytes, st);
    else if (P.rt)
        rc = maxc <= 4 ? launch_fast<ORDER, false, 4, false, true>(P, T, tiles, smem_bytes, st)
                       : launch_fast<ORDER, false, 8, false, true>(P, T, tiles, smem_bytes, st);
    else if (P.n_scales > 1)
        rc = maxc <= 6 ? launch_fast<ORDER, true, 6>(P, T, tiles, smem_bytes, st)
                       : launch_fast<ORDER, true, 8>(P, T, tiles, smem_bytes, st);
    else
        rc = maxc <= 4 ? launch_fast<ORDER, false, 4>(P, T, tiles, smem_bytes, st)
                       : launch_fast<ORDER, false, 8>(P, T, tiles, smem_bytes, st);
    if (rc != HDR_OK) return rc;
    if (P.flags & HDR_FLAG_FAST_ONLY) return HDR_OK;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    COUNT_LAUNCH();
    lpa_slow_kernel<ORDER><<<nsm * 4, 128, 0, st>>>(P);
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("lpa_slow_kernel launch");
    return HDR_OK;
}

// Pre-computed-weight mode: applies when the output grid is the
// reference grid and every sensor is translation-only.  Then, for an output
// pixel q = (j, i), sensor pixel x = j + k maps to X = fl(x + T02) and
// dx = X - j = k + T02 up to the rounding of fl(x + T02) (< 3e-13 for
// |x| < 2^12): the window of every pixel of a parity class (j & 1, i & 1)
// contains the same offsets with the same weights.  The tables are built with
// the reference's arithmetic at a representative pixel; a tap closer than
// 1e-9 r^2 to the support boundary (where that rounding could flip the
// membership test) disables the mode.
// Row-tap mode: the same construction for the translation-only sensors of a
// rig on the reference grid when PAT does not apply (ICI scales, order 2 or a
// rotated sensor elsewhere in the rig).  Per (sensor, channel, class) the
// sensor rows of the largest window, each with the exact dy and its taps in
// column order; d2 is convex along a row, so each scale's members are one run
// [lo[k], hi[k]).  Any tap within 1e-9 r_k^2 of any scale's support boundary
// disables the mode (the per-pixel rounding could flip membership there).
static bool build_rowtaps(DevParams &P, std::vector<unsigned char> &table) {
    int shift;
    if (P.sx == 1.0 && P.sy == 1.0)
        shift = 0;
    else if (P.sx == 0.5 && P.sy == 0.5)
        shift = 1;  // 2x output grid: classes repeat every 4 output pixels
    else
        return false;
    const int period = 2 << shift;
    bool any = false;
    for (int s = 0; s < P.n_sensors; ++s) {
        const DevSensor &S = P.s[s];
        if (!S.separable) continue;
        if (!(S.T[0] == 1.0 && S.T[4] == 1.0)) return false;  // separable but scaled
        if (fabs(S.T[2]) > 64 || fabs(S.T[5]) > 64 || S.width > 4096 || S.height > 4096)
            return false;
        any = true;
    }
    if (!any) return false;
    RtHeader hd;
    memset(&hd, 0, sizeof(hd));
    std::vector<TapRow> rows;
    std::vector<RowTap> taps;
    for (int s = 0; s < P.n_sensors; ++s) {
        const DevSensor &S = P.s[s];
        if (!S.separable) continue;
        int tile[4];
        for (int ph = 0; ph < 4; ++ph)
            for (int c = 0; c < 3; ++c)
                if ((S.phmask[c] >> ph) & 1) tile[ph] = c;
        const int pw = S.rw >> 1, plane = pw * (S.rh >> 1);
        for (int c = 0; c < 3; ++c) {
            double rmax2 = 0.0, rmax = 0.0;
            for (int k = 0; k < P.n_scales; ++k) {
                rmax2 = fmax(rmax2, P.r2[c][k]);
                rmax = fmax(rmax, P.r[c][k]);
            }
            const int R = (int)ceil(rmax + fabs(S.T[2]) + fabs(S.T[5])) + 2;
            for (int cl = 0; cl < period * period; ++cl) {
                // representative output pixel of the class and its anchor
                const int j = 128 + cl % period, i = 128 + cl / period;
                const double qx = ((double)j + 0.5) * P.sx + -0.5;  // qcoord (lpa.py:222-223)
                const double qy = ((double)i + 0.5) * P.sy + -0.5;
                const int ax = j >> shift, ay = i >> shift;
                hd.row0[s][c][cl] = (int)rows.size();
                for (int m = -R; m <= R; ++m) {
                    const int y = ay + m;
                    TapRow row;
                    memset(&row, 0, sizeof(row));
                    row.first = (int)taps.size();
                    std::vector<double> d2s;
                    for (int k2 = -R; k2 <= R; ++k2) {
                        const int x = ax + k2;
                        if (tile[((y & 1) << 1) | (x & 1)] != c) continue;
                        const double X = (1.0 * (double)x + 0.0 * (double)y) + S.T[2];
                        const double Y = (0.0 * (double)x + 1.0 * (double)y) + S.T[5];
                        const double dx = X - qx, dy = Y - qy;
                        const double d2 = dx * dx + dy * dy;
                        for (int k = 0; k < P.n_scales; ++k)
                            if (fabs(d2 - P.r2[c][k]) <= 1e-9 * P.r2[c][k]) return false;
                        if (d2 > rmax2) continue;
                        RowTap t;
                        t.dx = dx;
                        t.d2f = (float)d2;
                        const int ph = ((y & 1) << 1) | (x & 1);
                        t.off = (int)sizeof(float2) *
                                (ph * plane + ((y >> 1) - (ay >> 1)) * pw + ((x >> 1) - (ax >> 1)));
                        taps.push_back(t);
                        d2s.push_back(d2);
                        row.dy = dy;
                    }
                    const int n = (int)d2s.size();
                    if (!n) continue;
                    if (n > 255) return false;
                    for (int k = 0; k < P.n_scales; ++k) {
                        int lo = n, hi = 0;
                        for (int u = 0; u < n; ++u)
                            if (d2s[u] <= P.r2[c][k]) {
                                lo = std::min(lo, u);
                                hi = u + 1;
                            }
                        if (lo >= hi) lo = hi = 0;
                        row.lo[k] = (unsigned char)lo;
                        row.hi[k] = (unsigned char)hi;
                    }
                    rows.push_back(row);
                }
                hd.nrow[s][c][cl] = (int)rows.size() - hd.row0[s][c][cl];
            }
        }
    }
    hd.n_rows = (int)rows.size();
    const size_t bytes =
        sizeof(RtHeader) + rows.size() * sizeof(TapRow) + taps.size() * sizeof(RowTap);
    if (bytes > RT_TABLE_BYTES) return false;
    table.resize(bytes);
    memcpy(table.data(), &hd, sizeof(hd));
    memcpy(table.data() + sizeof(hd), rows.data(), rows.size() * sizeof(TapRow));
    memcpy(table.data() + sizeof(hd) + rows.size() * sizeof(TapRow), taps.data(),
           taps.size() * sizeof(RowTap));
    P.rt_period = period;
    P.rt_shift = shift;
    P.tab_bytes = (int)bytes;
    return true;
}

// Device copy of a host table without a host->device memcpy (graph-capturable,
// no host buffer lifetime): the bytes travel in kernel parameters, one chunk
// per launch.
struct __align__(16) TableChunk {
    unsigned char bytes[24576];
};
__global__ void table_copy_kernel(const __grid_constant__ TableChunk ch, unsigned char *dst,
                                  int n) {
    for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < n / 16; i += blockDim.x * gridDim.x)
        ((uint4 *)dst)[i] = ((const uint4 *)ch.bytes)[i];
}
static int upload_table(const std::vector<unsigned char> &table, unsigned char *dst,
                        cudaStream_t st) {
    static thread_local TableChunk ch;
    const size_t n = (table.size() + 15) & ~(size_t)15;
    for (size_t off = 0; off < n; off += sizeof(ch.bytes)) {
        const size_t len = std::min(sizeof(ch.bytes), n - off);
        memset(ch.bytes, 0, sizeof(ch.bytes));
        memcpy(ch.bytes, table.data() + off, std::min(len, table.size() - off));
        COUNT_LAUNCH();
        table_copy_kernel<<<4, 256, 0, st>>>(ch, dst + off, (int)len);
        if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("table_copy_kernel launch");
    }
    return HDR_OK;
}

static bool build_taps(DevParams &P, std::vector<Tap> &taps) {
    taps.clear();
    if (P.n_scales != 1 || P.sx != 1.0 || P.sy != 1.0) return false;
    for (int s = 0; s < P.n_sensors; ++s) {
        const DevSensor &S = P.s[s];
        if (!(S.T[0] == 1.0 && S.T[1] == 0.0 && S.T[3] == 0.0 && S.T[4] == 1.0)) return false;
        if (fabs(S.T[2]) > 64 || fabs(S.T[5]) > 64 || S.width > 4096 || S.height > 4096)
            return false;
    }
    for (int s = 0; s < P.n_sensors; ++s) {
        const DevSensor &S = P.s[s];
        int tile[4];
        for (int ph = 0; ph < 4; ++ph)
            for (int c = 0; c < 3; ++c)
                if ((S.phmask[c] >> ph) & 1) tile[ph] = c;
        for (int c = 0; c < 3; ++c) {
            const double r = P.r[c][0], r2 = P.r2[c][0], hi = P.hinv[c][0];
            const int R = (int)ceil(r + fabs(S.T[2]) + fabs(S.T[5])) + 1;
            std::vector<Tap> cls[4];
            for (int cl = 0; cl < 4; ++cl) {
                const int j = 64 + (cl & 1), i = 64 + (cl >> 1);  // representative pixel
                const double qx = (double)j, qy = (double)i;      // qcoord(j, 1.0) == j
                for (int m = -R; m <= R; ++m)
                    for (int k = -R; k <= R; ++k) {
                        const int x = j + k, y = i + m;
                        if (tile[((y & 1) << 1) | (x & 1)] != c) continue;
                        const double X = (1.0 * (double)x + 0.0 * (double)y) + S.T[2];
                        const double Y = (0.0 * (double)x + 1.0 * (double)y) + S.T[5];
                        const double dx = X - qx, dy = Y - qy;
                        const double d2 = dx * dx + dy * dy;
                        if (fabs(d2 - r2) <= 1e-9 * r2) return false;  // near-tie: general path
                        if (d2 > r2) continue;
                        const double q = hi * dx * dx + hi * dy * dy;
                        // sample (x, y) lives in phase plane ((y&1), (x&1)) at
                        // ((y-oy)>>1, (x-ox)>>1); the pixel (j, i) has base
                        // ((i-oy)>>1)*pw + ((j-ox)>>1).  With ox, oy even the
                        // difference depends only on (k, m) and the class.
                        const int pw = S.rw >> 1, plane = pw * (S.rh >> 1);
                        const int ph = ((y & 1) << 1) | (x & 1);
                        Tap t;
                        t.dx = dx;
                        t.dy = dy;
                        t.W = (float)exp(-q);
                        t.delta = ph * plane + ((y >> 1) - (i >> 1)) * pw + ((x >> 1) - (j >> 1));
                        cls[cl].push_back(t);
                    }
            }
            for (int py = 0; py < 2; ++py) {
                const size_t n = std::max(cls[py * 2].size(), cls[py * 2 + 1].size());
                P.pat_cnt[s][c][py] = (int)n;
                for (int px = 0; px < 2; ++px) {
                    std::vector<Tap> &v = cls[py * 2 + px];
                    Tap pad;
                    memset(&pad, 0, sizeof(pad));  // W = 0: no contribution, not counted
                    while (v.size() < n) v.push_back(pad);
                    P.pat_off[s][c][py * 2 + px] = (int)taps.size();
                    taps.insert(taps.end(), v.begin(), v.end());
                }
            }
        }
    }
    if (taps.size() * sizeof(Tap) > TAP_PARAM_BYTES) return false;
    P.n_taps = (int)taps.size();
    return true;
}


}  // namespace hdrlpa

using namespace hdrlpa;

extern "C" {



int hdr_lpa_abi_version(void) { return HDR_LPA_ABI_VERSION; }

unsigned long long hdr_lpa_launch_count(void) { return g_launches.load(); }

const char *hdr_lpa_last_error(void) { return g_last_error; }

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

// Workspace layout: [header][phase planes of every sensor]
// [exact radiometry LUT of every sensor][work items].  LUT: 65536 x
// (f_hat, 1/den) float64 per sensor, indexed by the raw value (scalar
// calibration only).  Phase planes: per sensor [4][phg][pwg] float2 with
// pwg = ceil(w/2) rounded up to a multiple of 4 (32-B rows: the pre-pass
// writes 4 float2 per thread), phg = ceil(h/2).
static size_t phase_bytes(const HdrSensor &s) {
    const size_t pwg = (size_t)(((s.width + 1) / 2 + 3) & ~3), phg = (size_t)((s.height + 1) / 2);
    return 4 * pwg * phg * sizeof(float2);
}

int hdr_lpa_workspace_bytes(const HdrSensor *sensors, int n_sensors, int out_w, int out_h,
                            size_t *bytes) {
    if (!sensors || n_sensors < 1 || n_sensors > MAXS) return HDR_ERR_ARG;
    if (out_w <= 0 || out_h <= 0 || !bytes) return HDR_ERR_ARG;
    if ((size_t)out_w * out_h >= (1ull << 30)) return HDR_ERR_ARG;  // item packing
    size_t planes = 0;
    for (int s = 0; s < n_sensors; ++s) {
        if (sensors[s].width <= 0 || sensors[s].height <= 0) return HDR_ERR_ARG;
        planes += phase_bytes(sensors[s]);
    }
    *bytes = WS_HEADER + RT_TABLE_BYTES + planes + (size_t)n_sensors * LUT_BYTES +
             (size_t)out_w * out_h * 3 * sizeof(uint32_t);
    return HDR_OK;
}

// Validation and DevParams set-up shared by the plain and steered entry points.
static int setup_params(const HdrSensor *sensors, int n_sensors, const HdrParams *params,
                        int out_w, int out_h, double ref_w, double ref_h, int row_begin,
                        int row_end, const HdrOutputs *out, void *workspace,
                        size_t workspace_bytes, DevParams &P, double &fastR) {
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
    if ((size_t)(row_end - row_begin) * out_w >= (1ull << 26)) {  // work-item packing
        snprintf(g_last_error, sizeof(g_last_error),
                 "row band of %zu pixels: split calls into bands of < 2^26 output pixels",
                 (size_t)(row_end - row_begin) * out_w);
        return HDR_ERR_ARG;
    }
    if ((uintptr_t)workspace & 255) return HDR_ERR_ARG;

    memset(&P, 0, sizeof(P));
    for (int s = 0; s < n_sensors; ++s) {
        const int rc = fill_sensor(sensors[s], P.s[s]);
        if (rc != HDR_OK) return rc;
    }
    size_t need = 0;
    if (hdr_lpa_workspace_bytes(sensors, n_sensors, out_w, out_h, &need) != HDR_OK)
        return HDR_ERR_ARG;
    if (workspace_bytes < need) return HDR_ERR_WORKSPACE;
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
    P.prec_floor = 10.0;  // e/s: the parity tests' relative-error floor (oracle/compare.py)
    fastR = 0.0;
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
            P.h[c][k] = h;
            fastR = fmax(fastR, r);
        }
    P.fast_R = fastR;
    P.rgb = out->rgb;
    P.grad = out->grad;
    P.sidx = out->scale_idx;
    P.outcome = out->outcome;
    P.value = out->value;
    P.count = out->count;
    P.work = out->work;
    P.flags = params->flags;
    P.work_count = (uint32_t *)workspace;
    P.rt_global = (const unsigned char *)workspace + WS_HEADER;
    char *wsp = (char *)workspace + WS_HEADER + RT_TABLE_BYTES;
    for (int s = 0; s < n_sensors; ++s) {
        DevSensor &d = P.s[s];
        d.phase = (float2 *)wsp;
        d.pwg = ((d.width + 1) / 2 + 3) & ~3;
        d.phg = (d.height + 1) / 2;
        wsp += phase_bytes(sensors[s]);
    }
    for (int s = 0; s < n_sensors; ++s) {
        P.s[s].lut = (double2 *)wsp;
        wsp += LUT_BYTES;
    }
    P.work_items = (uint32_t *)wsp;

    return HDR_OK;
}

static int launch_prepass(const DevParams &P, cudaStream_t st) {
    int maxsat = 0;
    for (int s = 0; s < P.n_sensors; ++s)
        if (!P.s[s].planes) maxsat = max(maxsat, P.s[s].sat);
    if (maxsat > 0) {
        COUNT_LAUNCH();
        radiance_lut_kernel<<<dim3((maxsat + 255) / 256, P.n_sensors), 256, 0, st>>>(P);
        if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("radiance_lut_kernel launch");
    }
    int maxpw = 0, maxph = 0;
    for (int s = 0; s < P.n_sensors; ++s) {
        maxpw = max(maxpw, P.s[s].pwg);
        maxph = max(maxph, P.s[s].phg);
    }
    dim3 grid((maxpw / 4 + 31) / 32, (maxph + 3) / 4, P.n_sensors);
    COUNT_LAUNCH();
    radiance_phase_kernel<<<grid, dim3(32, 4), 0, st>>>(P);
    return cudaPeekAtLastError() == cudaSuccess ? HDR_OK : cuda_fail("radiance_phase_kernel launch");
}

// Staged-region geometry, shared-memory layout, tap tables (when allowed) and
// TMA descriptors of the fast kernels, for windows up to radius fastR.
static int setup_staging(DevParams &P, int n_sensors, double fastR, bool allow_taps, TapParam &T,
                         std::vector<unsigned char> &rt_table, int &smem_bytes, int &maxc) {
    // Staged region per sensor: tile extent in sensor space + 2 x window
    // half-width (+ rounding/alignment slack).  Shared memory: pre-computed
    // taps, then two plane buffers, each holding per sensor the four staged
    // (f_hat, 1/den) phase planes and the f64 coordinate tables.
    int smem = 0;
    maxc = 1;
    auto take = [&](int bytes) {
        const int off = smem;
        smem += (bytes + 64 + 127) & ~127;  // 128-B aligned (TMA destinations) + read slack
        return off;
    };
    for (int s = 0; s < n_sensors; ++s) {
        DevSensor &d = P.s[s];
        const double ex = (TW - 1) * P.sx, ey = (TH - 1) * P.sy;
        const double wx = fabs(d.N[0]) * ex + fabs(d.N[1]) * ey + 2.0 * fastR * d.nrow0;
        const double wy = fabs(d.N[2]) * ex + fabs(d.N[3]) * ey + 2.0 * fastR * d.nrow1;
        // + 2 for floor/ceil of the bbox ends, + 7 / + 1 for aligning the origin
        // down to a multiple of 8 columns / 2 rows
        int rw = (int)ceil(wx) + 2 + 7, rh = (int)ceil(wy) + 2 + 1;
        rw = (rw + 7) & ~7;  // TMA box inner extent: multiple of 16 bytes
        rh += rh & 1;
        d.rw = rw;
        d.rh = rh;
        // columns of one Bayer phase inside a window bbox: <= floor(r |N row 0|) + 2
        maxc = max(maxc, (int)floor(fastR * d.nrow0) + 2);
    }
    std::vector<Tap> taps;
    P.pat = allow_taps && build_taps(P, taps) ? 1 : 0;
    if (P.pat) {
        P.off_taps = take((int)(taps.size() * sizeof(Tap)));
        // SoA layout (TapXY[n], TapW[n]) in the kernel parameter
        const size_t n = taps.size();
        TapXY *xy = (TapXY *)T.bytes;
        TapW *w = (TapW *)(T.bytes + n * sizeof(TapXY));
        for (size_t i = 0; i < n; ++i) {
            xy[i].dx = taps[i].dx;
            xy[i].dy = taps[i].dy;
            w[i].W = taps[i].W;
            w[i].off = taps[i].delta * (int)sizeof(float2);
        }
        P.tab_bytes = (int)(n * sizeof(Tap));
    } else if (allow_taps) {
        P.rt = build_rowtaps(P, rt_table) ? 1 : 0;
        if (P.rt) P.off_taps = take(P.tab_bytes);
    }
    P.plane_base = smem;
    smem = 0;
    for (int s = 0; s < n_sensors; ++s) {
        DevSensor &d = P.s[s];
        d.off_vi = take(d.rw * d.rh * 8);  // [4][rh/2][rw/2] float2
        d.off_tx0 = take(d.rw * 8);
        d.off_tx3 = take(d.rw * 8);
        d.off_ty1 = take(d.rh * 8);
        d.off_ty4 = take(d.rh * 8);
    }
    P.buf_stride = smem;
    smem_bytes = P.plane_base + NBUF * P.buf_stride;
    if (smem_bytes > 200 * 1024) return HDR_ERR_ARG;  // window too large for the staged path
    for (int s = 0; s < n_sensors; ++s)
        if (!encode_phase_map(P.s[s], &P.tmap[s])) {
            snprintf(g_last_error, sizeof(g_last_error), "cuTensorMapEncodeTiled failed (sensor %d)", s);
            return HDR_ERR_CUDA;
        }

    return HDR_OK;
}

int hdr_lpa_reconstruct(const HdrSensor *sensors, int n_sensors, const HdrParams *params,
                        int out_w, int out_h, double ref_w, double ref_h, int row_begin,
                        int row_end, const HdrOutputs *out, void *workspace,
                        size_t workspace_bytes, void *stream) {
    DevParams P;
    double fastR = 0.0;
    {
        const int rc = setup_params(sensors, n_sensors, params, out_w, out_h, ref_w, ref_h,
                                    row_begin, row_end, out, workspace, workspace_bytes, P, fastR);
        if (rc != HDR_OK) return rc;
    }
    static thread_local TapParam T;  // kernel-parameter image of the tap table
    std::vector<unsigned char> rt_table;
    int smem_bytes = 0, maxc = 1;
    {
        const int rc = setup_staging(P, n_sensors, fastR, true, T, rt_table, smem_bytes, maxc);
        if (rc != HDR_OK) return rc;
    }
    cudaStream_t st = (cudaStream_t)stream;
    P.tiles_y = (row_end - row_begin + TH - 1) / TH;
    P.tiles_x = (out_w + TW - 1) / TW;
    const int tiles = P.tiles_x * P.tiles_y;
    if (cudaMemsetAsync(workspace, 0, sizeof(uint32_t), st) != cudaSuccess)
        return cuda_fail("cudaMemsetAsync");
    if (P.rt && upload_table(rt_table, (unsigned char *)P.rt_global, st) != HDR_OK)
        return HDR_ERR_CUDA;
    if (launch_prepass(P, st) != HDR_OK) return HDR_ERR_CUDA;  // per-frame radiometry
    int rc;
    switch (P.order) {
        case 0: rc = launch_all<0>(P, T, tiles, smem_bytes, maxc, st); break;
        case 1: rc = launch_all<1>(P, T, tiles, smem_bytes, maxc, st); break;
        default: rc = launch_all<2>(P, T, tiles, smem_bytes, maxc, st); break;
    }
    return rc;
}

int hdr_lpa_reconstruct_steered(const HdrSensor *sensors, int n_sensors,
                                const HdrParams *params, const HdrSteering *steering, int out_w,
                                int out_h, double ref_w, double ref_h, int row_begin, int row_end,
                                const HdrOutputs *out, void *workspace, size_t workspace_bytes,
                                void *stream) {
    if (!steering || !steering->theta || !steering->sigma || !steering->gamma) return HDR_ERR_ARG;
    if (params && params->n_scales != 1) return HDR_ERR_ARG;  // CALPA is fixed-scale
    DevParams P;
    double fastR = 0.0;
    const int rc = setup_params(sensors, n_sensors, params, out_w, out_h, ref_w, ref_h, row_begin,
                                row_end, out, workspace, workspace_bytes, P, fastR);
    if (rc != HDR_OK) return rc;
    P.st_theta = steering->theta;
    P.st_sigma = steering->sigma;
    P.st_gamma = steering->gamma;
    cudaStream_t st = (cudaStream_t)stream;
    // fast path: tiles staged for the largest steered radius (max_radius)
    static thread_local TapParam T;
    std::vector<unsigned char> rt_table;
    int smem_bytes = 0, maxc = 1;
    P.fast_R = P.max_radius;
    const bool staged =
        setup_staging(P, n_sensors, P.max_radius, false, T, rt_table, smem_bytes, maxc) == HDR_OK;
    if (cudaMemsetAsync(workspace, 0, sizeof(uint32_t), st) != cudaSuccess)
        return cuda_fail("cudaMemsetAsync");
    if (launch_prepass(P, st) != HDR_OK) return HDR_ERR_CUDA;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (staged) {
        P.tiles_y = (P.row_end - P.row_begin + TH - 1) / TH;
        P.tiles_x = (out_w + TW - 1) / TW;
        const int tiles = P.tiles_x * P.tiles_y;
        int rc2;
        switch (P.order) {
            case 0: rc2 = launch_fast<0, false, 8, false, false, true>(P, T, tiles, smem_bytes, st); break;
            case 1: rc2 = launch_fast<1, false, 8, false, false, true>(P, T, tiles, smem_bytes, st); break;
            default: rc2 = launch_fast<2, false, 8, false, false, true>(P, T, tiles, smem_bytes, st); break;
        }
        if (rc2 != HDR_OK) return rc2;
        if (P.flags & HDR_FLAG_FAST_ONLY) return HDR_OK;
        const int grid = nsm * 4;
        switch (P.order) {
            case 0: COUNT_LAUNCH(); lpa_steered_slow_kernel<0><<<grid, 128, 0, st>>>(P); break;
            case 1: COUNT_LAUNCH(); lpa_steered_slow_kernel<1><<<grid, 128, 0, st>>>(P); break;
            default: COUNT_LAUNCH(); lpa_steered_slow_kernel<2><<<grid, 128, 0, st>>>(P); break;
        }
        return cudaPeekAtLastError() == cudaSuccess ? HDR_OK
                                                    : cuda_fail("lpa_steered_slow_kernel launch");
    }
    // windows too large to stage: every pixel-channel through the exact kernel
    const int grid = nsm * 8;
    switch (P.order) {
        case 0: COUNT_LAUNCH(); lpa_steered_kernel<0><<<grid, 128, 0, st>>>(P); break;
        case 1: COUNT_LAUNCH(); lpa_steered_kernel<1><<<grid, 128, 0, st>>>(P); break;
        default: COUNT_LAUNCH(); lpa_steered_kernel<2><<<grid, 128, 0, st>>>(P); break;
    }
    return cudaPeekAtLastError() == cudaSuccess ? HDR_OK : cuda_fail("lpa_steered_kernel launch");
}

int hdr_lpa_evaluate_samples(const HdrSampleIndex *index, const double *qx, const double *qy,
                             int m, const double *an_h11, const double *an_h12,
                             const double *an_h22, const double *an_r0, double iso_hinv,
                             double iso_r0, int order, double max_radius, double cond_threshold,
                             int weight_mode, double *out_val, double *out_gx, double *out_gy,
                             void *stream) {
    if (!index || !qx || !qy || m < 0 || !out_val || !out_gx || !out_gy) return HDR_ERR_ARG;
    if (order < 0 || order > 2) return HDR_ERR_ARG;
    if (weight_mode != HDR_WEIGHT_VARIANCE && weight_mode != HDR_WEIGHT_SIGMA) return HDR_ERR_ARG;
    if (m == 0) return HDR_OK;
    if (index->n < 0 || index->nx <= 0 || index->ny <= 0) return HDR_ERR_ARG;
    const bool two = an_h11 != nullptr;
    if (two && (!an_h12 || !an_h22 || !an_r0)) return HDR_ERR_ARG;
    if (index->n == 0) return HDR_ERR_ARG;  // caller fills NaN (lpa.py:346-350)
    if (!index->packed || !index->cell_start) return HDR_ERR_ARG;
    CsrIndex ix{index->packed, index->cell_start, index->x0, index->y0, index->nx, index->ny};
    CsrQuery Q;
    memset(&Q, 0, sizeof(Q));
    Q.qx = qx;
    Q.qy = qy;
    if (two) {
        Q.an[0] = an_h11;
        Q.an[1] = an_h12;
        Q.an[2] = an_h22;
        Q.an[3] = an_r0;
    }
    Q.iso_hinv = iso_hinv;
    Q.iso_r0 = iso_r0;
    Q.max_radius = max_radius;
    Q.cond = cond_threshold;
    Q.order = order;
    Q.use_sigma = weight_mode == HDR_WEIGHT_SIGMA;
    Q.m = m;
    Q.val = out_val;
    Q.gx = out_gx;
    Q.gy = out_gy;
    const int grid = min((m + 127) / 128, 148 * 16);
    cudaStream_t st = (cudaStream_t)stream;
    switch (order) {
        case 0: COUNT_LAUNCH(); lpa_samples_kernel<0><<<grid, 128, 0, st>>>(ix, Q); break;
        case 1: COUNT_LAUNCH(); lpa_samples_kernel<1><<<grid, 128, 0, st>>>(ix, Q); break;
        default: COUNT_LAUNCH(); lpa_samples_kernel<2><<<grid, 128, 0, st>>>(ix, Q); break;
    }
    return cudaPeekAtLastError() == cudaSuccess ? HDR_OK : cuda_fail("lpa_samples_kernel launch");
}

int hdr_steering_field(const float *gx, const float *gy, int width, int height,
                       int gradient_window, double lambda1, double lambda2, double alpha,
                       double sigma_max, double gradient_scale, double *theta, double *sigma,
                       double *gamma, void *stream) {
    if (!gx || !gy || !theta || !sigma || !gamma || width <= 0 || height <= 0) return HDR_ERR_ARG;
    if (gradient_window < 3 || gradient_window % 2 == 0) return HDR_ERR_ARG;
    if (!(gradient_scale > 0) || !isfinite(gradient_scale)) return HDR_ERR_ARG;
    if (alpha < 0 || lambda1 < 0 || !(lambda2 > 0)) return HDR_ERR_ARG;
    SteerConsts K;
    K.half = gradient_window / 2;
    K.wstd = gradient_window / 4.0;
    K.lam1 = lambda1;
    K.lam2 = lambda2;
    K.alpha = alpha;
    K.sigma_max = sigma_max;
    K.inv_scale = 1.0 / gradient_scale;
    dim3 grid((width + 127) / 128, height);
    COUNT_LAUNCH();
    steering_field_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(gx, gy, width, height, K, theta,
                                                                  sigma, gamma);
    return cudaPeekAtLastError() == cudaSuccess ? HDR_OK : cuda_fail("steering_field_kernel launch");
}

int hdr_saturation_mask(const HdrSensor *sensor, uint32_t *out_bits, int words_per_row,
                        void *stream) {
    if (!sensor || !out_bits) return HDR_ERR_ARG;
    DevSensor d;
    const int rc = fill_sensor(*sensor, d);
    if (rc != HDR_OK) return rc;
    if (words_per_row < (d.width + 31) / 32) return HDR_ERR_SHAPE;
    dim3 grid((d.width + 255) / 256, d.height);
    COUNT_LAUNCH();
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
    COUNT_LAUNCH();
    radiance_planes_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
        d, weight_mode == HDR_WEIGHT_SIGMA, value, inv_den);
    return cudaPeekAtLastError() == cudaSuccess ? HDR_OK : HDR_ERR_CUDA;
}

int hdr_sample_planes(const HdrSensor *sensor, double *value, double *sigma, void *stream) {
    if (!sensor || !value || !sigma) return HDR_ERR_ARG;
    DevSensor d;
    const int rc = fill_sensor(*sensor, d);
    if (rc != HDR_OK) return rc;
    dim3 grid((d.width + 255) / 256, d.height);
    COUNT_LAUNCH();
    sample_planes_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(d, value, sigma);
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
    COUNT_LAUNCH();
    fp64_probe_kernel<<<blocks, 256, 0, st>>>(sink, iters / 8, 0.999999, 1e-7);  // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0, st);
        COUNT_LAUNCH();
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
