// sweeps.cuh -- window sweeps (global / staged tile) and the accumulation
// policies (row-factored moments and variances) shared by all paths.
#pragma once

#include "config.cuh"

namespace hdrlpa {

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
    __device__ __forceinline__ void begin_row(double dy, double dyy) {
        dy_ = dy;
        dyy_ = dyy;
    }
    __device__ __forceinline__ void end_row(double, double) {}
    __device__ __forceinline__ void sample(bool ok, double v, float iv, double dx, double dy,
                                           double dxx, double dyy, float d2f, bool = true) {
        body(ok, v, iv, dx, dy, dxx, dyy, d2f);
    }
    template <bool CNT = true>  // the body counts (ok flag) either way
    __device__ __forceinline__ void general(bool ok, double v, float iv, double dx, double dy,
                                            double dxx, double dyy, float d2f, bool = true) {
        body(ok, v, iv, dx, dy, dxx, dyy, d2f);
    }
    __device__ __forceinline__ void count_add(int) {}
    double dy_, dyy_;  // the row's offset (row taps pass it to begin_row)
    __device__ __forceinline__ void row_count(int) {}  // the body counts (ok flag)
    __device__ __forceinline__ void first_rt(double dy, double dyy, float2 e, double dx, double dxx,
                                             float d2f, bool inner = true) {
        begin_row(dy, dyy);
        sample_rt(e, dx, dxx, d2f, inner);
    }
    __device__ __forceinline__ void sample_rt(float2 e, double dx, double dxx, float d2f,
                                              bool = true) {
        body(e.y > 0.f, (double)e.x, e.y, dx, dy_, dxx, dyy_, d2f);
    }
};

// MRG4: the staged planes are the co-sited merged float4 planes
// (sum 1/den, sum f_hat/den, sum |f_hat|/den, count; one "sensor"), and the
// policy takes them through sample4() (CALPA's steered pass on co-sited rigs).
// RT: 0 no row taps; 1 row taps counting the valid samples per tap; 2 row taps
// counting every tap of a row (no count / work planes requested: an upper
// bound is enough, the solve's positive-definiteness and condition tests
// imply count >= p)
template <int MAXC, bool BRANCHY, int RT = 0, bool MRG4 = false>
struct TileSweep {
    const DevParams &P;
    const unsigned char *sm;
    const int (*org)[2];
    // the query point lives in a per-thread shared-memory slot and is re-read
    // at each use: under the order-2 kernels' register pressure the compiler
    // otherwise re-derives it (three float64 operations) inside the sample loops
    uint32_t qslot;
    __device__ __forceinline__ double qx() const {
        double v;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(qslot));
        return v;
    }
    __device__ __forceinline__ double qy() const {
        double v;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(qslot + 8u));
        return v;
    }
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
    // taps inside r_k by construction; masked samples carry 1/den = 0).
    // kin >= 0: each sample also carries the inner scale's window weight
    // W[kin] (0 outside r_kin): a fused traversal, variance at kin, moments at k.
    template <class Pol>
    __device__ __forceinline__ void tap_rows(int s, int c, int k, Pol &pol, int kin = -1) const {
        const DevSensor &S = P.s[s];
        const int pm = P.rt_period - 1;
        const int cls = (py & pm) * P.rt_period + (px & pm);
        const int2 rr = ((const int2 *)rt)[((s * 3 + c) * P.rt_ncls + cls) * P.rt_nj + k];
        const double *rdy = (const double *)(rt + P.rt_dy_off);
        const uint32_t *rfn = (const uint32_t *)(rt + P.rt_fn_off);
        const RowTap *taps = (const RowTap *)(rt + P.rt_taps_off);
        const int pw = S.rw >> 1;
        // the pixel's anchor: its own sensor pixel (sx = 1) or cell (sx = 1/2)
        const int ax = px >> P.rt_shift, ay = py >> P.rt_shift;
        // 32-bit shared address of the anchor's sample; a tap's packed word
        // holds its byte offset as 24-bit two's complement under kmin << 24,
        // so (vb + word) mod 2^24 is the sample's address (shared addresses
        // are < 2^24) and kmin <= kin is word < (kin + 1) << 24
        const uint32_t vb = smem_addr(sm) + S.off_vi +
                            8 * (((ay - org[s][1]) >> 1) * pw + ((ax - org[s][0]) >> 1));
        const uint32_t klim = (uint32_t)(kin + 1) << 24;
        for (int ri = rr.x; ri < rr.x + rr.y; ++ri) {
            const double dy = rdy[ri], dyy = dy * dy;
            const uint32_t fn = rfn[ri];
            const RowTap *t = taps + (fn & ((1u << RT_ROW_N_SHIFT) - 1));
            const RowTap *te = t + (fn >> RT_ROW_N_SHIFT);
            int n;  // the row's sample count (RT 1) or tap count (RT 2)
            {  // every row run holds >= 1 tap: the first one opens the row's sums
                const RowTap T = *t;
                const uint32_t a = (vb + (uint32_t)T.off) & 0xFFFFFFu;
                HDR_BOUNDS(P, a >= smem_addr(sm) + S.off_vi &&
                                  a + 8 <= smem_addr(sm) + S.off_vi + S.rw * S.rh * 8);
                const float2 e = lds_f2(a);
                pol.first_rt(dy, dyy, e, T.dx, T.dx * T.dx, T.d2f, (uint32_t)T.off < klim);
                if constexpr (RT == 1) n = e.y > 0.f ? 1 : 0;
            }
#ifndef HDR_RT_UNROLL
#define HDR_RT_UNROLL 1
#endif
            constexpr int kRtUnroll = HDR_RT_UNROLL;
#pragma unroll kRtUnroll
            for (++t; t < te; ++t) {
                const RowTap T = *t;
                const uint32_t a = (vb + (uint32_t)T.off) & 0xFFFFFFu;
                HDR_BOUNDS(P, a >= smem_addr(sm) + S.off_vi &&
                                  a + 8 <= smem_addr(sm) + S.off_vi + S.rw * S.rh * 8);
                const float2 e = lds_f2(a);
                pol.sample_rt(e, T.dx, T.dx * T.dx, T.d2f, (uint32_t)T.off < klim);
                if constexpr (RT == 1) n += e.y > 0.f ? 1 : 0;
            }
            if constexpr (RT != 1) n = (int)(fn >> RT_ROW_N_SHIFT);
            pol.row_count(n);
            pol.end_row(dy, dyy);
        }
    }

    // Traversal with row hooks: for separable sensors every sample of a row
    // shares dy, so a policy can accumulate per-row sums (begin_row / sample /
    // end_row); rotated sensors go through pol.general() per sample.
    template <class Pol>
    __device__ __forceinline__ void rows(int c, int k, double r, double r2, Pol &pol,
                                         int kin = -1) const {
        const double r2in = kin >= 0 ? P.r2[c][kin] : r2;  // exact float64 membership
        for (int s = 0; s < P.n_sensors; ++s) {
            const DevSensor &S = P.s[s];
            const int pm = S.phmask[c];
            if (!pm) continue;
            if constexpr (RT) {
                // RT mode: every separable sensor is translation-only and tapped
                if (S.separable) {
                    tap_rows(s, c, k, pol, kin);
                    continue;
                }
            }
            const int ox = org[s][0], oy = org[s][1];
            const float2 *vi = (const float2 *)(sm + S.off_vi);
            const double *tx0 = (const double *)(sm + S.off_tx0);
            const double *ty4 = (const double *)(sm + S.off_ty4);
            const int pw = S.rw >> 1, plane = pw * (S.rh >> 1);
            int xlo, xhi, ylo, yhi;
            window_bbox(S, qx(), qy(), r, xlo, xhi, ylo, yhi);
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
                                HDR_BOUNDS(P, xs + 2 * i - ox >= 0 && xs + 2 * i - ox < S.rw);
                                cdx[i] = __dsub_rn(tx0[xs + 2 * i - ox], qx());  // X(x) - qx
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
                            HDR_BOUNDS(P, ly >= 0 && ly < S.rh);
                            const double dy = __dsub_rn(ty4[ly], qy());  // Y(y) - qy
                            const double dyy = __dmul_rn(dy, dy);
                            if (dyy > r2) continue;
                            const int rb = colbase + (ly >> 1) * pw;
                            // the row's real columns (the padded tail reads the take() slack)
                            HDR_BOUNDS(P, rb >= 0 &&
                                              rb + (nc - c0 < MAXC ? nc - c0 : MAXC) <= 4 * plane);
                            pol.begin_row(dy, dyy);
                            // orders 0-1: branch-free over the row (candidates outside the
                            // disk or without a sample contribute with weight 0); order 2
                            // (27 DFMA per sample) only visits the samples inside.
#pragma unroll
                            for (int i = 0; i < MAXC; ++i) {
                                const double d2 = __dadd_rn(cdxx[i], dyy);
                                if constexpr (MRG4) {
                                    const float4 e = ((const float4 *)vi)[rb + i];
                                    const bool ok = (d2 <= r2) && (e.x > 0.f);
                                    pol.sample4(ok, e, cdx[i], dy, cdxx[i], dyy, (float)d2);
                                } else if constexpr (BRANCHY) {
                                    if (d2 <= r2) {
                                        const float2 e = vi[rb + i];
                                        if (e.y > 0.f)
                                            pol.sample(true, (double)e.x, e.y, cdx[i], dy, cdxx[i],
                                                       dyy, (float)d2, d2 <= r2in);
                                    }
                                } else {
                                    const float2 e = vi[rb + i];
                                    const bool ok = (d2 <= r2) && (e.y > 0.f);
                                    pol.sample(ok, (double)e.x, e.y, cdx[i], dy, cdxx[i], dyy,
                                               (float)d2, d2 <= r2in);
                                }
                            }
                            pol.end_row(dy, dyy);
                        }
                    }
                }
            } else {
                // interleaved coordinate tables {fl(T00 x), fl(T10 x)} per column and
                // {fl(T01 y), fl(T11 y)} per row (staging.cuh)
                const double2 *txi = (const double2 *)(sm + S.off_tx0);
                const double2 *tyi = (const double2 *)(sm + S.off_ty1);
                const double T2 = S.T[2], T5 = S.T[5];
                // sensor-space position of q relative to the bbox corner (fp32 pre-test)
                const double u = qx() - T2, v = qy() - T5;
                const float fcx = (float)(S.N[0] * u + S.N[1] * v - (double)xlo);
                const float fcy = (float)(S.N[2] * u + S.N[3] * v - (double)ylo);
                const float r2hi = (float)r2 + 1e-3f;
                const float a0 = S.Tf[0], a1 = S.Tf[1], a3 = S.Tf[2], a4 = S.Tf[3];
                // |T_lin e|^2 <= r2hi as a quadratic in e_x along a sensor row:
                // al ex^2 + 2 be ey ex + ga ey^2 - r2hi <= 0 (fp32, widened by
                // 0.01 px: a superset of the exact float64 test below)
                const float al = fmaf(a0, a0, a3 * a3), be = fmaf(a0, a1, a3 * a4),
                            ga = fmaf(a1, a1, a4 * a4), inva = 1.f / al;
                for (int ph = 0; ph < 4; ++ph) {
                    if (!((pm >> ph) & 1)) continue;
                    const int py = ph >> 1, px = ph & 1;
                    const int ys = ylo + ((py - ylo) & 1), xs = xlo + ((px - xlo) & 1);
                    float ey = (float)(ys - ylo) - fcy;
                    for (int y = ys; y <= yhi; y += 2, ey += 2.f) {
                        const float bq = be * ey;
                        const float disc = fmaf(bq, bq, -al * fmaf(ga * ey, ey, -r2hi));
                        if (!(disc >= 0.f)) continue;
                        const float sq = sqrtf(disc);
                        // the row's chord, relative to xlo: x - xlo = ex + fcx
                        int x0 = xlo + (int)ceilf(fmaf(-bq - sq, inva, fcx) - 0.01f);
                        const int x1 = min(xhi, xlo + (int)floorf(fmaf(-bq + sq, inva, fcx) + 0.01f));
                        x0 = max(x0, xs);
                        x0 += (x0 - xs) & 1;
                        const int ly = y - oy;
                        const double2 ty = tyi[ly];  // (fl(T01 y), fl(T11 y))
                        const int rb = ph * plane + (ly >> 1) * pw - (ox >> 1);
                        // straight-line body (the chord pre-test leaves few candidates
                        // outside the disk): masked and outside samples take weight 0
                        const int ncand = ((x1 - x0) >> 1) + 1;  // <= 0: empty chord
                        const float2 *pe = vi + rb + (x0 >> 1);
                        const double2 *pt = txi + (x0 - ox);
                        for (int j = 0; j < ncand; ++j, ++pe, pt += 2) {
                            HDR_BOUNDS(P, rb + (x0 >> 1) + j >= 0 && rb + (x0 >> 1) + j < 4 * plane &&
                                              x0 - ox + 2 * j >= 0 && x0 - ox + 2 * j < S.rw &&
                                              ly >= 0 && ly < S.rh);
                            const float2 e = *pe;
                            const double2 tx = *pt;
                            const double X = __dadd_rn(__dadd_rn(tx.x, ty.x), T2);
                            const double Y = __dadd_rn(__dadd_rn(tx.y, ty.y), T5);
                            const double dx = __dsub_rn(X, qx()), dy = __dsub_rn(Y, qy());
                            const double dxx = __dmul_rn(dx, dx), dyy = __dmul_rn(dy, dy);
                            const double d2 = __dadd_rn(dxx, dyy);  // _kernels.py:160-162
                            const bool ok = (e.y > 0.f) && !(d2 > r2);
                            pol.template general<RT != 2>(ok, (double)e.x, e.y, dx, dy, dxx,
                                                          dyy, (float)d2, d2 <= r2in);
                        }
                        // RT 2: the row's candidates as its count (an upper bound)
                        if constexpr (RT == 2) pol.count_add(ncand > 0 ? ncand : 0);
                    }
                }
            }
        }
    }
};

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
    float fcnt;  // sample4: the merged positions' sample counts (exact in fp32; no
                 // per-sample float-to-int conversion on the XU pipe)
    __device__ __forceinline__ void begin_row(double, double) {
#pragma unroll
        for (int n = 0; n <= 2 * ORDER; ++n) S[n] = 0.0;
#pragma unroll
        for (int n = 0; n <= ORDER; ++n) T[n] = 0.0;
        cnt = 0;
        fcnt = 0.f;
    }
    __device__ __forceinline__ void sample(bool ok, double v, float iv, double dx, double,
                                           double dxx, double, float d2f, bool = true) {
        const float w32 = ok ? ex2_approx(-hl * d2f) * iv : 0.f;
        const double w = (double)w32, y = ok ? v : 0.0;
        acc.sabs = fmaf(w32, fabsf((float)y), acc.sabs);
        // S_n += w dx^n and T_n += (w y) dx^n as fused multiply-adds (dx^2 is
        // the cached column square, dx^3 and dx^4 independent products)
        double px[5];
        px[1] = dx;
        px[2] = dxx;
        if (ORDER >= 2) {
            px[3] = dx * dxx;
            px[4] = dxx * dxx;
        }
        S[0] += w;
#pragma unroll
        for (int n = 1; n <= 2 * ORDER; ++n) S[n] = fma(w, px[n], S[n]);
        const double wy = w * y;
        T[0] += wy;
#pragma unroll
        for (int n = 1; n <= ORDER; ++n) T[n] = fma(wy, px[n], T[n]);
        cnt += ok ? 1 : 0;
    }
    // row tap (RT): every tap lies inside the disk and a masked sample is
    // staged as (0, 0), so no select is needed (its weight and value are 0)
    __device__ __forceinline__ void sample_rt(float2 e, double dx, double dxx, float d2f,
                                              bool = true) {
        const float w32 = ex2_approx(-hl * d2f) * e.y;
        const double w = (double)w32, y = (double)e.x;
        acc.sabs = fmaf(w32, fabsf(e.x), acc.sabs);
        double px[5];
        px[1] = dx;
        px[2] = dxx;
        if (ORDER >= 2) {
            px[3] = dx * dxx;
            px[4] = dxx * dxx;
        }
        S[0] += w;
#pragma unroll
        for (int n = 1; n <= 2 * ORDER; ++n) S[n] = fma(w, px[n], S[n]);
        const double wy = w * y;
        T[0] += wy;
#pragma unroll
        for (int n = 1; n <= ORDER; ++n) T[n] = fma(wy, px[n], T[n]);
    }
    // row taps: the sweep counts the row (row_count, before end_row)
    __device__ __forceinline__ void row_count(int n) {
        cnt = n;
        fcnt = 0.f;
    }
    // the first tap of a row run: opens the row sums (no zeroing)
    __device__ __forceinline__ void first_rt(double, double, float2 e, double dx, double dxx,
                                             float d2f, bool = true) {
        const float w32 = ex2_approx(-hl * d2f) * e.y;
        const double w = (double)w32, y = (double)e.x;
        acc.sabs = fmaf(w32, fabsf(e.x), acc.sabs);
        double px[5];
        px[1] = dx;
        px[2] = dxx;
        if (ORDER >= 2) {
            px[3] = dx * dxx;
            px[4] = dxx * dxx;
        }
        S[0] = w;
#pragma unroll
        for (int n = 1; n <= 2 * ORDER; ++n) S[n] = w * px[n];
        const double wy = w * y;
        T[0] = wy;
#pragma unroll
        for (int n = 1; n <= ORDER; ++n) T[n] = wy * px[n];
    }
    // co-sited merged sample: w = W sum 1/den, wy = W sum f_hat/den (fp32),
    // the bound's sum w |y| from W sum |f_hat|/den, count = the sensors' samples
    __device__ __forceinline__ void sample4(bool ok, float4 e, double dx, double dxx, float W) {
        W = ok ? W : 0.f;
        const double w = (double)(W * e.x), wy = (double)(W * e.y);
        acc.sabs = fmaf(W, e.z, acc.sabs);
        double px[5];
        px[1] = dx;
        px[2] = dxx;
        if (ORDER >= 2) {
            px[3] = dx * dxx;
            px[4] = dxx * dxx;
        }
        S[0] += w;
#pragma unroll
        for (int n = 1; n <= 2 * ORDER; ++n) S[n] = fma(w, px[n], S[n]);
        T[0] += wy;
#pragma unroll
        for (int n = 1; n <= ORDER; ++n) T[n] = fma(wy, px[n], T[n]);
        fcnt += ok ? e.w : 0.f;
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
        acc.count += cnt + (int)fcnt;
    }
    // CNT = false: the sweep counts the row's candidates (count_add)
    template <bool CNT = true>
    __device__ __forceinline__ void general(bool ok, double v, float iv, double dx, double dy,
                                            double dxx, double dyy, float d2f, bool = true) {
        const float w = ex2_approx(-hl * d2f) * (ok ? iv : 0.f);
        const double y = ok ? v : 0.0;
        acc.sabs = fmaf(w, fabsf((float)y), acc.sabs);
        acc.add_fast((double)w, y, dx, dy, dxx, dyy, CNT ? (ok ? 1 : 0) : 0);
    }
    __device__ __forceinline__ void count_add(int n) { acc.count += n; }
};

// The fast path's ICI variance v = sum t (phi.g)^2 is a sum of nonnegative
// terms, accumulated in float32 (HDR_VAR32, default): its relative error is
// at most (n + 3) 2^-24 for n nonzero terms (the FMA rounding per term, plus
// fl32(phi.g), its square and t), i.e. (n + 3) 2^-25 on the standard
// deviation, which ici() adds to the interval error bounds (n = the scale's
// sample count).  Values outside [1e-30, 1e37] go to the exact path.
#ifndef HDR_VAR32
#define HDR_VAR32 1
#endif
#if HDR_VAR32
using var_t = float;
__device__ __forceinline__ void var_add(float &v, float t32, double, float pf) {
    v = fmaf(t32, pf * pf, v);
}
#else
using var_t = double;
__device__ __forceinline__ void var_add(double &v, float t32, double pg, float) {
    v = fma((double)t32, pg * pg, v);
}
#endif
constexpr double VAR32_EPS_TERM = HDR_VAR32 ? 3.1e-8 : 0.0;  // (1.03 * 2^-25 per term on sd)

// Row-factored variance sweep (ICI, fast path): phi.g = c0(dy) + dx (c1(dy) + g3 dx).
// Also accumulates T = sum w |phi.g| |y| (fp32): the sharp precision bound of
// c0 (fit_precise_sharp).
template <int ORDER>
struct RowVariance {
    const double *g;
    float hl;
    bool sig;
    var_t v;
    double c0, c1;
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
    __device__ __forceinline__ void row_count(int) {}
    __device__ __forceinline__ void end_row(double, double) {}
    __device__ __forceinline__ void sample(bool ok, double y, float iv, double dx, double, double,
                                           double, float d2f, bool = true) {
        const float W = ok ? ex2_approx(-hl * d2f) : 0.f;
        const float t32 = sig ? W * W : W * W * iv;
        double pg = c0;
        if (ORDER == 1) pg = fma(dx, c1, c0);
        if (ORDER == 2) pg = fma(dx, fma(g[3], dx, c1), c0);
        if (ok) {
            const float pf = (float)pg;
            var_add(v, t32, pg, pf);
            T = fmaf(W * iv, fabsf(pf) * fabsf((float)y), T);
        }
    }
    __device__ __forceinline__ void first_rt(double dy, double dyy, float2 e, double dx,
                                             double dxx, float d2f, bool = true) {
        begin_row(dy, dyy);
        sample_rt(e, dx, dxx, d2f);
    }
    __device__ __forceinline__ void sample_rt(float2 e, double dx, double, float d2f,
                                              bool = true) {
        const float W = ex2_approx(-hl * d2f);
        // masked samples: 1/den = 0 (variance weights W^2/den vanish; sigma
        // weights W^2 need the mask)
        const float t32 = sig ? (e.y > 0.f ? W * W : 0.f) : W * W * e.y;
        double pg = c0;
        if (ORDER == 1) pg = fma(dx, c1, c0);
        if (ORDER == 2) pg = fma(dx, fma(g[3], dx, c1), c0);
        const float pf = (float)pg;
        var_add(v, t32, pg, pf);
        T = fmaf(W * e.y, fabsf(pf) * fabsf(e.x), T);
    }
    __device__ __forceinline__ void count_add(int) {}
    template <bool CNT = true>
    __device__ __forceinline__ void general(bool ok, double y, float iv, double dx, double dy,
                                            double dxx, double dyy, float d2f, bool = true) {
        const float W = ex2_approx(-hl * d2f) * (ok ? 1.f : 0.f);
        const float t32 = sig ? W * W : W * W * iv;
        double pg = g[0];
        if (ORDER >= 1) pg += dx * g[1] + dy * g[2];
        if (ORDER >= 2) pg += dxx * g[3] + (dx * dy) * g[4] + dyy * g[5];  // dx*dy: shared with the moments
        // W = 0 when !ok: both sums take zero contributions (no branch)
        const float pf = (float)pg;
        var_add(v, t32, pg, pf);
        T = fmaf(W * iv, fabsf(pf) * fabsf((float)y), T);
    }
};

// Fused traversal of ICI: the variance sweep of scale kin (samples flagged
// `inner`) and the moment sweep of the next scale k (all samples of its
// larger window) in one pass over the window of scale k.
template <int ORDER>
struct FusedVarMom {
    RowVariance<ORDER> &V;
    RowMoments<ORDER> &M;
    __device__ __forceinline__ void begin_row(double dy, double dyy) {
        V.begin_row(dy, dyy);
        M.begin_row(dy, dyy);
    }
    __device__ __forceinline__ void end_row(double dy, double dyy) {
        M.end_row(dy, dyy);
        V.end_row(dy, dyy);
    }
    __device__ __forceinline__ void row_count(int n) { M.row_count(n); }
    __device__ __forceinline__ void sample(bool ok, double v, float iv, double dx, double dy,
                                           double dxx, double dyy, float d2f, bool inner) {
        M.sample(ok, v, iv, dx, dy, dxx, dyy, d2f);
        if (inner) V.sample(ok, v, iv, dx, dy, dxx, dyy, d2f);
    }
    // rotated sensors: inner differs between the lanes of a warp, so both
    // halves run unconditionally (the variance with weight 0 outside r_kin)
    template <bool CNT = true>
    __device__ __forceinline__ void general(bool ok, double v, float iv, double dx, double dy,
                                            double dxx, double dyy, float d2f, bool inner) {
        M.template general<CNT>(ok, v, iv, dx, dy, dxx, dyy, d2f);
        V.general(ok && inner, v, iv, dx, dy, dxx, dyy, d2f);
    }
    __device__ __forceinline__ void count_add(int n) { M.count_add(n); }
    __device__ __forceinline__ void first_rt(double dy, double dyy, float2 e, double dx,
                                             double dxx, float d2f, bool inner) {
        V.begin_row(dy, dyy);
        M.first_rt(dy, dyy, e, dx, dxx, d2f);
        if (inner) V.sample_rt(e, dx, dxx, d2f);
    }
    // row taps: inner is uniform across the warp (class-uniform tap lists)
    __device__ __forceinline__ void sample_rt(float2 e, double dx, double dxx, float d2f,
                                              bool inner) {
        M.sample_rt(e, dx, dxx, d2f);
        if (inner) V.sample_rt(e, dx, dxx, d2f);
    }
};

template <class Sweep>
struct HasRows {
    static constexpr bool value = false;
};
template <int MAXC, bool BRANCHY, int RT, bool MRG4>
struct HasRows<TileSweep<MAXC, BRANCHY, RT, MRG4>> {
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
            acc.add_fast((double)w, y, dx, dy, dxx, dyy, ok ? 1 : 0);
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
    if (P.rgb) P.rgb[(size_t)pix * 3 + c] = o;
    if (P.rgb_half) P.rgb_half[(size_t)pix * 3 + c] = __half_as_ushort(__float2half_rn(o * P.half_scale));
    if (!P.diag) return;
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

}  // namespace hdrlpa
