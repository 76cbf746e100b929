// exact_ref.cuh -- the exact path's reference-order re-evaluation of one
// window, for the rare p = 3 condition decisions the float64 bounds leave
// open (solve_exact's FIT_CRITICAL).
//
// There the reference's trigonometric eigenvalue range (_kernels.py:38-71)
// can turn last-bit differences of the moment sums into percent-level
// differences of lambda_min (near-degenerate windows, acos of an argument
// within ~1e-14 of 1), so the decision depends on the summation order.  This
// re-evaluation enumerates the window's samples exactly as _fit_at walks the
// SampleIndex (radiometry.py:208-242, _kernels.py:130-182): unit cells
// row-major over floor(X), floor(Y), inside a cell the samples in
// frames_to_samples order (sensor-major, raster), weights exp(-q) / den with
// the reference's division and den, sums unfused in the reference's order,
// then _fit_at's decision and _chol_solve (ref_decide).  One sequential pass
// per lane (every lane of a group computes the same bits).
#pragma once

#include "sweeps.cuh"

namespace hdrlpa {

// f_hat and the reference's den (sigma^2 in variance mode, sqrt(sigma^2) in
// sigma mode; radiometry.py:240, _kernels.py:165-167) of sensor pixel (x, y)
__device__ __forceinline__ bool radiance_den(const DevSensor &S, int x, int y, int use_sigma,
                                             double &f, double &den) {
    if (x < 0 || y < 0 || x >= S.width || y >= S.height) return false;
    const int raw = (int)__ldg(S.raw + (size_t)y * S.pitch + x);
    if (raw >= S.sat) return false;
    const size_t i = (size_t)y * S.width + x;
    if (S.defective && __ldg(S.defective + i)) return false;
    const double b = S.bias_p ? __ldg(S.bias_p + i) : S.bias;
    const double a = S.nonuni_p ? __ldg(S.nonuni_p + i) : S.nonuni;
    const double vr = S.readvar_p ? __ldg(S.readvar_p + i) : S.readvar;
    double sg;
    radiometry_sigma(S, raw, b, a, vr, f, sg);
    den = __dmul_rn(sg, sg);
    if (use_sigma) den = __dsqrt_rn(den);
    return true;
}

// _fit_at (_kernels.py:104-200) at query (qx, qy) with window H^-1 = (h11,
// h12; h12, h22) and radius r, over channel c of the rig's raw frames in the
// reference's sample order.  FIT_OK (coef = C0, C1, C2) or FIT_FAIL.
template <int ORDER>
__device__ int ref_fit_at(const DevParams &P, int c, double qx, double qy, double h11, double h12,
                          double h22, double radius, double *coef, double *g = nullptr) {
    constexpr int PN = NC<ORDER>::P;
    double A[6][6], rhs[6];
#pragma unroll
    for (int a = 0; a < PN; ++a) {
        rhs[a] = 0.0;
#pragma unroll
        for (int b = 0; b < PN; ++b) A[a][b] = 0.0;
    }
    int count = 0;
    const double r2 = __dmul_rn(radius, radius);
    const int gx0 = (int)floor(qx - radius), gx1 = (int)floor(qx + radius);
    const int gy0 = (int)floor(qy - radius), gy1 = (int)floor(qy + radius);
    const double h12x2 = __dmul_rn(2.0, h12);
    for (int gy = gy0; gy <= gy1; ++gy)
        for (int gx = gx0; gx <= gx1; ++gx)
            for (int s = 0; s < P.n_sensors; ++s) {
                const DevSensor &S = P.s[s];
                const int pm = S.phmask[c];
                if (!pm) continue;
                // sensor pixels whose position can fall in the unit cell: the
                // bounding box of the cell's preimage (its four corners through
                // N = T_lin^-1), widened by 1e-6 px against rounding
                int xlo = INT_MAX, xhi = INT_MIN, ylo = INT_MAX, yhi = INT_MIN;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double u = (double)(gx + (k & 1)) - S.T[2];
                    const double v = (double)(gy + (k >> 1)) - S.T[5];
                    const double sx = S.N[0] * u + S.N[1] * v, sy = S.N[2] * u + S.N[3] * v;
                    xlo = min(xlo, (int)ceil(sx - 1e-6));
                    xhi = max(xhi, (int)floor(sx + 1e-6));
                    ylo = min(ylo, (int)ceil(sy - 1e-6));
                    yhi = max(yhi, (int)floor(sy + 1e-6));
                }
                xlo = max(xlo, 0);
                ylo = max(ylo, 0);
                xhi = min(xhi, S.width - 1);
                yhi = min(yhi, S.height - 1);
                for (int y = ylo; y <= yhi; ++y) {
                    const double yd = (double)y;
                    const double t1y = __dmul_rn(S.T[1], yd), t4y = __dmul_rn(S.T[4], yd);
                    for (int x = xlo; x <= xhi; ++x) {
                        if (!((pm >> (((y & 1) << 1) | (x & 1))) & 1)) continue;
                        const double xd = (double)x;
                        const double X = __dadd_rn(__dadd_rn(__dmul_rn(S.T[0], xd), t1y), S.T[2]);
                        const double Y = __dadd_rn(__dadd_rn(__dmul_rn(S.T[3], xd), t4y), S.T[5]);
                        if ((int)floor(X) != gx || (int)floor(Y) != gy) continue;  // another cell
                        double f, den;
                        if (!radiance_den(S, x, y, P.use_sigma, f, den)) continue;
                        const double dx = __dsub_rn(X, qx), dy = __dsub_rn(Y, qy);
                        if (__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) > r2) continue;
                        const double q = __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(h11, dx), dx),
                                                             __dmul_rn(__dmul_rn(h12x2, dx), dy)),
                                                   __dmul_rn(__dmul_rn(h22, dy), dy));
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
                        for (int a = 0; a < PN; ++a) {
                            const double wa = __dmul_rn(w, phi[a]);
                            rhs[a] = __dadd_rn(rhs[a], __dmul_rn(wa, f));
#pragma unroll
                            for (int b = a; b < PN; ++b)
                                A[a][b] = __dadd_rn(A[a][b], __dmul_rn(wa, phi[b]));
                        }
                        ++count;
                    }
                }
            }
    const int st = ref_decide<PN>(A, rhs, count, P.cond, coef);
    if (st == FIT_OK && g) {  // g = A^-1 e1 (the ICI variance), same factorisation
        double e1[6] = {1.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        if (!chol_solve_ref<PN>(A, e1, g)) return FIT_FAIL;
    }
    return st;
}

// A FIT_CRITICAL decision of solve_exact settled in the reference's order:
// FIT_OK (the coefficients replaced by the reference-order ones) or FIT_FAIL.
template <int ORDER>
__device__ __forceinline__ int settle_critical(const DevParams &P, int c, double qx, double qy,
                                               double h11, double h12, double h22, double r,
                                               Fit &fit) {
    double coef[6], g[6];
    if (ref_fit_at<ORDER>(P, c, qx, qy, h11, h12, h22, r, coef, g) != FIT_OK) return FIT_FAIL;
    fit.c0 = coef[0];
    fit.c1 = ORDER >= 1 ? coef[1] : 0.0;
    fit.c2 = ORDER >= 1 ? coef[2] : 0.0;
#pragma unroll
    for (int a = 0; a < NC<ORDER>::P; ++a) fit.g[a] = g[a];
    return FIT_OK;
}

}  // namespace hdrlpa
