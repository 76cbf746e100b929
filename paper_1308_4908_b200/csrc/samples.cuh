// samples.cuh -- scattered-sample mode: lpa_evaluate over a CSR SampleIndex.
#pragma once

#include "config.cuh"

namespace hdrlpa {

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
    // the cells [cx_lo, cx_hi] of one cell row are consecutive in the CSR
    // order, so their rows form ONE range: the same samples in the same order
    // as the reference's cell-by-cell loop, without the per-cell loop (whose
    // lane-dependent trip counts left ~40 % of each warp idle)
    for (int cy = cy_lo; cx_lo <= cx_hi && cy <= cy_hi; ++cy) {
        const int64_t row = (int64_t)cy * ix.nx;
        {
            const int64_t k1 = ix.cell_start[row + cx_hi + 1];
            for (int64_t k = ix.cell_start[row + cx_lo]; k < k1; ++k) {
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
    return ref_decide<P>(A, rhs, count, cond, coef);
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

}  // namespace hdrlpa
