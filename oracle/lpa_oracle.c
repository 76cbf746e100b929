/*
 * lpa_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker and the CPU
 * baseline arm of bench.py).  Nothing in the product path links, loads or
 * calls this file.
 *
 * A plain-C, float64 restatement of the reference's CPU path
 *   hdrfuse.frames_to_samples  (pkg/src/hdrfuse/radiometry.py:303-349)
 *   hdrfuse.SampleIndex        (pkg/src/hdrfuse/radiometry.py:208-242)
 *   hdrfuse.reconstruct_frame  (pkg/src/hdrfuse/lpa.py:379-433)
 *   _kernels.lpa_evaluate      (pkg/src/hdrfuse/_kernels.py:203-300)
 *   _kernels._fit_at           (pkg/src/hdrfuse/_kernels.py:104-200)
 *   _kernels._sym_eig_range    (pkg/src/hdrfuse/_kernels.py:26-73)
 *   _kernels._chol_solve       (pkg/src/hdrfuse/_kernels.py:76-101)
 * plus the ICI scale-selection extension specified in DESIGN.md ("ICI
 * spec"), which the reference does not have (parity for ICI is pinned only
 * by this oracle's own known-answer tests).
 *
 * Floating-point operations are written in the reference's evaluation
 * order and the file is compiled with -ffp-contract=off, so for orders 0
 * and 1 the outputs reproduce the reference bit for bit (checked against
 * the reference's golden SHA-256, tests/test_oracle_golden.py).  For
 * order 2 the reference obtains (lmin, lmax) from LAPACK dsyevd through
 * numba (_kernels.py:72); the Python wrapper hands this file the same
 * scipy.linalg.cython_lapack dsyevd entry point, so the accept/reject
 * decision is the reference's own.  Without it a cyclic Jacobi is used.
 *
 * Parallelism: OpenMP over queries (the reference's numba prange over
 * query chunks, _kernels.py:249); outputs are per query, so results are
 * identical at any thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OK 0
#define TOO_FEW 1
#define ILL 2

typedef void (*dsyevd_fn)(char *, char *, int *, double *, int *, double *,
                          double *, int *, int *, int *, int *);
static dsyevd_fn g_dsyevd = NULL;

void oracle_set_dsyevd(void *fn) { g_dsyevd = (dsyevd_fn)fn; }
int oracle_has_dsyevd(void) { return g_dsyevd != NULL; }

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* one sensor: raw frame + capture parameters + calibration (planes or scalars) */
typedef struct {
    int width, height;
    const uint16_t *raw;         /* height*width, row-major */
    int saturation_level;
    double exposure_time, gain, exposure_scaling;
    double T[6];                 /* 2x3 row-major affine, sensor (x,y) -> reference */
    int tile[4];                 /* channel at [(y%2)*2 + x%2] (bayer.py:24-29) */
    const double *bias;          /* nullable plane; else bias_s */
    const double *readvar;
    const double *nonuni;
    double bias_s, readvar_s, nonuni_s;
    const uint8_t *defective;    /* nullable, 1 = discard (radiometry.py:316-317) */
    int sensor_id;               /* SensorConfig.sensor_id (radiometry.py:335) */
} OSensor;

typedef struct {
    double x, y, v, var;         /* packed row (radiometry.py:238-242) */
} Row;

typedef struct {
    int64_t n;
    int x0, y0, nx, ny;
    int64_t *cell_start;
    Row *packed;
} OIndex;

/* --------------------------------------------------------------------------
 * Radiometry (radiometry.py:264-336).  Returns 1 if the pixel yields a sample.
 * ------------------------------------------------------------------------ */
static int pixel_sample(const OSensor *s, int64_t i, double *X, double *Y,
                        double *val, double *sig, int *chan) {
    int w = s->width;
    uint16_t y = s->raw[i];
    if ((int)y >= s->saturation_level) return 0;              /* :298-300, :315 */
    if (s->defective && s->defective[i]) return 0;            /* :316-317 */
    int64_t py = i / w, px = i % w;
    double xd = (double)px, yd = (double)py;
    /* apply_transform :79-84, T00*x + T01*y + T02 evaluated left to right */
    *X = s->T[0] * xd + s->T[1] * yd + s->T[2];
    *Y = s->T[3] * xd + s->T[4] * yd + s->T[5];
    double b = s->bias ? s->bias[i] : s->bias_s;
    double a = s->nonuni ? s->nonuni[i] : s->nonuni_s;
    double vr = s->readvar ? s->readvar[i] : s->readvar_s;
    double g = s->gain, t = s->exposure_time, n = s->exposure_scaling;
    double denom = g * t * n * a;                              /* :264-268 */
    double f = ((double)y - b) / denom;                        /* :271-279 */
    double d2 = denom * denom;
    double shot = g * g * t * a * n * (f > 0.0 ? f : 0.0);     /* :294 */
    double var = (shot + vr) / d2;                             /* :295 */
    double qv = (1.0 / 12.0) / d2;                             /* :327 */
    double m = var;
    if (!(var >= qv)) m = qv;     /* np.maximum(variances, quant_var), no NaNs here */
    *val = f;
    *sig = sqrt(m);                                            /* :328 */
    *chan = s->tile[(py % 2) * 2 + (px % 2)];                  /* bayer.py:54-59 */
    return 1;
}

/* Per-sample export for radiometry parity tests: arrays sized to the total
 * pixel count; returns the number of samples written (sensor-major, raster). */
int64_t oracle_frames_to_samples(const OSensor *sensors, int n_sensors,
                                 double *pos, uint8_t *chan, double *val,
                                 double *sig, int32_t *sid) {
    int64_t k = 0;
    for (int si = 0; si < n_sensors; ++si) {
        const OSensor *s = &sensors[si];
        int64_t npx = (int64_t)s->width * s->height;
        for (int64_t i = 0; i < npx; ++i) {
            double X, Y, v, sg;
            int c;
            if (!pixel_sample(s, i, &X, &Y, &v, &sg, &c)) continue;
            pos[2 * k] = X;
            pos[2 * k + 1] = Y;
            chan[k] = (uint8_t)c;
            val[k] = v;
            sig[k] = sg;
            sid[k] = sensors[si].sensor_id;  /* radiometry.py:335 */
            ++k;
        }
    }
    return k;
}

/* SampleIndex (radiometry.py:218-242): unit-cell grid over one channel, stable
 * counting sort by cell == np.argsort(kind="stable"). */
static void build_index(const OSensor *sensors, int n_sensors, int channel, OIndex *ix) {
    int64_t n = 0;
    for (int si = 0; si < n_sensors; ++si) {
        const OSensor *s = &sensors[si];
        int64_t npx = (int64_t)s->width * s->height;
        for (int64_t i = 0; i < npx; ++i) {
            double X, Y, v, sg;
            int c;
            if (pixel_sample(s, i, &X, &Y, &v, &sg, &c) && c == channel) ++n;
        }
    }
    ix->n = n;
    Row *rows = (Row *)malloc(sizeof(Row) * (n ? n : 1));
    int64_t k = 0;
    double xmin = INFINITY, xmax = -INFINITY, ymin = INFINITY, ymax = -INFINITY;
    for (int si = 0; si < n_sensors; ++si) {
        const OSensor *s = &sensors[si];
        int64_t npx = (int64_t)s->width * s->height;
        for (int64_t i = 0; i < npx; ++i) {
            double X, Y, v, sg;
            int c;
            if (!pixel_sample(s, i, &X, &Y, &v, &sg, &c) || c != channel) continue;
            rows[k].x = X;
            rows[k].y = Y;
            rows[k].v = v;
            rows[k].var = sg * sg;                             /* sigmas ** 2, :240 */
            if (X < xmin) xmin = X;
            if (X > xmax) xmax = X;
            if (Y < ymin) ymin = Y;
            if (Y > ymax) ymax = Y;
            ++k;
        }
    }
    if (n) {
        ix->x0 = (int)floor(xmin);
        ix->y0 = (int)floor(ymin);
        ix->nx = (int)floor(xmax) - ix->x0 + 1;
        ix->ny = (int)floor(ymax) - ix->y0 + 1;
    } else {
        ix->x0 = ix->y0 = 0;
        ix->nx = ix->ny = 1;
    }
    int64_t ncell = (int64_t)ix->nx * ix->ny;
    ix->cell_start = (int64_t *)calloc(ncell + 1, sizeof(int64_t));
    int64_t *cellof = (int64_t *)malloc(sizeof(int64_t) * (n ? n : 1));
    for (int64_t j = 0; j < n; ++j) {
        int64_t c = ((int64_t)floor(rows[j].y) - ix->y0) * ix->nx +
                    ((int64_t)floor(rows[j].x) - ix->x0);
        cellof[j] = c;
        ix->cell_start[c + 1]++;
    }
    for (int64_t c = 0; c < ncell; ++c) ix->cell_start[c + 1] += ix->cell_start[c];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (ncell ? ncell : 1));
    memcpy(fill, ix->cell_start, sizeof(int64_t) * ncell);
    ix->packed = (Row *)malloc(sizeof(Row) * (n ? n : 1));
    for (int64_t j = 0; j < n; ++j) ix->packed[fill[cellof[j]]++] = rows[j];
    free(fill);
    free(cellof);
    free(rows);
}

static void free_index(OIndex *ix) {
    free(ix->cell_start);
    free(ix->packed);
}

/* --------------------------------------------------------------------------
 * _sym_eig_range (_kernels.py:26-73)
 * ------------------------------------------------------------------------ */
static void jacobi_eig_range(const double A[6][6], int p, double *lmin, double *lmax) {
    double M[6][6];
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j) M[i][j] = A[i][j];
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0;
        for (int i = 0; i < p; ++i)
            for (int j = i + 1; j < p; ++j) off += M[i][j] * M[i][j];
        if (off == 0.0) break;
        for (int pp = 0; pp < p; ++pp)
            for (int q = pp + 1; q < p; ++q) {
                if (M[pp][q] == 0.0) continue;
                double theta = (M[q][q] - M[pp][pp]) / (2.0 * M[pp][q]);
                double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < p; ++k) {
                    double mkp = M[k][pp], mkq = M[k][q];
                    M[k][pp] = c * mkp - s * mkq;
                    M[k][q] = s * mkp + c * mkq;
                }
                for (int k = 0; k < p; ++k) {
                    double mpk = M[pp][k], mqk = M[q][k];
                    M[pp][k] = c * mpk - s * mqk;
                    M[q][k] = s * mpk + c * mqk;
                }
            }
    }
    double lo = M[0][0], hi = M[0][0];
    for (int i = 1; i < p; ++i) {
        if (M[i][i] < lo) lo = M[i][i];
        if (M[i][i] > hi) hi = M[i][i];
    }
    *lmin = lo;
    *lmax = hi;
}

static void sym_eig_range(const double A[6][6], int p, double *lmin, double *lmax) {
    if (p == 1) {
        *lmin = *lmax = A[0][0];
        return;
    }
    if (p == 3) {
        double a11 = A[0][0], a22 = A[1][1], a33 = A[2][2];
        double a12 = A[0][1], a13 = A[0][2], a23 = A[1][2];
        double q = (a11 + a22 + a33) / 3.0;
        double p1 = a12 * a12 + a13 * a13 + a23 * a23;
        double e1 = a11 - q, e2 = a22 - q, e3 = a33 - q;
        double p2 = e1 * e1 + e2 * e2 + e3 * e3 + 2.0 * p1;   /* (x)**2 == x*x */
        double scale = fabs(a11) + fabs(a22) + fabs(a33) + 1e-300;
        if (p2 <= 1e-30 * scale * scale) {
            *lmin = *lmax = q;
            return;
        }
        double pp = sqrt(p2 / 6.0);
        double b11 = (a11 - q) / pp, b22 = (a22 - q) / pp, b33 = (a33 - q) / pp;
        double b12 = a12 / pp, b13 = a13 / pp, b23 = a23 / pp;
        double detb = b11 * (b22 * b33 - b23 * b23) - b12 * (b12 * b33 - b23 * b13) +
                      b13 * (b12 * b23 - b22 * b13);
        double r = detb / 2.0;
        if (r < -1.0)
            r = -1.0;
        else if (r > 1.0)
            r = 1.0;
        double phi = acos(r) / 3.0;
        *lmax = q + 2.0 * pp * cos(phi);
        *lmin = q + 2.0 * pp * cos(phi + 2.0 * M_PI / 3.0);
        return;
    }
    if (g_dsyevd) {
        /* same call numba makes for np.linalg.eigvalsh: JOBZ='N', UPLO='L',
         * workspace query first (numba/_lapack.c numba_ez_rsyevd) */
        double a[36], w[6], wq;
        int n = p, lda = p, lwork = -1, liwork = -1, iwq, info = 0;
        char jobz = 'N', uplo = 'L';
        for (int j = 0; j < p; ++j)
            for (int i = 0; i < p; ++i) a[j * p + i] = A[i][j];
        g_dsyevd(&jobz, &uplo, &n, a, &lda, w, &wq, &lwork, &iwq, &liwork, &info);
        lwork = (int)wq;
        liwork = iwq;
        double *work = (double *)malloc(sizeof(double) * (lwork > 1 ? lwork : 1));
        int *iwork = (int *)malloc(sizeof(int) * (liwork > 1 ? liwork : 1));
        g_dsyevd(&jobz, &uplo, &n, a, &lda, w, work, &lwork, iwork, &liwork, &info);
        free(work);
        free(iwork);
        *lmin = w[0];
        *lmax = w[p - 1];
        return;
    }
    jacobi_eig_range(A, p, lmin, lmax);
}

/* _chol_solve (_kernels.py:76-101) */
static int chol_solve(const double A[6][6], const double *b, int p, double *coef,
                      double L[6][6]) {
    double work[6];
    for (int i = 0; i < p; ++i)
        for (int j = 0; j <= i; ++j) {
            double s = A[i][j];
            for (int k = 0; k < j; ++k) s -= L[i][k] * L[j][k];
            if (i == j) {
                if (s <= 0.0) return 0;
                L[i][i] = sqrt(s);
            } else {
                L[i][j] = s / L[j][j];
            }
        }
    for (int i = 0; i < p; ++i) {
        double s = b[i];
        for (int k = 0; k < i; ++k) s -= L[i][k] * work[k];
        work[i] = s / L[i][i];
    }
    for (int i = p - 1; i >= 0; --i) {
        double s = work[i];
        for (int k = i + 1; k < p; ++k) s -= L[k][i] * coef[k];
        coef[i] = s / L[i][i];
    }
    return 1;
}

typedef struct {
    double coef[6];
    double A[6][6];
    double rhs[6];
    double L[6][6];
    int count;
} FitScratch;

/* _fit_at (_kernels.py:104-200) */
static int fit_at(double qx, double qy, double h11, double h12, double h22,
                  double radius, int order, double cond_threshold, const OIndex *ix,
                  int use_sigma, FitScratch *S) {
    int p = (order + 1) * (order + 2) / 2;
    double phi[6];
    memset(S->A, 0, sizeof(S->A));
    memset(S->rhs, 0, sizeof(S->rhs));
    int count = 0;
    double r2 = radius * radius;
    int cx_lo = (int)floor(qx - radius) - ix->x0;
    int cx_hi = (int)floor(qx + radius) - ix->x0;
    int cy_lo = (int)floor(qy - radius) - ix->y0;
    int cy_hi = (int)floor(qy + radius) - ix->y0;
    if (cx_lo < 0) cx_lo = 0;
    if (cy_lo < 0) cy_lo = 0;
    if (cx_hi >= ix->nx) cx_hi = ix->nx - 1;
    if (cy_hi >= ix->ny) cy_hi = ix->ny - 1;
    for (int cy = cy_lo; cy <= cy_hi; ++cy) {
        int64_t row = (int64_t)cy * ix->nx;
        for (int cx = cx_lo; cx <= cx_hi; ++cx) {
            int64_t cell = row + cx;
            for (int64_t k = ix->cell_start[cell]; k < ix->cell_start[cell + 1]; ++k) {
                const Row *R = &ix->packed[k];
                double dx = R->x - qx;
                double dy = R->y - qy;
                if (dx * dx + dy * dy > r2) continue;
                double q = h11 * dx * dx + 2.0 * h12 * dx * dy + h22 * dy * dy;
                double den = R->var;
                if (use_sigma) den = sqrt(den);
                double w = exp(-q) / den;
                phi[0] = 1.0;
                if (order >= 1) {
                    phi[1] = dx;
                    phi[2] = dy;
                }
                if (order >= 2) {
                    phi[3] = dx * dx;
                    phi[4] = dx * dy;
                    phi[5] = dy * dy;
                }
                for (int a = 0; a < p; ++a) {
                    double wa = w * phi[a];
                    S->rhs[a] += wa * R->v;
                    for (int b = a; b < p; ++b) S->A[a][b] += wa * phi[b];
                }
                ++count;
            }
        }
    }
    S->count = count;
    if (count < p) return TOO_FEW;
    for (int a = 0; a < p; ++a)
        for (int b = a + 1; b < p; ++b) S->A[b][a] = S->A[a][b];
    if (p == 1) {
        if (S->A[0][0] <= 0.0) return TOO_FEW;
        S->coef[0] = S->rhs[0] / S->A[0][0];
        return OK;
    }
    double lmin, lmax;
    sym_eig_range(S->A, p, &lmin, &lmax);
    if (lmin <= 0.0 || lmax > cond_threshold * lmin) return ILL;
    if (!chol_solve(S->A, S->rhs, p, S->coef, S->L)) return ILL;
    return OK;
}

/* variance of the fitted constant term (ICI spec): v = sum w^2 var (phi.g)^2,
 * g = A^{-1} e1, over the same window as the fit. */
static double fit_variance(double qx, double qy, double h11, double h12, double h22,
                           double radius, int order, const OIndex *ix, int use_sigma,
                           const FitScratch *S) {
    int p = (order + 1) * (order + 2) / 2;
    double g[6], z[6];
    if (p == 1) {
        g[0] = 1.0 / S->A[0][0];
    } else {
        for (int i = 0; i < p; ++i) {
            double s = (i == 0) ? 1.0 : 0.0;
            for (int k = 0; k < i; ++k) s -= S->L[i][k] * z[k];
            z[i] = s / S->L[i][i];
        }
        for (int i = p - 1; i >= 0; --i) {
            double s = z[i];
            for (int k = i + 1; k < p; ++k) s -= S->L[k][i] * g[k];
            g[i] = s / S->L[i][i];
        }
    }
    double r2 = radius * radius, v = 0.0;
    int cx_lo = (int)floor(qx - radius) - ix->x0;
    int cx_hi = (int)floor(qx + radius) - ix->x0;
    int cy_lo = (int)floor(qy - radius) - ix->y0;
    int cy_hi = (int)floor(qy + radius) - ix->y0;
    if (cx_lo < 0) cx_lo = 0;
    if (cy_lo < 0) cy_lo = 0;
    if (cx_hi >= ix->nx) cx_hi = ix->nx - 1;
    if (cy_hi >= ix->ny) cy_hi = ix->ny - 1;
    for (int cy = cy_lo; cy <= cy_hi; ++cy) {
        int64_t row = (int64_t)cy * ix->nx;
        for (int cx = cx_lo; cx <= cx_hi; ++cx) {
            int64_t cell = row + cx;
            for (int64_t k = ix->cell_start[cell]; k < ix->cell_start[cell + 1]; ++k) {
                const Row *R = &ix->packed[k];
                double dx = R->x - qx;
                double dy = R->y - qy;
                if (dx * dx + dy * dy > r2) continue;
                double q = h11 * dx * dx + 2.0 * h12 * dx * dy + h22 * dy * dy;
                double den = R->var;
                if (use_sigma) den = sqrt(den);
                double w = exp(-q) / den;
                double pg = g[0];
                if (order >= 1) pg += dx * g[1] + dy * g[2];
                if (order >= 2) pg += dx * dx * g[3] + dx * dy * g[4] + dy * dy * g[5];
                v += w * w * R->var * (pg * pg);
            }
        }
    }
    return v;
}

/* Outcome code per query: 0xFF = NaN (no order succeeded); otherwise
 * order*16 + radius-step (0 = base radius) of the accepted fit. */
#define OUT_NAN 0xFF

/* lpa_evaluate body for one isotropic query (_kernels.py:257-300; the
 * two_phase branch is CALPA-only and not on this path). */
static void ladder_eval(double qx, double qy, double hinv, double r0, int order0,
                        double max_radius, double cond_threshold, const OIndex *ix,
                        int use_sigma, FitScratch *S, double *val, double *gx, double *gy,
                        uint8_t *outcome, uint16_t *count) {
    for (int order = order0; order >= 0; --order) {
        double r = r0;
        if (r > max_radius) r = max_radius;
        int step = 0;
        for (;;) {
            int st = fit_at(qx, qy, hinv, 0.0, hinv, r, order, cond_threshold, ix, use_sigma, S);
            if (st == OK) {
                *val = S->coef[0];
                if (order >= 1) {
                    *gx = S->coef[1];
                    *gy = S->coef[2];
                } else {
                    *gx = NAN;
                    *gy = NAN;
                }
                *outcome = (uint8_t)(order * 16 + (step < 15 ? step : 15));
                *count = (uint16_t)(S->count < 65535 ? S->count : 65535);
                return;
            }
            if (r >= max_radius * (1.0 - 1e-12)) break;
            r = r * 1.5;
            if (r > max_radius) r = max_radius;       /* min(r*1.5, max_radius) */
            ++step;
        }
    }
    *val = NAN;
    *gx = NAN;
    *gy = NAN;
    *outcome = OUT_NAN;
    *count = 0;
}

/*
 * One channel over an output grid.
 *   xs (out_w), ys (out_h): query coordinates (lpa.py:213-224, computed by caller)
 *   n_scales == 1: fixed-scale LPA at hinv[0], r0[0] (lpa.py:322-376)
 *   n_scales  > 1: ICI over hinv[k], rk[k]
 * Outputs (out_h*out_w, row-major): val/gx/gy float64 (unclamped), outcome u8,
 * scale index u8.
 */
int oracle_reconstruct_channel(const OSensor *sensors, int n_sensors, int channel,
                               const double *xs, int out_w, const double *ys, int out_h,
                               int order, int n_scales, const double *hinv, const double *rk,
                               double max_radius, double cond_threshold, int use_sigma,
                               double gamma, int n_threads, double *val, double *gx,
                               double *gy, uint8_t *outcome, uint8_t *scale_idx,
                               uint16_t *count) {
    OIndex ix;
    build_index(sensors, n_sensors, channel, &ix);
    int64_t m = (int64_t)out_w * out_h;
    if (ix.n == 0) {                                            /* lpa.py:346-350 */
        for (int64_t i = 0; i < m; ++i) {
            val[i] = gx[i] = gy[i] = NAN;
            outcome[i] = OUT_NAN;
            scale_idx[i] = 0;
            count[i] = 0;
        }
        free_index(&ix);
        return 0;
    }
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#endif
#pragma omp parallel
    {
        FitScratch S, best;
#pragma omp for schedule(dynamic, 256)
        for (int64_t i = 0; i < m; ++i) {
            double qx = xs[i % out_w], qy = ys[i / out_w];
            scale_idx[i] = 0;
            if (n_scales <= 1) {
                ladder_eval(qx, qy, hinv[0], rk[0], order, max_radius, cond_threshold, &ix,
                            use_sigma, &S, &val[i], &gx[i], &gy[i], &outcome[i], &count[i]);
                continue;
            }
            /* ICI: k = 0 must succeed at the requested order, else reference ladder */
            double r0 = rk[0] > max_radius ? max_radius : rk[0];
            int st = fit_at(qx, qy, hinv[0], 0.0, hinv[0], r0, order, cond_threshold, &ix,
                            use_sigma, &S);
            if (st != OK) {
                ladder_eval(qx, qy, hinv[0], rk[0], order, max_radius, cond_threshold, &ix,
                            use_sigma, &S, &val[i], &gx[i], &gy[i], &outcome[i], &count[i]);
                continue;
            }
            double v = fit_variance(qx, qy, hinv[0], 0.0, hinv[0], r0, order, &ix, use_sigma, &S);
            double sd = sqrt(v);
            double L = S.coef[0] - gamma * sd, U = S.coef[0] + gamma * sd;
            best = S;
            int kbest = 0;
            for (int k = 1; k < n_scales; ++k) {
                double r = rk[k] > max_radius ? max_radius : rk[k];
                st = fit_at(qx, qy, hinv[k], 0.0, hinv[k], r, order, cond_threshold, &ix,
                            use_sigma, &S);
                if (st != OK) break;
                v = fit_variance(qx, qy, hinv[k], 0.0, hinv[k], r, order, &ix, use_sigma, &S);
                sd = sqrt(v);
                double lo = S.coef[0] - gamma * sd, hi = S.coef[0] + gamma * sd;
                if (lo > L) L = lo;
                if (hi < U) U = hi;
                if (L > U) break;
                best = S;
                kbest = k;
            }
            val[i] = best.coef[0];
            if (order >= 1) {
                gx[i] = best.coef[1];
                gy[i] = best.coef[2];
            } else {
                gx[i] = gy[i] = NAN;
            }
            outcome[i] = (uint8_t)(order * 16);
            scale_idx[i] = (uint8_t)kbest;
            count[i] = (uint16_t)(best.count < 65535 ? best.count : 65535);
        }
    }
    free_index(&ix);
    return 0;
}


/* ==========================================================================
 * CALPA (structure-adaptive second pass, reference steering.py)
 * ======================================================================== */

/* steering_field_kernel (_kernels.py:310-392): per output pixel, weighted
 * gradient energy over a (2 half + 1)^2 window -> (theta, sigma, gamma).
 * gx, gy are the gradient planes already divided by gradient_scale. */
void oracle_steering_field(const double *gx, const double *gy, int w, int h, int half,
                           double wstd, double lam1, double lam2, double alpha,
                           double sigma_max, double *theta, double *sigma, double *gamma,
                           int n_threads) {
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#endif
#pragma omp parallel for schedule(dynamic, 4)
    for (int yy = 0; yy < h; ++yy) {
        for (int xx = 0; xx < w; ++xx) {
            double s11 = 0.0, s12 = 0.0, s22 = 0.0;
            int n = 0;
            for (int dy = -half; dy <= half; ++dy) {
                int iy = yy + dy;
                if (iy < 0 || iy >= h) continue;
                for (int dx = -half; dx <= half; ++dx) {
                    int ix = xx + dx;
                    if (ix < 0 || ix >= w) continue;
                    double g1 = gx[(int64_t)iy * w + ix], g2 = gy[(int64_t)iy * w + ix];
                    if (!(isfinite(g1) && isfinite(g2))) continue;
                    double wgt = exp(-(double)(dx * dx + dy * dy) / (2.0 * wstd * wstd));
                    s11 += wgt * g1 * g1;
                    s12 += wgt * g1 * g2;
                    s22 += wgt * g2 * g2;
                    ++n;
                }
            }
            int64_t o = (int64_t)yy * w + xx;
            if (n == 0) {
                theta[o] = 0.0;
                sigma[o] = 1.0;
                gamma[o] = 1.0;
                continue;
            }
            /* _eig2_minmax (_kernels.py:303-307) */
            double m = 0.5 * (s11 + s22);
            double d = hypot(0.5 * (s11 - s22), s12);
            double lmin = m - d, lmax = m + d;
            if (lmin < 0.0) lmin = 0.0;
            double s1 = sqrt(lmax), s2 = sqrt(lmin);
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
            double denom = s2 + lam1, sg;
            if (denom == 0.0)
                sg = (s1 + lam1 == 0.0) ? 1.0 : sigma_max;
            else
                sg = (s1 + lam1) / denom;
            if (sg > sigma_max) sg = sigma_max;
            theta[o] = th;
            sigma[o] = sg;
            gamma[o] = pow((s1 * s2 + lam2) / n, alpha);
        }
    }
}

/* lpa_evaluate with two_phase (_kernels.py:257-300): per order, the
 * anisotropic window (per-query Hinv, r0) then the isotropic one, each with
 * the radius ladder. */
int oracle_reconstruct_channel_steered(const OSensor *sensors, int n_sensors, int channel,
                                       const double *xs, int out_w, const double *ys,
                                       int out_h, int order0, const double *an_h11,
                                       const double *an_h12, const double *an_h22,
                                       const double *an_r0, double iso_hinv, double iso_r0,
                                       double max_radius, double cond_threshold,
                                       int use_sigma, int n_threads, double *val, double *gx,
                                       double *gy, uint8_t *outcome) {
    OIndex ix;
    build_index(sensors, n_sensors, channel, &ix);
    int64_t m = (int64_t)out_w * out_h;
    if (ix.n == 0) {
        for (int64_t i = 0; i < m; ++i) {
            val[i] = gx[i] = gy[i] = NAN;
            outcome[i] = OUT_NAN;
        }
        free_index(&ix);
        return 0;
    }
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#endif
#pragma omp parallel
    {
        FitScratch S;
#pragma omp for schedule(dynamic, 256)
        for (int64_t i = 0; i < m; ++i) {
            double qx = xs[i % out_w], qy = ys[i / out_w];
            int done = 0;
            for (int order = order0; order >= 0 && !done; --order) {
                for (int phase = 0; phase < 2 && !done; ++phase) {
                    double h11, h12, h22, r;
                    if (phase == 0) {
                        h11 = an_h11[i];
                        h12 = an_h12[i];
                        h22 = an_h22[i];
                        r = an_r0[i];
                    } else {
                        h11 = iso_hinv;
                        h12 = 0.0;
                        h22 = iso_hinv;
                        r = iso_r0;
                    }
                    if (r > max_radius) r = max_radius;
                    int step = 0;
                    for (;;) {
                        int st = fit_at(qx, qy, h11, h12, h22, r, order, cond_threshold, &ix,
                                        use_sigma, &S);
                        if (st == OK) {
                            val[i] = S.coef[0];
                            if (order >= 1) {
                                gx[i] = S.coef[1];
                                gy[i] = S.coef[2];
                            } else {
                                gx[i] = gy[i] = NAN;
                            }
                            outcome[i] = (uint8_t)(order * 16 + phase * 8 + (step < 7 ? step : 7));
                            done = 1;
                            break;
                        }
                        if (r >= max_radius * (1.0 - 1e-12)) break;
                        r = r * 1.5;
                        if (r > max_radius) r = max_radius;
                        ++step;
                    }
                }
            }
            if (!done) {
                val[i] = gx[i] = gy[i] = NAN;
                outcome[i] = OUT_NAN;
            }
        }
    }
    free_index(&ix);
    return 0;
}
