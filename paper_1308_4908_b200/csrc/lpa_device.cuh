// lpa_device.cuh -- device-side building blocks of the unified HDR LPA operator
// (sm_100a).  Reference semantics cited as pkg/src/hdrfuse/<file>:<line>.
//
// Precision design:
//   * sample positions, offsets d = X - q and the support test |d|^2 > r^2 are
//     float64 in the reference's exact operation order (no FMA contraction:
//     __dmul_rn/__dadd_rn), so the sample SET of every window is the
//     reference's, bit for bit;
//   * radiance f_hat and the inverse weight denominator are rounded to fp32
//     once per staged pixel; the Gaussian window is fp32 (MUFU ex2);
//   * the normal equations are accumulated in float64 (DFMA) for order >= 1
//     -- SURVEY.md s6.3 measured that fp32 sums break the 1e-4 parity bar --
//     and solved by an in-register fp64 Cholesky.  Order 0 accumulates fp32.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "hdr_lpa.h"

namespace hdrlpa {

constexpr int MAXS = HDR_LPA_MAX_SENSORS;
constexpr int MAXJ = HDR_LPA_MAX_SCALES;

// fit status codes (_kernels.py:15-18) + the fast path's "needs exact decision"
constexpr int FIT_OK = 0;
constexpr int FIT_FAIL = 1;   // TOO_FEW / ILL_CONDITIONED (decided)
constexpr int FIT_AMBIG = 2;  // condition number too close to the threshold to decide from bounds
constexpr int FIT_PREC = 3;   // decisions sound, value needs the float64 recomputation (fit_precise)
// exact path, p = 3: the reference's closed-form eigenvalue range decides on
// rounding noise (near-singular window, or cond within reach of the
// threshold): settled by a reference-order re-evaluation (exact_ref.cuh)
constexpr int FIT_CRITICAL = 4;
// p = 3 windows whose condition number may exceed CLOSED_FORM_SAFE * threshold
// are not decided from bounds: the closed form's lambda_min carries an
// absolute error up to ~1e-8 lambda_max on near-degenerate windows, so only
// cond < 0.1 threshold is certainly accepted by it as well
constexpr double CLOSED_FORM_SAFE = 0.1;

struct DevSensor {
    const uint16_t *raw;
    int width, height, pitch, sat;
    int phmask[3];            // bit ph set <=> tile[ph] == channel
    int separable;            // T01 == 0 && T10 == 0 -> X(x), Y(y) separable
    double T[6];              // sensor -> reference
    double N[4];              // inverse of the linear part
    double nrow0, nrow1;      // |N row 0|, |N row 1| (window bbox half-widths per unit radius)
    // radiometry (radiometry.py:264-336)
    double bias, readvar, nonuni;
    const double *bias_p, *readvar_p, *nonuni_p;
    const uint8_t *defective;
    double g, t, n;
    double inv_denom, inv_denom2, c_shot, qv;  // scalar-calibration constants
    float bias_f, readvar_f, inv_denom_f, inv_denom2_f, c_shot_f, qv_f;
    int planes;               // any calibration plane present
    int vec_raw;              // raw base 16-B aligned and pitch % 8 == 0
    // fast-path staging geometry
    int rw, rh;               // staged region (even), phase planes are (rh/2) x (rw/2)
    int off_vi;               // byte offset (in a plane buffer) of the 4 staged phase planes
    double2 *lut;             // exact (f_hat, 1/den) per raw value (scalar calibration)
    float2 *phase;            // global phase planes [4][phg][pwg] of (f_hat, 1/den) (workspace)
    int pwg, phg;             // their padded width (float2 elements) and height
    int off_tx0, off_tx3;     // f64 column tables: X(x) (separable) or {fl(T00*x), fl(T10*x)}
    int off_ty1, off_ty4;     // f64 row tables: Y(y) at off_ty4 (separable) or
                              // {fl(T01*y), fl(T11*y)} at off_ty1 (off_tx3: unused, = off_tx0)
    float Tf[4];              // fp32 linear part (pre-test of rotated sensors)
};

// Pre-computed window tap (aligned / translation-only rigs on the reference
// grid): sensor offset (k, m) from the output pixel, exact float64 offset
// d = X - q and window weight W = exp(-|d|^2 / h).
struct Tap {
    double dx, dy;
    float W;
    int delta;  // offset of the sample in the sensor's phase planes relative to the pixel's base
};
// Device layout of the tap table (structure of arrays, one LDS.128 + one
// LDS.64 per tap): n x TapXY, then n x TapW.
struct __align__(16) TapXY {
    double dx, dy;
};
struct TapW {
    float W;
    int off;  // delta in bytes (float2 elements x 8)
};
// The tap table travels as a __grid_constant__ kernel parameter (kernel
// parameters may total 32764 B; DevParams takes ~5.6 KB): no device copy whose
// lifetime could outlive the caller's workspace.
constexpr int TAP_PARAM_BYTES = 26752;  // 1114 PAT taps
struct __align__(16) TapParam {
    unsigned char bytes[TAP_PARAM_BYTES];
};
struct NoTaps {};
// Row taps (RT mode): per (translation-only sensor, channel, parity class) the
// taps of the largest ICI window in (sensor row, column) order, each with its
// exact offset dx, |d|^2 (fp32, for the window weight), its byte offset in the
// staged phase planes and the smallest scale whose disk contains it.  Per
// scale k a list of rows {exact dy, the run of taps inside r_k}: |d|^2 is
// convex along a row, so each scale's members are one contiguous run.  A
// traversal of scale k reads only its own rows and taps -- no membership
// test, no empty rows -- and the fused ICI traversal tells the inner scale's
// members by kmin <= kin.
constexpr int RT_CLASSES = 16;  // (out x mod period) + period * (out y mod period), period <= 4
struct __align__(16) RowTap {
    double dx;
    float d2f;
    int off;  // bits 0-23: byte offset of the sample from the pixel's phase-plane position
              // (signed, 24 bits); bits 24-31: smallest scale index whose disk holds the tap
};
__host__ __device__ constexpr int rt_pack(int off, int kmin) { return (off & 0xffffff) | (kmin << 24); }
__device__ __forceinline__ int rt_off(int v) { return (v << 8) >> 8; }
__device__ __forceinline__ int rt_kmin(int v) { return (int)((unsigned)v >> 24); }
// Table layout: int2 {first row, row count} per (sensor, channel, class, scale)
// (index ((s * 3 + c) * rt_ncls + cls) * rt_nj + k), then the rows as two
// arrays (dy: double[n_rows], first | n << 20: uint32[n_rows]), then RowTap[].
constexpr int RT_ROW_N_SHIFT = 20;

struct DevParams {
    CUtensorMap tmap[MAXS];   // per-sensor 3-D maps over the phase planes (box = staged region)
    DevSensor s[MAXS];
    int n_sensors, order, n_scales, use_sigma;
    int out_w, out_h, row_begin, row_end;
    int tiles_x, tiles_y;
    int merged;               // co-sited tap mode: one merged plane set replaces the sensors' (PAT 3/4)
    int pad1b;
    double sx, sy;            // ref_w / out_w, ref_h / out_h  (lpa.py:222-223)
    double r[3][MAXJ];        // min(3 sqrt(h), max_radius)     (lpa.py:353, _kernels.py:276-277)
    double r2[3][MAXJ];       // r * r
    float hl[3][MAXJ];        // log2(e) / h  (window exponent in exp2 form, fast path)
    double hinv[3][MAXJ];     // 1 / h (float64 window exponent, exact path)
    double h[3][MAXJ];        // the window scales themselves
    double max_radius, cond, gamma;
    double fast_R;            // radius the staged tiles cover
    float *rgb;
    uint16_t *rgb_half;       // optional fp16 copy (scaled)
    float half_scale;
    float *grad;
    uint8_t *sidx;
    uint8_t *outcome;
    float *value;
    uint16_t *count;
    uint32_t *work;
    int flags;
    int diag;                 // any diagnostic plane (grad, sidx, outcome, value, count, work) requested
    // pre-computed-weight mode: taps per (sensor, channel, pixel parity class)
    int pat, n_taps, off_taps, tab_bytes;  // tab_bytes: kernel-parameter table size (PAT or RT)
    int rt;                         // row-tap mode (ICI / order 2 with translation-only sensors)
    int rt_period, rt_shift;        // RT: class period (2 / 4) and anchor shift (0 / 1) for sx 1 / 0.5
    int rt_ncls, rt_nj;             // RT: classes (period^2) and scales of the table
    int rt_dy_off, rt_fn_off, rt_taps_off;  // RT: byte offsets of the row arrays and RowTap[]
    const unsigned char *rt_global; // RT: the table in the workspace (copied to shared memory)
    int plane_base, buf_stride;     // shared memory: plane buffer b at plane_base + b*buf_stride
    int pat_off[MAXS][3][4];        // first tap of (sensor, channel, class = (y&1)*2 + (x&1))
    int pat_cnt[MAXS][3][4];        // taps of (sensor, channel, class)
    uint32_t *work_count;
    uint32_t *tile_counter;          // fast kernel: next tile to hand out (workspace header)
    uint32_t *slow_counter;          // exact path: next work item to evaluate
    uint32_t *fault;                 // HDR_FAULT_* bits raised by a kernel (workspace header)
    // float64 recomputations of a fit whose fast-path decisions stood (kk > 0):
    // enqueued from the END of work_items (slot item_cap - 1 - i) and evaluated
    // by lpa_precise_kernel before lpa_slow_kernel takes the full evaluations
    uint32_t *prec_count;            // workspace header word 4
    uint32_t *prec_counter;          // word 5: next recomputation to evaluate
    uint32_t item_cap;               // work_items capacity
    uint32_t all_items;              // > 0: no fast kernel; the exact path evaluates every
                                     // (pixel, channel) of the band (item i: pixel i / 3, channel i % 3)
    uint32_t *work_items;
    // CALPA steered pass: per output pixel steering field (theta, sigma, gamma)
    const double *st_theta, *st_sigma, *st_gamma;
    double prec_floor;              // fit_precise: radiance below which only absolute precision counts
};

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Output pixel centre in reference coordinates (lpa.py:222-223):
// (j + 0.5) * (ref / out) - 0.5, no contraction.
__device__ __forceinline__ double qcoord(int j, double s) {
    return __dadd_rn(__dmul_rn(__dadd_rn((double)j, 0.5), s), -0.5);
}

// Radiance sample of one sensor pixel (radiometry.py:271-336), rounded to fp32:
// .x = f_hat (electrons/s), .y = 1/den with den = sigma^2 (variance mode) or
// sigma (sigma mode, _kernels.py:166-167); .y == 0 marks "no sample"
// (saturated, defective or outside the frame).
// Radiometric conversion of one raw digital value at sensor pixel (x, y),
// which the caller has checked lies inside the frame.
__device__ __forceinline__ float2 radiance_from_raw(const DevSensor &S, int raw, int x, int y,
                                                    int use_sigma) {
    if (raw >= S.sat) return make_float2(0.f, 0.f);                       // :298-300
    const size_t i = (size_t)y * S.width + x;
    if (S.defective && __ldg(S.defective + i)) return make_float2(0.f, 0.f);  // :316-317
    float f, var;
    if (!S.planes) {
        // scalar calibration: fp32 with precomputed reciprocals (values are
        // rounded to fp32 anyway; relative error ~2 ulp of fp32)
        f = ((float)raw - S.bias_f) * S.inv_denom_f;                       // :279
        const float shot = S.c_shot_f * fmaxf(f, 0.f);                     // :294
        var = fmaxf((shot + S.readvar_f) * S.inv_denom2_f, S.qv_f);        // :295, :327-328
    } else {
        const double b = S.bias_p ? __ldg(S.bias_p + i) : S.bias;
        const double a = S.nonuni_p ? __ldg(S.nonuni_p + i) : S.nonuni;
        const double vr = S.readvar_p ? __ldg(S.readvar_p + i) : S.readvar;
        const double denom = S.g * S.t * S.n * a;                          // :265
        const double fd = ((double)raw - b) / denom;
        const double d2 = denom * denom;
        const double shot = S.g * S.g * S.t * a * S.n * fmax(fd, 0.0);
        f = (float)fd;
        var = (float)fmax((shot + vr) / d2, (1.0 / 12.0) / d2);
    }
    const float iv = use_sigma ? rsqrtf(var) : __frcp_rn(var);
    return make_float2(f, iv);
}

// Radiance sample of one sensor pixel (radiometry.py:271-336), rounded to fp32:
// .x = f_hat (electrons/s), .y = 1/den with den = sigma^2 (variance mode) or
// sigma (sigma mode, _kernels.py:166-167); .y == 0 marks "no sample"
// (saturated, defective or outside the frame).
__device__ __forceinline__ float2 radiance_sample(const DevSensor &S, int x, int y, int use_sigma) {
    if (x < 0 || y < 0 || x >= S.width || y >= S.height) return make_float2(0.f, 0.f);
    const int raw = (int)__ldg(S.raw + (size_t)y * S.pitch + x);
    return radiance_from_raw(S, raw, x, y, use_sigma);
}

// float64 radiometry in the reference's operation order (the oracle's
// pixel_sample; radiometry.py:264-336, radiometry.py:240 stores sigma^2,
// _kernels.py:165-167 divides by sigma^2 or sqrt(sigma^2)).  Returns false
// for "no sample"; iv = 1/den (one rounding more than the reference's W/den).
// Used by the exact (slow) path, whose results must not inherit the fp32
// rounding of the staged phase planes.
// f_hat and the reference's sigma = sqrt(max(var, quantisation floor))
__device__ __forceinline__ void radiometry_sigma(const DevSensor &S, int raw, double b, double a,
                                                 double vr, double &f, double &sg) {
    const double denom = __dmul_rn(__dmul_rn(__dmul_rn(S.g, S.t), S.n), a);
    f = __ddiv_rn(__dsub_rn((double)raw, b), denom);
    const double d2 = __dmul_rn(denom, denom);
    const double shot = __dmul_rn(
        __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(S.g, S.g), S.t), a), S.n), f > 0.0 ? f : 0.0);
    const double var = __ddiv_rn(__dadd_rn(shot, vr), d2);
    const double qv = __ddiv_rn(1.0 / 12.0, d2);
    sg = __dsqrt_rn(var >= qv ? var : qv);
}
__device__ __forceinline__ void radiometry_exact(const DevSensor &S, int raw, double b, double a,
                                                 double vr, int use_sigma, double &f, double &iv) {
    double sg;
    radiometry_sigma(S, raw, b, a, vr, f, sg);
    double den = __dmul_rn(sg, sg);  // SampleIndex stores sigma**2 (radiometry.py:240)
    if (use_sigma) den = __dsqrt_rn(den);
    iv = __drcp_rn(den);
}
// Scalar calibration: the per-frame LUT over raw values (radiance_lut_kernel).
__device__ __forceinline__ bool radiance_exact(const DevSensor &S, int x, int y, int use_sigma,
                                               double &f, double &iv) {
    if (x < 0 || y < 0 || x >= S.width || y >= S.height) return false;
    const int raw = (int)__ldg(S.raw + (size_t)y * S.pitch + x);
    if (raw >= S.sat) return false;
    const size_t i = (size_t)y * S.width + x;
    if (S.defective && __ldg(S.defective + i)) return false;
    if (!S.planes) {
        const double2 e = __ldg(S.lut + raw);
        f = e.x;
        iv = e.y;
        return true;
    }
    const double b = S.bias_p ? __ldg(S.bias_p + i) : S.bias;
    const double a = S.nonuni_p ? __ldg(S.nonuni_p + i) : S.nonuni;
    const double vr = S.readvar_p ? __ldg(S.readvar_p + i) : S.readvar;
    radiometry_exact(S, raw, b, a, vr, use_sigma, f, iv);
    return true;
}

// Sensor-space bounding box of the support disk |X - q| <= r.  In real
// arithmetic the ellipse T^{-1}(disk) lies in [c - h, c + h]; the rounding of
// c and h (~1e-13 px) can only add candidates, which the exact float64
// membership test then rejects.
__device__ __forceinline__ void window_bbox(const DevSensor &S, double qx, double qy, double r,
                                            int &xlo, int &xhi, int &ylo, int &yhi) {
    const double u = qx - S.T[2], v = qy - S.T[5];
    const double cx = S.N[0] * u + S.N[1] * v;
    const double cy = S.N[2] * u + S.N[3] * v;
    const double hx = r * S.nrow0, hy = r * S.nrow1;
    xlo = (int)floor(cx - hx);
    xhi = (int)ceil(cx + hx);
    ylo = (int)floor(cy - hy);
    yhi = (int)ceil(cy + hy);
}

// ---------------------------------------------------------------------------
// Moment accumulators (_kernels.py:155-182).  P = number of coefficients.
// ---------------------------------------------------------------------------
template <int P>
__device__ __forceinline__ constexpr int uidx(int a, int c) {  // packed upper index, a <= c
    return a * P - a * (a - 1) / 2 + (c - a);
}

// Basis exponents: phi_a = dx^I[a] dy^J[a] (lpa.py:104-118 order)
__device__ __forceinline__ constexpr int basis_i(int a) { return a == 1 ? 1 : a == 3 ? 2 : a == 4 ? 1 : 0; }
__device__ __forceinline__ constexpr int basis_j(int a) { return a == 2 ? 1 : a == 4 ? 1 : a == 5 ? 2 : 0; }
// Index of the monomial dx^i dy^j (degree-major, then by j)
__device__ __forceinline__ constexpr int midx(int i, int j) { return (i + j) * (i + j + 1) / 2 + j; }

// A (P(P+1)/2 packed upper entries) and b.  For P = 6 the normal matrix is
// stored as its 15 distinct moments M_ij = sum w dx^i dy^j (i + j <= 4; A is a
// Hankel-like arrangement of them): 15 accumulators instead of 21, and the
// row-factored sweeps add S_i dy^j into them directly.  fill_A expands.
template <int P>
struct Acc {
    static constexpr int NA = P * (P + 1) / 2;
    static constexpr bool MOM = (P == 6);
    static constexpr int NS = MOM ? 15 : NA;  // stored entries
    double A[NS];   // P <= 3: upper triangle, row-major packed; P = 6: moments M[midx(i, j)]
    double b[P];
    int count;
    float sabs;     // fast paths: sum w |y| (fp32), for the precision bound (fit_precise)
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < NS; ++i) A[i] = 0.0;
#pragma unroll
        for (int i = 0; i < P; ++i) b[i] = 0.0;
        count = 0;
        sabs = 0.f;
    }
    // A += w phi phi^T, b += w phi y with phi = [1, dx, dy, dx^2, dx dy, dy^2][:P]
    __device__ __forceinline__ void add(double wd, double yd, double dx, double dy, double dxx,
                                        double dyy, int inc = 1) {
        if constexpr (MOM) {
            double m[15];
            m[1] = dx;
            m[2] = dy;
            m[3] = dxx;
            m[4] = __dmul_rn(dx, dy);
            m[5] = dyy;
            m[6] = dxx * dx;
            m[7] = dxx * dy;
            m[8] = dx * dyy;
            m[9] = dyy * dy;
            m[10] = dxx * dxx;
            m[11] = dxx * m[4];
            m[12] = dxx * dyy;
            m[13] = m[4] * dyy;
            m[14] = dyy * dyy;
            A[0] += wd;
#pragma unroll
            for (int k = 1; k < 15; ++k) A[k] = fma(wd, m[k], A[k]);
            const double wy = wd * yd;
            b[0] += wy;
#pragma unroll
            for (int a = 1; a < 6; ++a) b[a] = fma(wy, m[midx(basis_i(a), basis_j(a))], b[a]);
        } else {
            double phi[3];
            phi[0] = 1.0;
            if (P >= 3) {
                phi[1] = dx;
                phi[2] = dy;
            }
            int k = 0;
#pragma unroll
            for (int a = 0; a < P; ++a) {
                const double wa = (a == 0) ? wd : wd * phi[a];
                b[a] = fma(wa, yd, b[a]);
#pragma unroll
                for (int c = a; c < P; ++c) {
                    A[k] = (c == 0) ? A[k] + wa : fma(wa, phi[c], A[k]);
                    ++k;
                }
            }
        }
        count += inc;
    }
    // Fast-path form of add() (fp32-derived weights, tolerance-checked): the
    // order-2 moments as w dx^i (depth-2 products) times powers of dy, fewer
    // float64 operations than the m[] products (29 instead of 32 per sample).
    __device__ __forceinline__ void add_fast(double wd, double yd, double dx, double dy,
                                             double dxx, double dyy, int inc) {
        if constexpr (MOM) {
            double u[5];
            u[0] = wd;
            u[1] = wd * dx;
            u[2] = wd * dxx;
            u[3] = u[1] * dxx;
            u[4] = u[2] * dxx;
            const double dy3 = dyy * dy, dy4 = dyy * dyy;
#pragma unroll
            for (int i = 0; i <= 4; ++i) A[midx(i, 0)] += u[i];
#pragma unroll
            for (int i = 0; i <= 3; ++i) A[midx(i, 1)] = fma(u[i], dy, A[midx(i, 1)]);
#pragma unroll
            for (int i = 0; i <= 2; ++i) A[midx(i, 2)] = fma(u[i], dyy, A[midx(i, 2)]);
#pragma unroll
            for (int i = 0; i <= 1; ++i) A[midx(i, 3)] = fma(u[i], dy3, A[midx(i, 3)]);
            A[midx(0, 4)] = fma(u[0], dy4, A[midx(0, 4)]);
            const double wy = wd * yd;
            b[0] += wy;
            b[1] = fma(wy, dx, b[1]);
            b[2] = fma(wy, dy, b[2]);
            b[3] = fma(wy, dxx, b[3]);
            b[4] = fma(wy, dx * dy, b[4]);
            b[5] = fma(wy, dyy, b[5]);
            count += inc;
        } else {
            add(wd, yd, dx, dy, dxx, dyy, inc);
        }
    }
    // Co-sited samples merged (PAT 3/4): the weight wd = W sum_s 1/den_s and
    // the weighted value wyd = W sum_s y_s/den_s of one position, so
    // b += wyd phi (the same sums as add() over the position's samples).
    __device__ __forceinline__ void add_wy(double wd, double wyd, double dx, double dy, double dxx,
                                           double dyy) {
        if constexpr (MOM) {
            double m[15];
            m[1] = dx;
            m[2] = dy;
            m[3] = dxx;
            m[4] = __dmul_rn(dx, dy);
            m[5] = dyy;
            m[6] = dxx * dx;
            m[7] = dxx * dy;
            m[8] = dx * dyy;
            m[9] = dyy * dy;
            m[10] = dxx * dxx;
            m[11] = dxx * m[4];
            m[12] = dxx * dyy;
            m[13] = m[4] * dyy;
            m[14] = dyy * dyy;
            A[0] += wd;
#pragma unroll
            for (int k = 1; k < 15; ++k) A[k] = fma(wd, m[k], A[k]);
            b[0] += wyd;
#pragma unroll
            for (int a = 1; a < 6; ++a) b[a] = fma(wyd, m[midx(basis_i(a), basis_j(a))], b[a]);
        } else {
            double phi[3];
            phi[0] = 1.0;
            if (P >= 3) {
                phi[1] = dx;
                phi[2] = dy;
            }
            b[0] += wyd;
#pragma unroll
            for (int a = 1; a < P; ++a) b[a] = fma(wyd, phi[a], b[a]);
            int k = 0;
#pragma unroll
            for (int a = 0; a < P; ++a) {
                const double wa = (a == 0) ? wd : wd * phi[a];
#pragma unroll
                for (int c = a; c < P; ++c) {
                    A[k] = (c == 0) ? A[k] + wa : fma(wa, phi[c], A[k]);
                    ++k;
                }
            }
        }
    }
    // packed upper triangle of A
    __device__ __forceinline__ void fill_A(double *out) const {
        if constexpr (MOM) {
#pragma unroll
            for (int a = 0; a < P; ++a)
#pragma unroll
                for (int c = a; c < P; ++c)
                    out[uidx<P>(a, c)] = A[midx(basis_i(a) + basis_i(c), basis_j(a) + basis_j(c))];
        } else {
#pragma unroll
            for (int i = 0; i < NA; ++i) out[i] = A[i];
        }
    }
};


// Result of a solved window: coefficients and g = A^{-1} e1 (for the ICI variance)
struct Fit {
    double c0, c1, c2;
    double g[6];
};

// In-register Cholesky of the packed SPD matrix (_kernels.py:76-101).
// Returns false on a non-positive pivot.  L is packed lower, row-major.
template <int P>
__device__ __forceinline__ bool cholesky(const double *A, double *L, double *inv) {
#pragma unroll
    for (int i = 0; i < P; ++i) {
#pragma unroll
        for (int j = 0; j <= i; ++j) {
            double s = A[uidx<P>(j, i)];
#pragma unroll
            for (int k = 0; k < j; ++k) s -= L[i * (i + 1) / 2 + k] * L[j * (j + 1) / 2 + k];
            if (i == j) {
                if (!(s > 0.0)) return false;
                const double ri = rsqrt(s);
                L[i * (i + 1) / 2 + i] = s * ri;
                inv[i] = ri;
            } else {
                L[i * (i + 1) / 2 + j] = s * inv[j];
            }
        }
    }
    return true;
}

// Solve from the Cholesky factor; also L^{-1} to get the condition bounds and
// g = A^{-1} e1.  cu/cl: upper/lower bounds on lambda_max/lambda_min:
//   lambda_max <= tr(A), lambda_min >= 1/tr(A^{-1})        -> cu = tr(A) tr(A^{-1})
//   lambda_max >= max_i A_ii, lambda_max(A^{-1}) >= max_i (A^{-1})_ii -> cl
template <int P>
__device__ __forceinline__ void chol_finish(const double *A, const double *b, const double *L,
                                            const double *inv, Fit &fit, double &cu, double &cl) {
    double z[P], c[P];
#pragma unroll
    for (int i = 0; i < P; ++i) {
        double s = b[i];
#pragma unroll
        for (int k = 0; k < i; ++k) s -= L[i * (i + 1) / 2 + k] * z[k];
        z[i] = s * inv[i];
    }
#pragma unroll
    for (int i = P - 1; i >= 0; --i) {
        double s = z[i];
#pragma unroll
        for (int k = i + 1; k < P; ++k) s -= L[k * (k + 1) / 2 + i] * c[k];
        c[i] = s * inv[i];
    }
    fit.c0 = c[0];
    fit.c1 = (P >= 3) ? c[1] : 0.0;
    fit.c2 = (P >= 3) ? c[2] : 0.0;
    // L^{-1} one column at a time (x = L^{-1} e_j, x_i = 0 for i < j):
    // (A^{-1})_jj = |x|^2, and column 0 gives g = A^{-1} e1 = L^{-T} x by
    // back substitution -- at most one column live, not the whole inverse
    double trA = 0.0, mA = 0.0, trI = 0.0, mI = 0.0;
    double x0[P];
#pragma unroll
    for (int j = 0; j < P; ++j) {
        const double ajj = A[uidx<P>(j, j)];
        trA += ajj;
        mA = fmax(mA, ajj);
        double x[P];
        x[j] = inv[j];
        double dj = x[j] * x[j];
#pragma unroll
        for (int i = j + 1; i < P; ++i) {
            double s = 0.0;
#pragma unroll
            for (int k = j; k < i; ++k) s += L[i * (i + 1) / 2 + k] * x[k];
            x[i] = -s * inv[i];
            dj += x[i] * x[i];
        }
        if (j == 0) {
#pragma unroll
            for (int i = 0; i < P; ++i) x0[i] = x[i];
        }
        trI += dj;
        mI = fmax(mI, dj);
    }
#pragma unroll
    for (int i = P - 1; i >= 0; --i) {
        double s = x0[i];
#pragma unroll
        for (int k = i + 1; k < P; ++k) s -= L[k * (k + 1) / 2 + i] * fit.g[k];
        fit.g[i] = s * inv[i];
    }
    cu = trA * trI;
    cl = mA * mI;
}

// Fast decision: OK / FAIL / AMBIG, with the reference's tests
// (_kernels.py:184-199): count < p, A00 <= 0 (p == 1), cond > threshold, pivot <= 0.
// grad = false: the gradient coefficients c1, c2 are not needed (no gradient
// plane requested) and are left unset by the 3x3 path.
template <int P>
__device__ __forceinline__ int solve_fast(const Acc<P> &acc, double cond, Fit &fit,
                                          bool grad = true) {
    if (acc.count < P) return FIT_FAIL;
    if constexpr (P == 1) {
        if (!(acc.A[0] > 0)) return FIT_FAIL;
        fit.c0 = acc.b[0] / acc.A[0];
        fit.c1 = fit.c2 = 0.0;
        fit.g[0] = 1.0 / acc.A[0];
        return FIT_OK;
    } else if constexpr (P == 3) {
        // 3x3: adjugate.  Positive definiteness by Sylvester (a > 0, ad - b^2 > 0,
        // det > 0: where the reference's Cholesky would hit a pivot <= 0),
        // A^-1 = adj(A)/det gives c, g = A^-1 e1 and the same two-sided
        // condition bounds as the Cholesky path (tr A tr A^-1 and
        // max A_ii max (A^-1)_ii); float64 rounding of the cofactors moves them
        // by <= cond * 1e-16 relative, far inside the 1e-5 margin.
        const double a = acc.A[0], b = acc.A[1], cc = acc.A[2];
        const double d = acc.A[3], e = acc.A[4], f = acc.A[5];
        const double C00 = fma(d, f, -e * e), C01 = fma(cc, e, -b * f), C02 = fma(b, e, -cc * d);
        const double C11 = fma(a, f, -cc * cc), C12 = fma(b, cc, -a * e), C22 = fma(a, d, -b * b);
        const double det = fma(a, C00, fma(b, C01, cc * C02));
        // not positive definite in float64 (count >= 3): a near-singular window,
        // on which the reference's closed form decides on rounding noise
        if (!(a > 0.0) || !(C22 > 0.0) || !(det > 0.0)) return FIT_AMBIG;
        // The cofactors are differences of products: near-singular windows
        // (e.g. coincident samples of identical sensors at a frame corner) leave
        // them at rounding-noise level, where their ratios are meaningless.  A
        // window with cond <= 1e8 keeps every principal minor >= 1e-8 of the
        // product of its diagonal (interlacing) and det >= ~1e-8 of its terms,
        // so anything below 1e-10 is decided by the exact path.
        constexpr double kRel = 1e-10;
        if (!(C00 > kRel * d * f) || !(C11 > kRel * a * f) || !(C22 > kRel * a * d) ||
            !(det > kRel * (fabs(a * C00) + fabs(b * C01) + fabs(cc * C02))))
            return FIT_AMBIG;
        const double rd = 1.0 / det;
        const double b0 = acc.b[0], b1 = acc.b[1], b2 = acc.b[2];
        fit.c0 = fma(C00, b0, fma(C01, b1, C02 * b2)) * rd;
        if (grad) {
            fit.c1 = fma(C01, b0, fma(C11, b1, C12 * b2)) * rd;
            fit.c2 = fma(C02, b0, fma(C12, b1, C22 * b2)) * rd;
        } else {
            fit.c1 = fit.c2 = 0.0;
        }
        fit.g[0] = C00 * rd;
        fit.g[1] = C01 * rd;
        fit.g[2] = C02 * rd;
        const double cu = (a + d + f) * ((C00 + C11 + C22) * rd);
        if (!(cu >= 9.0 * (1.0 - 1e-6))) return FIT_AMBIG;  // tr A tr A^-1 >= p^2 always
        // accepted only where the reference's closed form certainly accepts
        // too (cond < CLOSED_FORM_SAFE threshold; the fp32 weights move cond
        // by ~1e-6 relative); everything else is decided by the exact path
        if (cu <= cond * CLOSED_FORM_SAFE) return FIT_OK;
        return FIT_AMBIG;
    } else {
        double A[P * (P + 1) / 2], L[P * (P + 1) / 2], inv[P];
        acc.fill_A(A);
        if (!cholesky<P>(A, L, inv)) return FIT_FAIL;  // pivot <= 0: far beyond 1e8
        double cu, cl;
        chol_finish<P>(A, acc.b, L, inv, fit, cu, cl);
        const double margin = 1e-5;  // >> relative eigenvalue perturbation of fp32 weights
        if (cu <= cond * (1.0 - margin)) return FIT_OK;
        if (cl >= cond * (1.0 + margin)) return FIT_FAIL;
        return FIT_AMBIG;
    }
}

// Precision escalation of the fast path.  Its weights and values carry fp32
// rounding (relative <= FAST_EPS per sample); the resulting error of
// c0 = g . sum w phi y is bounded by FAST_EPS * max|g . phi| * sum w |y|
// with max|g . phi| <= |g0| + r (|g1| + |g2|) + r^2 (|g3| + |g4| + |g5|).
// A fit whose bound exceeds FAST_TOL relative to max(|c0|, floor) -- dark
// pixels next to much brighter samples, where order-2 kernels' negative
// lobes amplify the rounding -- is re-done by the exact path.
constexpr double FAST_EPS = 4e-7;
// co-sited merged planes (PAT 3/4): + the product y_s/den_s, the sums over
// <= PAT_MAXS sensors and W * sum (<= 5 more fp32 roundings)
constexpr double FAST_EPS_MERGED = 7e-7;
constexpr double FAST_TOL = 2e-5;
// relative error allowance of the fast path's ICI standard deviations (fp32
// weights through g = A^-1 e1; ~25x FAST_EPS)
constexpr double ICI_SD_EPS = 1e-5;
template <int P>
__device__ __forceinline__ bool fit_precise(const Fit &fit, float sabs, double r, double floor,
                                            double eps = FAST_EPS) {
    double G = fabs(fit.g[0]);
    if (P >= 3) G += r * (fabs(fit.g[1]) + fabs(fit.g[2]));
    if (P >= 6) G += r * r * (fabs(fit.g[3]) + fabs(fit.g[4]) + fabs(fit.g[5]));
    return G * (double)sabs <= (FAST_TOL / eps) * fmax(fabs(fit.c0), floor);
}
// Sharp form: with T = sum w |g.phi| |y|, first-order perturbation of the
// weights (by the residuals y - phi.c) and values gives |dc0| <~ 2 FAST_EPS T.
__device__ __forceinline__ bool fit_precise_sharp(double c0, float T, double floor) {
    return 2.0 * FAST_EPS * (double)T <= FAST_TOL * fmax(fabs(c0), floor);
}

// ---------------------------------------------------------------------------
// Exact eigenvalue range for the slow path (_kernels.py:26-73)
// ---------------------------------------------------------------------------
// _chol_solve (_kernels.py:76-101) in the reference's operation order
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

// p == 3: the reference's trigonometric closed form, same operation order
__device__ __forceinline__ void eig_range3(const double *A, double &lmin, double &lmax) {
    const double a11 = A[uidx<3>(0, 0)], a22 = A[uidx<3>(1, 1)], a33 = A[uidx<3>(2, 2)];
    const double a12 = A[uidx<3>(0, 1)], a13 = A[uidx<3>(0, 2)], a23 = A[uidx<3>(1, 2)];
    const double q = __ddiv_rn(__dadd_rn(__dadd_rn(a11, a22), a33), 3.0);
    const double p1 = __dadd_rn(__dadd_rn(__dmul_rn(a12, a12), __dmul_rn(a13, a13)), __dmul_rn(a23, a23));
    const double e1 = __dsub_rn(a11, q), e2 = __dsub_rn(a22, q), e3 = __dsub_rn(a33, q);
    const double p2 = __dadd_rn(
        __dadd_rn(__dadd_rn(__dmul_rn(e1, e1), __dmul_rn(e2, e2)), __dmul_rn(e3, e3)),
        __dmul_rn(2.0, p1));
    const double scale = fabs(a11) + fabs(a22) + fabs(a33) + 1e-300;
    if (p2 <= 1e-30 * scale * scale) {
        lmin = lmax = q;
        return;
    }
    const double pp = sqrt(__ddiv_rn(p2, 6.0));
    const double b11 = __ddiv_rn(e1, pp), b22 = __ddiv_rn(e2, pp), b33 = __ddiv_rn(e3, pp);
    const double b12 = __ddiv_rn(a12, pp), b13 = __ddiv_rn(a13, pp), b23 = __ddiv_rn(a23, pp);
    const double t1 = __dmul_rn(b11, __dsub_rn(__dmul_rn(b22, b33), __dmul_rn(b23, b23)));
    const double t2 = __dmul_rn(b12, __dsub_rn(__dmul_rn(b12, b33), __dmul_rn(b23, b13)));
    const double t3 = __dmul_rn(b13, __dsub_rn(__dmul_rn(b12, b23), __dmul_rn(b22, b13)));
    double r = __ddiv_rn(__dadd_rn(__dsub_rn(t1, t2), t3), 2.0);
    r = fmin(fmax(r, -1.0), 1.0);
    const double phi = __ddiv_rn(acos(r), 3.0);
    const double tp = __dmul_rn(2.0, pp);
    lmax = __dadd_rn(q, __dmul_rn(tp, cos(phi)));
    lmin = __dadd_rn(q, __dmul_rn(tp, cos(__dadd_rn(phi, 2.0943951023931953))));  // 2.0 * math.pi / 3.0
}

// eig_range3 plus a bound `err` on how far the reference's closed form could
// move lambda_min / lambda_max given last-bit differences of A (summation
// order) and of libm: the argument r of acos carries an error dr (HDR_CF_DR),
// and d acos / dr = 1 / sqrt(1 - r^2) blows up on near-degenerate windows
// (two eigenvalues close, r -> +-1), where the eigenvalues move by up to
// 2 p dr / (3 sqrt(1 - r^2)) -- ~1e-8 lambda_max at r = 1.
// lmin_cap: the largest lambda_min the closed form can return whatever the
// rounding of its acos argument (phi >= 0, so cos(phi + 2 pi / 3) <= -1/2:
// lambda_min <= q - p), which keeps rank-deficient windows certainly rejected.
// dr: a bound on |r_reference - r_here| -- the sums differ by the summation
// order (~count ulps worst case) and libm's last bits; r's sensitivity to
// them is ~10x on these windows (lambda_max dominates, B = (A - qI)/p)
#ifndef HDR_CF_DR
#define HDR_CF_DR 1e-13
#endif
__device__ __forceinline__ void eig_range3_err(const double *A, double &lmin, double &lmax,
                                               double &err, double &lmin_cap) {
    eig_range3(A, lmin, lmax);
    const double a11 = A[uidx<3>(0, 0)], a22 = A[uidx<3>(1, 1)], a33 = A[uidx<3>(2, 2)];
    const double a12 = A[uidx<3>(0, 1)], a13 = A[uidx<3>(0, 2)], a23 = A[uidx<3>(1, 2)];
    const double q = (a11 + a22 + a33) / 3.0;
    const double e1 = a11 - q, e2 = a22 - q, e3 = a33 - q;
    const double p2 = e1 * e1 + e2 * e2 + e3 * e3 + 2.0 * (a12 * a12 + a13 * a13 + a23 * a23);
    const double pp = sqrt(p2 / 6.0);
    constexpr double dr = HDR_CF_DR;
    double r = 0.0;
    if (pp > 0.0) {
        const double b11 = e1 / pp, b22 = e2 / pp, b33 = e3 / pp;
        const double b12 = a12 / pp, b13 = a13 / pp, b23 = a23 / pp;
        r = 0.5 * (b11 * (b22 * b33 - b23 * b23) - b12 * (b12 * b33 - b23 * b13) +
                   b13 * (b12 * b23 - b22 * b13));
    }
    const double s2 = fmax(1.0 - r * r, dr);
    const double round_q = 1e-14 * (fabs(a11) + fabs(a22) + fabs(a33));
    err = 2.0 * pp * dr / (3.0 * sqrt(s2)) + round_q;
    lmin_cap = q - pp + round_q;
}

// p == 6: cyclic Jacobi (the reference calls LAPACK dsyevd, _kernels.py:72)
static __device__ __noinline__ void eig_range6(const double *A, double &lmin, double &lmax) {
    double M[6][6];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int j = i; j < 6; ++j) M[i][j] = M[j][i] = A[uidx<6>(i, j)];
    for (int sweep = 0; sweep < 30; ++sweep) {
        double off = 0.0, diag = 0.0;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
            diag += M[i][i] * M[i][i];
#pragma unroll
            for (int j = i + 1; j < 6; ++j) off += M[i][j] * M[i][j];
        }
        if (off <= 1e-40 * diag) break;
#pragma unroll
        for (int p = 0; p < 6; ++p)
#pragma unroll
            for (int q = p + 1; q < 6; ++q) {
                const double apq = M[p][q];
                if (apq == 0.0) continue;
                const double theta = (M[q][q] - M[p][p]) / (2.0 * apq);
                const double t = copysign(1.0, theta) / (fabs(theta) + sqrt(theta * theta + 1.0));
                const double c = rsqrt(t * t + 1.0), s = t * c;
#pragma unroll
                for (int k = 0; k < 6; ++k) {
                    const double mkp = M[k][p], mkq = M[k][q];
                    M[k][p] = c * mkp - s * mkq;
                    M[k][q] = s * mkp + c * mkq;
                }
#pragma unroll
                for (int k = 0; k < 6; ++k) {
                    const double mpk = M[p][k], mqk = M[q][k];
                    M[p][k] = c * mpk - s * mqk;
                    M[q][k] = s * mpk + c * mqk;
                }
            }
    }
    lmin = lmax = M[0][0];
#pragma unroll
    for (int i = 1; i < 6; ++i) {
        lmin = fmin(lmin, M[i][i]);
        lmax = fmax(lmax, M[i][i]);
    }
}

// _fit_at's decision and solve (_kernels.py:184-199) on upper-triangle sums
// accumulated in the reference's order: count < p, A00 <= 0 (p == 1), the
// eigenvalue-range test (closed form for p == 3, Jacobi for p == 6), then
// _chol_solve.  Shared by the scattered-sample kernel and the exact path's
// reference-order re-evaluation (exact_ref.cuh).
template <int P>
__device__ __forceinline__ int ref_decide(double (&A)[6][6], const double *rhs, int count,
                                          double cond, double *coef) {
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

// Exact decision (slow path), mirroring _fit_at's tail (_kernels.py:184-200).
template <int P>
__device__ __forceinline__ int solve_exact(const Acc<P> &acc, double cond, Fit &fit) {
    if (acc.count < P) return FIT_FAIL;
    if constexpr (P == 1) {
        if (!(acc.A[0] > 0)) return FIT_FAIL;
        fit.c0 = acc.b[0] / acc.A[0];
        fit.c1 = fit.c2 = 0.0;
        fit.g[0] = 1.0 / acc.A[0];
        return FIT_OK;
    } else {
        // Both of the reference's rejections (eigenvalue test, Cholesky pivot)
        // give FIT_FAIL, so their order does not matter.  The float64
        // condition bounds decide whenever they are 1e-5 clear of the
        // threshold (their rounding error is <= cond * 1e-16, and so is the
        // reference's eigenvalues'); only the rest pays for the eigenvalues.
        double A[P * (P + 1) / 2], L[P * (P + 1) / 2], inv[P];
        acc.fill_A(A);
        if constexpr (P == 3) {
            // the reference's closed form (_kernels.py:38-71) decides; where its
            // rounding could land on either side of the threshold, the
            // reference-order re-evaluation does (FIT_CRITICAL, exact_ref.cuh).
            // cond <= CLOSED_FORM_SAFE threshold (the bound tr A tr A^-1) is
            // accepted by the closed form whatever its rounding.
            if (cholesky<P>(A, L, inv)) {
                double cu, cl;
                chol_finish<P>(A, acc.b, L, inv, fit, cu, cl);
                if (cu <= cond * CLOSED_FORM_SAFE) return FIT_OK;
            }
            double lmin, lmax, err, cap;
            eig_range3_err(A, lmin, lmax, err, cap);
            const double lo = lmin - err, hi = fmin(lmin + err, cap);
            if (hi <= 0.0 || lmax - err > cond * hi) return FIT_FAIL;
            if (!(lo > 0.0 && lmax + err <= cond * lo)) return FIT_CRITICAL;
            // cond <= threshold: the reference's _chol_solve succeeds
            if (!cholesky<P>(A, L, inv)) return FIT_CRITICAL;
            double cu, cl;
            chol_finish<P>(A, acc.b, L, inv, fit, cu, cl);
            return FIT_OK;
        }
        if (!cholesky<P>(A, L, inv)) return FIT_FAIL;
        double cu, cl;
        chol_finish<P>(A, acc.b, L, inv, fit, cu, cl);
        if (cu <= cond * (1.0 - 1e-5)) return FIT_OK;
        if (cl >= cond * (1.0 + 1e-5)) return FIT_FAIL;
        double lmin, lmax;
        if constexpr (P == 3)
            eig_range3(A, lmin, lmax);
        else
            eig_range6(A, lmin, lmax);
        if (lmin <= 0.0 || lmax > cond * lmin) return FIT_FAIL;
        return FIT_OK;
    }
}

}  // namespace hdrlpa
