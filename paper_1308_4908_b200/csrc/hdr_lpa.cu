// hdr_lpa.cu -- host side and C ABI (include/hdr_lpa.h) of the sm_100a
// unified HDR LPA operator.  The kernels live in the headers; the per-order
// fast/slow kernel launches (launch_all<ORDER>) are instantiated in
// fast_o0.cu / fast_o1.cu / fast_o2.cu (separate translation units, compiled
// in parallel), everything else here.
//
// Pipeline per frame (one stream, no host synchronisation):
//   1. memset of the exact-path work counter (+ row-tap table copy, RT mode)
//   2. radiance_lut_kernel / radiance_phase_kernel: float64 radiometry LUT and
//      the fp32 (f_hat, 1/den) Bayer phase planes of every sensor
//   3. lpa_fast_kernel: persistent CTAs over 32x8 output tiles, staged by TMA;
//      one thread per pixel fits R, G, B (taps / row taps / sweeps, ICI,
//      CALPA steering) and appends every fit it cannot decide exactly, or
//      whose fp32 rounding could exceed the tolerance, to a work list
//   4. lpa_slow_kernel / lpa_steered_slow_kernel: the reference's complete
//      semantics in float64 for the work list (_kernels.py:257-300)
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
#include "launch.cuh"
#include "frame_kernels.cuh"
#include "calpa.cuh"
#include "samples.cuh"
#include "sample_index.cuh"
#include "simulate.cuh"

namespace hdrlpa {

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

thread_local char g_last_error[256] = "";
// kernel launches issued by this library since load (hdr_lpa_launch_count)
std::atomic<unsigned long long> g_launches{0};

int cuda_fail(const char *where) {
    const cudaError_t e = cudaGetLastError();
    snprintf(g_last_error, sizeof(g_last_error), "%s: %s", where, cudaGetErrorString(e));
    return HDR_ERR_CUDA;
}

int set_smem_attr(const void *fn, int bytes) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    return e == cudaSuccess ? HDR_OK : cuda_fail("cudaFuncSetAttribute(smem)");
}

// hdr_lpa_kernel_timer: an event pair around each eager fast-kernel launch
thread_local bool g_timer_on = false;
thread_local cudaEvent_t g_timer_ev[2] = {nullptr, nullptr};
thread_local bool g_timer_recorded = false;
bool timer_active(cudaStream_t st) {
    if (!g_timer_on) return false;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    return cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone;
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
// 16-B row pitch, so TMA is always applicable.  Co-sited merged planes hold
// float4 elements: [4][phg][4*pwg] floats, box 2*rw floats.
static bool encode_phase_map(const DevSensor &d, CUtensorMap *map, bool merged = false) {
    auto enc = tensor_map_encoder();
    const int fpe = merged ? 4 : 2;  // floats per element
    if (!enc || d.rw * fpe / 2 > 256 || (d.rh >> 1) > 256) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)d.pwg * fpe, (cuuint64_t)d.phg, 4};
    const cuuint64_t strides[2] = {(cuuint64_t)d.pwg * 4 * fpe,
                                   (cuuint64_t)d.pwg * 4 * fpe * d.phg};
    const cuuint32_t box[3] = {(cuuint32_t)(d.rw * fpe / 2), (cuuint32_t)(d.rh >> 1), 4};
    const cuuint32_t estr[3] = {1, 1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void *)d.phase, dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
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
    const int period = 2 << shift, ncls = period * period, nj = P.n_scales;
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
    std::vector<int> hdr((size_t)P.n_sensors * 3 * ncls * nj * 2, 0);  // int2 {row0, nrow}
    std::vector<double> row_dy;
    std::vector<uint32_t> row_fn;
    std::vector<RowTap> taps;
    for (int s = 0; s < P.n_sensors; ++s) {
        const DevSensor &S = P.s[s];
        if (!S.separable) continue;
        int tile[4];
        for (int ph = 0; ph < 4; ++ph)
            for (int c = 0; c < 3; ++c)
                if ((S.phmask[c] >> ph) & 1) tile[ph] = c;
        const int pw = S.rw >> 1, plane = pw * (S.rh >> 1);
        if (4 * plane * (int)sizeof(float2) >= (1 << 23)) return false;  // 24-bit offsets
        for (int c = 0; c < 3; ++c) {
            double rmax2 = 0.0, rmax = 0.0;
            for (int k = 0; k < nj; ++k) {
                rmax2 = fmax(rmax2, P.r2[c][k]);
                rmax = fmax(rmax, P.r[c][k]);
            }
            const int R = (int)ceil(rmax + fabs(S.T[2]) + fabs(S.T[5])) + 2;
            for (int cl = 0; cl < ncls; ++cl) {
                // representative output pixel of the class and its anchor
                const int j = 128 + cl % period, i = 128 + cl / period;
                const double qx = ((double)j + 0.5) * P.sx + -0.5;  // qcoord (lpa.py:222-223)
                const double qy = ((double)i + 0.5) * P.sy + -0.5;
                const int ax = j >> shift, ay = i >> shift;
                std::vector<double> kdy[MAXJ];
                std::vector<uint32_t> kfn[MAXJ];
                for (int m = -R; m <= R; ++m) {
                    const int y = ay + m;
                    const int first = (int)taps.size();
                    std::vector<double> d2s;
                    double dy = 0.0;
                    for (int k2 = -R; k2 <= R; ++k2) {
                        const int x = ax + k2;
                        if (tile[((y & 1) << 1) | (x & 1)] != c) continue;
                        // the reference's arithmetic: apply_transform (radiometry.py:84),
                        // d = X - q and |d|^2 (_kernels.py:160-162)
                        const double X = (1.0 * (double)x + 0.0 * (double)y) + S.T[2];
                        const double Y = (0.0 * (double)x + 1.0 * (double)y) + S.T[5];
                        const double dx = X - qx;
                        dy = Y - qy;
                        const double d2 = dx * dx + dy * dy;
                        for (int k = 0; k < nj; ++k)
                            if (fabs(d2 - P.r2[c][k]) <= 1e-9 * P.r2[c][k]) return false;
                        if (d2 > rmax2) continue;
                        int kmin = nj;
                        for (int k = nj - 1; k >= 0; --k)
                            if (d2 <= P.r2[c][k]) kmin = k;
                        const int ph = ((y & 1) << 1) | (x & 1);
                        const int off = (int)sizeof(float2) *
                                        (ph * plane + ((y >> 1) - (ay >> 1)) * pw + ((x >> 1) - (ax >> 1)));
                        RowTap t;
                        t.dx = dx;
                        t.d2f = (float)d2;
                        t.off = rt_pack(off, kmin);
                        taps.push_back(t);
                        d2s.push_back(d2);
                    }
                    const int n = (int)d2s.size();
                    for (int k = 0; k < nj; ++k) {
                        int lo = n, hi = 0;
                        for (int u = 0; u < n; ++u)
                            if (d2s[u] <= P.r2[c][k]) {
                                lo = std::min(lo, u);
                                hi = u + 1;
                            }
                        if (lo >= hi) continue;
                        for (int u = lo; u < hi; ++u)  // convexity: the run has no holes
                            if (!(d2s[u] <= P.r2[c][k])) return false;
                        if (hi - lo >= (1 << (32 - RT_ROW_N_SHIFT))) return false;
                        kdy[k].push_back(dy);
                        kfn[k].push_back((uint32_t)(first + lo) | ((uint32_t)(hi - lo) << RT_ROW_N_SHIFT));
                    }
                }
                for (int k = 0; k < nj; ++k) {
                    const size_t h = 2 * ((((size_t)s * 3 + c) * ncls + cl) * nj + k);
                    hdr[h] = (int)row_dy.size();
                    hdr[h + 1] = (int)kdy[k].size();
                    row_dy.insert(row_dy.end(), kdy[k].begin(), kdy[k].end());
                    row_fn.insert(row_fn.end(), kfn[k].begin(), kfn[k].end());
                }
            }
        }
    }
    if (taps.size() >= (1u << RT_ROW_N_SHIFT)) return false;
    const size_t a16 = 15;
    const size_t hbytes = (hdr.size() * sizeof(int) + a16) & ~a16;
    const size_t dybytes = (row_dy.size() * sizeof(double) + a16) & ~a16;
    const size_t fnbytes = (row_fn.size() * sizeof(uint32_t) + a16) & ~a16;
    const size_t bytes = hbytes + dybytes + fnbytes + taps.size() * sizeof(RowTap);
    if (bytes > RT_TABLE_BYTES) return false;
    table.assign(bytes, 0);
    memcpy(table.data(), hdr.data(), hdr.size() * sizeof(int));
    memcpy(table.data() + hbytes, row_dy.data(), row_dy.size() * sizeof(double));
    memcpy(table.data() + hbytes + dybytes, row_fn.data(), row_fn.size() * sizeof(uint32_t));
    memcpy(table.data() + hbytes + dybytes + fnbytes, taps.data(), taps.size() * sizeof(RowTap));
    P.rt_period = period;
    P.rt_shift = shift;
    P.rt_ncls = ncls;
    P.rt_nj = nj;
    P.rt_dy_off = (int)hbytes;
    P.rt_fn_off = (int)(hbytes + dybytes);
    P.rt_taps_off = (int)(hbytes + dybytes + fnbytes);
    P.tab_bytes = (int)bytes;
    if (getenv("HDR_DEBUG_RT"))
        fprintf(stderr, "row-tap table: %zu taps, %zu rows, %zu bytes\n", taps.size(),
                row_dy.size(), bytes);
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
    if (P.n_scales != 1 || P.sx != 1.0 || P.sy != 1.0 || P.n_sensors > PAT_MAXS) return false;
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
            // a warp of the tap kernel holds pixels of one class only, so each
            // class keeps its own tap count (no padding to the longer list)
            for (int cl = 0; cl < 4; ++cl) {
                P.pat_cnt[s][c][cl] = (int)cls[cl].size();
                P.pat_off[s][c][cl] = (int)taps.size();
                taps.insert(taps.end(), cls[cl].begin(), cls[cl].end());
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

int hdr_lpa_kernel_timer(int enable) {
    if (enable && !g_timer_ev[0]) {
        if (cudaEventCreate(&g_timer_ev[0]) != cudaSuccess ||
            cudaEventCreate(&g_timer_ev[1]) != cudaSuccess)
            return cuda_fail("cudaEventCreate");
    }
    g_timer_on = enable != 0;
    g_timer_recorded = false;
    return HDR_OK;
}

int hdr_lpa_kernel_timer_read(float *ms) {
    if (!ms || !g_timer_recorded) return HDR_ERR_ARG;
    if (cudaEventSynchronize(g_timer_ev[1]) != cudaSuccess) return cuda_fail("cudaEventSynchronize");
    if (cudaEventElapsedTime(ms, g_timer_ev[0], g_timer_ev[1]) != cudaSuccess)
        return cuda_fail("cudaEventElapsedTime");
    return HDR_OK;
}

const char *hdr_lpa_last_error(void) { return g_last_error; }

const char *hdr_lpa_status_string(int status) {
    switch (status) {
        case HDR_OK: return "ok";
        case HDR_ERR_ARG: return "invalid argument";
        case HDR_ERR_CONFIG: return "invalid sensor configuration";
        case HDR_ERR_SHAPE: return "dimension mismatch";
        case HDR_ERR_WORKSPACE: return "workspace too small";
        case HDR_ERR_CUDA: return "CUDA error";
        case HDR_ERR_FAULT: return "kernel fault";
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
    if (!sensors || !params || !out || (!out->rgb && !out->rgb_half) || !workspace)
        return HDR_ERR_ARG;
    if (out->rgb_half && !(out->half_scale > 0.f)) return HDR_ERR_ARG;
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
    P.rgb_half = out->rgb_half;
    P.half_scale = out->half_scale;
    P.grad = out->grad;
    P.sidx = out->scale_idx;
    P.outcome = out->outcome;
    P.value = out->value;
    P.count = out->count;
    P.work = out->work;
    P.flags = params->flags;
    P.diag = (P.grad || P.sidx || P.outcome || P.value || P.count || P.work) ? 1 : 0;
    P.work_count = (uint32_t *)workspace;
    P.tile_counter = (uint32_t *)workspace + 1;
    P.slow_counter = (uint32_t *)workspace + 2;
    P.fault = (uint32_t *)workspace + 3;
    P.prec_count = (uint32_t *)workspace + 4;
    P.prec_counter = (uint32_t *)workspace + 5;
    P.item_cap = (uint32_t)((size_t)out_w * out_h * 3);
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

static int launch_prepass(const DevParams &P, cudaStream_t st, bool merged = false) {
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
    COUNT_LAUNCH();
    if (merged) {  // co-sited sensors: one merged plane set (sensor 0's geometry)
        dim3 grid((P.s[0].pwg / 4 + 31) / 32, (2 * P.s[0].phg + 3) / 4, 1);
        radiance_merge_kernel<<<grid, dim3(32, 4), 0, st>>>(P);
        return cudaPeekAtLastError() == cudaSuccess ? HDR_OK
                                                    : cuda_fail("radiance_merge_kernel launch");
    }
    dim3 grid((maxpw / 4 + 31) / 32, (maxph + 3) / 4, P.n_sensors);
    radiance_phase_kernel<<<grid, dim3(32, 4), 0, st>>>(P);
    return cudaPeekAtLastError() == cudaSuccess ? HDR_OK : cuda_fail("radiance_phase_kernel launch");
}

// Co-sited rig: at least two sensors, all with sensor 0's translation-only
// transform (bitwise), frame size and Bayer phase, fixed scale on the
// reference grid -- the conditions under which every sensor's sample of a
// sensor pixel has the same position, offset and weight, and the tap table
// applies.  Their samples can then be merged per position (PAT 3/4).  The
// merged float4 planes need sensor 0's and sensor 1's plane workspace.
static bool cosited(const DevParams &P) {
    if (P.n_sensors < 2 || P.n_sensors > PAT_MAXS || (P.flags & HDR_FLAG_NO_MERGE)) return false;
    if (P.n_scales != 1 || P.sx != 1.0 || P.sy != 1.0) return false;
    const DevSensor &a = P.s[0];
    for (int s = 1; s < P.n_sensors; ++s) {
        const DevSensor &b = P.s[s];
        if (b.width != a.width || b.height != a.height) return false;
        for (int c = 0; c < 3; ++c)
            if (b.phmask[c] != a.phmask[c]) return false;
        if (memcmp(a.T, b.T, sizeof(a.T)) != 0) return false;
    }
    return (char *)P.s[1].phase == (char *)a.phase + (size_t)4 * a.pwg * a.phg * sizeof(float2);
}

// Staged-region geometry, shared-memory layout, tap tables (when allowed) and
// TMA descriptors of the fast kernels, for windows up to radius fastR.
constexpr int STAGING_TOO_LARGE = -1;  // setup_staging: the tiles do not fit shared memory
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
        // + 2 for floor/ceil of the bbox ends, + 3 / + 1 for aligning the origin
        // down to a multiple of 4 columns / 2 rows
        int rw = (int)ceil(wx) + 2 + 3, rh = (int)ceil(wy) + 2 + 1;
        rw = (rw + 3) & ~3;  // TMA box inner extent (rw floats): multiple of 16 bytes
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
            w[i].off = taps[i].delta * (P.merged ? (int)sizeof(float4) : (int)sizeof(float2));
        }
        P.tab_bytes = (int)(n * sizeof(Tap));
    } else if (P.merged && allow_taps) {
        return HDR_ERR_ARG;  // merged planes: the tap kernel or the steered sweep only
    } else if (allow_taps) {
        P.rt = build_rowtaps(P, rt_table) ? 1 : 0;
        if (P.rt) P.off_taps = take(P.tab_bytes);
    }
    P.plane_base = smem;
    smem = 0;
    for (int s = 0; s < n_sensors; ++s) {
        DevSensor &d = P.s[s];
        d.off_vi = take(d.rw * d.rh * (P.merged ? 16 : 8));  // [4][rh/2][rw/2] float2 / float4
        // coordinate tables (staging.cuh): separable X(x), Y(y); otherwise the
        // interleaved partial products {T00 x, T10 x}, {T01 y, T11 y}
        d.off_tx0 = take(d.rw * (d.separable ? 8 : 16));
        d.off_tx3 = d.off_tx0;
        d.off_ty1 = d.separable ? 0 : take(d.rh * 16);
        d.off_ty4 = d.separable ? take(d.rh * 8) : 0;
    }
    P.buf_stride = smem;
    smem_bytes = P.plane_base + nbuf_for(P.pat, P.st_theta != nullptr) * P.buf_stride;
    if (smem_bytes > 200 * 1024) return STAGING_TOO_LARGE;  // windows too large to stage
    for (int s = 0; s < n_sensors; ++s)
        if (!encode_phase_map(P.s[s], &P.tmap[s], P.merged != 0)) {
            snprintf(g_last_error, sizeof(g_last_error), "cuTensorMapEncodeTiled failed (sensor %d)", s);
            return HDR_ERR_CUDA;
        }

    return HDR_OK;
}

int hdr_lpa_reconstruct(const HdrSensor *sensors, int n_sensors, const HdrParams *params,
                        int out_w, int out_h, double ref_w, double ref_h, int row_begin,
                        int row_end, const HdrOutputs *out, void *workspace,
                        size_t workspace_bytes, void *stream) {
    NvtxRange nv("hdr_lpa_reconstruct");
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
    // co-sited sensors: the fast kernel sees one sensor whose staged planes
    // are the merged ones (falls back to the per-sensor tap / sweep kernels
    // when the tap table does not apply)
    static thread_local DevParams Pf;
    bool merged = false;
    if (cosited(P)) {
        Pf = P;
        Pf.n_sensors = 1;
        Pf.merged = 1;
        merged = setup_staging(Pf, 1, fastR, true, T, rt_table, smem_bytes, maxc) == HDR_OK;
    }
    if (!merged) {
        const int rc = setup_staging(P, n_sensors, fastR, true, T, rt_table, smem_bytes, maxc);
        if (rc == STAGING_TOO_LARGE) {
            // the staged tiles of this rig (many sensors, large windows or ICI
            // scales) do not fit shared memory: every (pixel, channel) goes
            // through the exact path, which reads the raw frames directly
            P.rt = 0;
            P.all_items = (uint32_t)((row_end - row_begin) * out_w * 3);
        } else if (rc != HDR_OK) {
            return rc;
        }
    }
    cudaStream_t st = (cudaStream_t)stream;
    P.tiles_y = (row_end - row_begin + TH - 1) / TH;
    P.tiles_x = (out_w + TW - 1) / TW;
    const int tiles = P.tiles_x * P.tiles_y;
    if (merged) {
        Pf.tiles_x = P.tiles_x;
        Pf.tiles_y = P.tiles_y;
    }
    const DevParams &PF = merged ? Pf : P;
    if (cudaMemsetAsync(workspace, 0, WS_HEADER_WORDS * sizeof(uint32_t), st) != cudaSuccess)
        return cuda_fail("cudaMemsetAsync");
    if (P.rt && upload_table(rt_table, (unsigned char *)P.rt_global, st) != HDR_OK)
        return HDR_ERR_CUDA;
    if (launch_prepass(P, st, merged) != HDR_OK) return HDR_ERR_CUDA;  // per-frame radiometry
    int rc;
    switch (P.order) {
        case 0: rc = launch_all<0>(PF, P, T, tiles, smem_bytes, maxc, st); break;
        case 1: rc = launch_all<1>(PF, P, T, tiles, smem_bytes, maxc, st); break;
        default: rc = launch_all<2>(PF, P, T, tiles, smem_bytes, maxc, st); break;
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
    // co-sited sensors (orders 1-2): the steered sweep reads the merged planes
    static thread_local DevParams Pf;
    bool merged = false;
    if (P.order >= 1 && cosited(P)) {
        Pf = P;
        Pf.n_sensors = 1;
        Pf.merged = 1;
        merged = setup_staging(Pf, 1, P.max_radius, false, T, rt_table, smem_bytes, maxc) == HDR_OK;
    }
    const bool staged =
        merged ||
        setup_staging(P, n_sensors, P.max_radius, false, T, rt_table, smem_bytes, maxc) == HDR_OK;
    if (cudaMemsetAsync(workspace, 0, WS_HEADER_WORDS * sizeof(uint32_t), st) != cudaSuccess)
        return cuda_fail("cudaMemsetAsync");
    if (launch_prepass(P, st, merged) != HDR_OK) return HDR_ERR_CUDA;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (staged) {
        P.tiles_y = (P.row_end - P.row_begin + TH - 1) / TH;
        P.tiles_x = (out_w + TW - 1) / TW;
        const int tiles = P.tiles_x * P.tiles_y;
        Pf.tiles_x = P.tiles_x;
        Pf.tiles_y = P.tiles_y;
        int rc2;
#ifndef HDR_STEER_MAXC
#define HDR_STEER_MAXC 4  // columns per branch-free chunk of the steered sweep (2/3/4/6/8: 0.75/0.83/0.67/0.77/0.89 ms)
#endif
        constexpr int SM = HDR_STEER_MAXC;
        switch (P.order) {
            case 0: rc2 = launch_fast<0, false, SM, 0, false, true>(P, T, tiles, smem_bytes, st); break;
            case 1:
                rc2 = merged ? launch_fast<1, false, SM, 0, false, true, true>(Pf, T, tiles, smem_bytes, st)
                             : launch_fast<1, false, SM, 0, false, true>(P, T, tiles, smem_bytes, st);
                break;
            default:
                rc2 = merged ? launch_fast<2, false, SM, 0, false, true, true>(Pf, T, tiles, smem_bytes, st)
                             : launch_fast<2, false, SM, 0, false, true>(P, T, tiles, smem_bytes, st);
                break;
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

static int steering_field(const float *gx, const float *gy, int width, int height,
                          int gradient_window, double lambda1, double lambda2, double alpha,
                          double sigma_max, double gradient_scale, const double *scale_dev,
                          double *theta, double *sigma, double *gamma, void *stream) {
    if (!gx || !gy || !theta || !sigma || !gamma || width <= 0 || height <= 0) return HDR_ERR_ARG;
    if (gradient_window < 3 || gradient_window % 2 == 0) return HDR_ERR_ARG;
    if (!scale_dev && (!(gradient_scale > 0) || !isfinite(gradient_scale))) return HDR_ERR_ARG;
    if (alpha < 0 || lambda1 < 0 || !(lambda2 > 0)) return HDR_ERR_ARG;
    SteerConsts K;
    K.half = gradient_window / 2;
    K.wstd = gradient_window / 4.0;
    K.lam1 = lambda1;
    K.lam2 = lambda2;
    K.alpha = alpha;
    K.sigma_max = sigma_max;
    K.inv_scale = scale_dev ? 0.0 : 1.0 / gradient_scale;
    K.scale_dev = scale_dev;
    K.scale = scale_dev ? 0.0 : gradient_scale;
    const int tiled_smem = stf_smem_bytes(K.half);
    if (tiled_smem <= 160 * 1024) {  // the tiled kernel (windows up to ~70 px)
        if (set_smem_attr((const void *)steering_field_tiled_kernel, tiled_smem) != HDR_OK)
            return HDR_ERR_CUDA;
        dim3 grid((width + STF_TW - 1) / STF_TW, (height + STF_TH - 1) / STF_TH);
        COUNT_LAUNCH();
        steering_field_tiled_kernel<<<grid, dim3(STF_TW, STF_TH), tiled_smem,
                                      (cudaStream_t)stream>>>(gx, gy, width, height, K, theta,
                                                              sigma, gamma);
        return cudaPeekAtLastError() == cudaSuccess ? HDR_OK
                                                    : cuda_fail("steering_field_tiled_kernel launch");
    }
    dim3 grid((width + 127) / 128, height);
    COUNT_LAUNCH();
    steering_field_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(gx, gy, width, height, K, theta,
                                                                  sigma, gamma);
    return cudaPeekAtLastError() == cudaSuccess ? HDR_OK : cuda_fail("steering_field_kernel launch");
}

int hdr_steering_field(const float *gx, const float *gy, int width, int height,
                       int gradient_window, double lambda1, double lambda2, double alpha,
                       double sigma_max, double gradient_scale, double *theta, double *sigma,
                       double *gamma, void *stream) {
    return steering_field(gx, gy, width, height, gradient_window, lambda1, lambda2, alpha,
                          sigma_max, gradient_scale, nullptr, theta, sigma, gamma, stream);
}

int hdr_steering_field_devscale(const float *gx, const float *gy, int width, int height,
                                int gradient_window, double lambda1, double lambda2,
                                double alpha, double sigma_max, const double *gradient_scale,
                                double *theta, double *sigma, double *gamma, void *stream) {
    if (!gradient_scale) return HDR_ERR_ARG;
    return steering_field(gx, gy, width, height, gradient_window, lambda1, lambda2, alpha,
                          sigma_max, 0.0, gradient_scale, theta, sigma, gamma, stream);
}

int hdr_gradient_scale_workspace_bytes(size_t *bytes) {
    if (!bytes) return HDR_ERR_ARG;
    *bytes = 3 * (size_t)QBINS * sizeof(unsigned) + 128;
    return HDR_OK;
}

int hdr_gradient_scale(const float *values, long long n, double q, double *scale,
                       void *workspace, size_t workspace_bytes, void *stream) {
    size_t need = 0;
    hdr_gradient_scale_workspace_bytes(&need);
    if (!values || n < 0 || !scale || !workspace || !(q >= 0.0 && q <= 1.0)) return HDR_ERR_ARG;
    if (n >= (1ll << 32)) return HDR_ERR_ARG;  // 32-bit histogram counters
    if (workspace_bytes < need) return HDR_ERR_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    unsigned *hist = (unsigned *)workspace, *hist0 = hist + QBINS, *hist1 = hist0 + QBINS;
    QuantileState *qs = (QuantileState *)(hist1 + QBINS);
    if (cudaMemsetAsync(workspace, 0, need, st) != cudaSuccess) return cuda_fail("quantile memset");
    const unsigned blocks = (unsigned)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148 * 8));
    if (set_smem_attr((const void *)absq_hist_hi_smem_kernel, QHIST_SMEM) != HDR_OK)
        return HDR_ERR_CUDA;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const unsigned hblocks =
        (unsigned)std::max<long long>(1, std::min<long long>((n + 1023) / 1024, nsm));
    COUNT_LAUNCH();
    absq_hist_hi_smem_kernel<<<hblocks, 1024, QHIST_SMEM, st>>>(values, n, hist, &qs->n);
    COUNT_LAUNCH();
    absq_select_kernel<<<1, 1024, 0, st>>>(hist, q, qs);
    COUNT_LAUNCH();
    absq_hist_lo_kernel<<<blocks, 256, 0, st>>>(values, n, qs, hist0, hist1);
    COUNT_LAUNCH();
    absq_finish_kernel<<<1, 1024, 0, st>>>(hist0, hist1, qs, scale);
    return cudaPeekAtLastError() == cudaSuccess ? HDR_OK : cuda_fail("gradient scale kernels");
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

// exclusive scan of n int64 in place-capable buffers, scratch >= scan_scratch(n)
static size_t scan_scratch(long long n) {
    size_t total = 0;
    while (n > SCAN_BLOCK) {
        n = (n + SCAN_BLOCK - 1) / SCAN_BLOCK;
        total += 2 * (size_t)n;
    }
    return total;
}
static int device_scan(const long long *in, long long *out, long long n, long long *scratch,
                       cudaStream_t st) {
    const long long nb = (n + SCAN_BLOCK - 1) / SCAN_BLOCK;
    COUNT_LAUNCH();
    scan_block_kernel<<<(unsigned)nb, SCAN_BLOCK, 0, st>>>(in, out, n, nb > 1 ? scratch : nullptr);
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("scan_block_kernel");
    if (nb > 1) {
        long long *sums = scratch, *offs = scratch + nb;
        const int rc = device_scan(sums, offs, nb, scratch + 2 * nb, st);
        if (rc != HDR_OK) return rc;
        COUNT_LAUNCH();
        scan_add_kernel<<<(unsigned)nb, SCAN_BLOCK, 0, st>>>(out, n, offs);
        if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("scan_add_kernel");
    }
    return HDR_OK;
}

int hdr_sample_index_workspace_bytes(long long n, long long ncells, size_t *bytes) {
    if (!bytes || n < 0 || ncells < 1) return HDR_ERR_ARG;
    // bbox (8 x int64) | counts (ncells + 1) | fill (ncells) | perm (n) | scan scratch
    *bytes = 8 * sizeof(long long) + (size_t)(2 * ncells + 1 + n) * sizeof(long long) +
             scan_scratch(ncells + 1) * sizeof(long long);
    return HDR_OK;
}

int hdr_sample_index_bbox(const double *positions, const uint8_t *channels, long long n,
                          int channel, long long *count, int *x0, int *y0, int *nx, int *ny,
                          void *workspace, void *stream) {
    if (!positions || !channels || n < 0 || !count || !x0 || !y0 || !nx || !ny || !workspace)
        return HDR_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    long long *bbox = (long long *)workspace;
    COUNT_LAUNCH();
    sample_bbox_init_kernel<<<1, 1, 0, st>>>(bbox);
    if (n > 0) {
        COUNT_LAUNCH();
        const long long blocks = std::min<long long>((n + 255) / 256, 148 * 8);
        sample_bbox_kernel<<<(unsigned)blocks, 256, 0, st>>>((const double2 *)positions, channels,
                                                             n, channel, bbox);
    }
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("sample_bbox_kernel");
    long long h[5];
    if (cudaMemcpyAsync(h, bbox, sizeof(h), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return cuda_fail("sample bbox read-back");
    *count = h[0];
    if (h[0] == 0) {  // empty index: one cell (radiometry.py: empty bbox)
        *x0 = *y0 = 0;
        *nx = *ny = 1;
        return HDR_OK;
    }
    const long long w = h[3] - h[1] + 1, hh = h[4] - h[2] + 1;
    if (h[1] < INT_MIN / 2 || h[2] < INT_MIN / 2 || w > (1 << 20) || hh > (1 << 20) ||
        w * hh > (1ll << 31)) {
        snprintf(g_last_error, sizeof(g_last_error), "sample bbox too large (%lld x %lld cells)",
                 w, hh);
        return HDR_ERR_ARG;
    }
    *x0 = (int)h[1];
    *y0 = (int)h[2];
    *nx = (int)w;
    *ny = (int)hh;
    return HDR_OK;
}

int hdr_sample_index_build(const double *positions, const uint8_t *channels, const double *values,
                           const double *sigmas, long long n, int channel, int x0, int y0, int nx,
                           int ny, long long *cell_start, double *packed, void *workspace,
                           size_t workspace_bytes, void *stream) {
    if (!positions || !channels || !values || !sigmas || !cell_start || !workspace || nx < 1 ||
        ny < 1 || n < 0)
        return HDR_ERR_ARG;
    const long long ncells = (long long)nx * ny;
    size_t need = 0;
    hdr_sample_index_workspace_bytes(n, ncells, &need);
    if (workspace_bytes < need) return HDR_ERR_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    long long *counts = (long long *)workspace + 8;
    unsigned long long *fill = (unsigned long long *)(counts + ncells + 1);
    long long *perm = (long long *)(fill + ncells);
    long long *scratch = perm + n;
    if (cudaMemsetAsync(counts, 0, (size_t)(2 * ncells + 1) * sizeof(long long), st) != cudaSuccess)
        return cuda_fail("sample index memset");
    const unsigned blocks = (unsigned)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148 * 8));
    const double2 *pos = (const double2 *)positions;
    COUNT_LAUNCH();
    cell_count_kernel<<<blocks, 256, 0, st>>>(pos, channels, n, channel, x0, y0, nx, counts);
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("cell_count_kernel");
    const int rc = device_scan(counts, cell_start, ncells + 1, scratch, st);
    if (rc != HDR_OK) return rc;
    COUNT_LAUNCH();
    cell_scatter_kernel<<<blocks, 256, 0, st>>>(pos, channels, n, channel, x0, y0, nx, cell_start,
                                                fill, perm);
    const unsigned cblocks = (unsigned)std::min<long long>((ncells + 255) / 256, 148 * 16);
    COUNT_LAUNCH();
    cell_order_kernel<<<cblocks, 256, 0, st>>>(pos, values, sigmas, ncells, cell_start, perm,
                                               (double4 *)packed);
    return cudaPeekAtLastError() == cudaSuccess ? HDR_OK : cuda_fail("cell_order_kernel");
}

int hdr_sample_count(const HdrSensor *sensor, const double *sigma, long long *count,
                     void *workspace, void *stream) {
    if (!sensor || !sigma || !count || !workspace) return HDR_ERR_ARG;
    DevSensor d;
    const int rc = fill_sensor(*sensor, d);
    if (rc != HDR_OK) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    // workspace: rows[h + 1] | start[h + 1] | scan scratch
    long long *rows = (long long *)workspace, *start = rows + d.height + 1;
    COUNT_LAUNCH();
    row_count_kernel<<<d.height, 256, 0, st>>>(sigma, d.width, d.height, rows);
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("row_count_kernel");
    long long *scratch = start + d.height + 1;
    // start[y] = kept pixels before row y; start[h] = total
    if (cudaMemsetAsync(rows + d.height, 0, sizeof(long long), st) != cudaSuccess)
        return cuda_fail("sample count memset");
    const int rc2 = device_scan(rows, start, d.height + 1, scratch, st);
    if (rc2 != HDR_OK) return rc2;
    if (cudaMemcpyAsync(count, start + d.height, sizeof(long long), cudaMemcpyDeviceToHost, st) !=
            cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return cuda_fail("sample count read-back");
    return HDR_OK;
}

int hdr_compact_samples(const HdrSensor *sensor, int sensor_id, const double *value,
                        const double *sigma, long long offset, double *positions,
                        uint8_t *channels, double *values, double *sigmas, int *sensor_ids,
                        const void *workspace, void *stream) {
    if (!sensor || !value || !sigma || !positions || !channels || !values || !sigmas ||
        !sensor_ids || !workspace || offset < 0)
        return HDR_ERR_ARG;
    DevSensor d;
    const int rc = fill_sensor(*sensor, d);
    if (rc != HDR_OK) return rc;
    const long long *start = (const long long *)workspace + d.height + 1;
    COUNT_LAUNCH();
    row_compact_kernel<<<d.height, 256, 0, (cudaStream_t)stream>>>(
        d, sensor_id, value, sigma, d.width, d.height, start, offset, (double2 *)positions,
        channels, values, sigmas, sensor_ids);
    return cudaPeekAtLastError() == cudaSuccess ? HDR_OK : cuda_fail("row_compact_kernel");
}

int hdr_sample_count_workspace_bytes(int height, size_t *bytes) {
    if (!bytes || height < 1) return HDR_ERR_ARG;
    *bytes = (size_t)(2 * ((long long)height + 1) + scan_scratch(height + 1)) * sizeof(long long);
    return HDR_OK;
}

int hdr_simulate_sensor(const float *gt, int gt_w, int gt_h, const HdrSensor *sensor,
                        unsigned long long seed, int sensor_id, int noise_free, void *stream) {
    if (!gt || gt_w < 1 || gt_h < 1 || !sensor || !sensor->raw) return HDR_ERR_ARG;
    DevSensor d;
    const int rc = fill_sensor(*sensor, d);
    if (rc != HDR_OK) return rc;
    if (d.planes || d.defective) return HDR_ERR_ARG;  // scalar noise truth only
    dim3 grid((d.width + 127) / 128, d.height);
    COUNT_LAUNCH();
    simulate_sensor_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(
        gt, gt_w, gt_h, d, seed, sensor_id, noise_free, (uint16_t *)d.raw, d.pitch);
    return cudaPeekAtLastError() == cudaSuccess ? HDR_OK : cuda_fail("simulate_sensor_kernel");
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

int hdr_lpa_workspace_status(const void *workspace, uint32_t *slow_items, uint32_t *fault,
                             void *stream) {
    if (!workspace) return HDR_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t hdr[WS_HEADER_WORDS];
    if (cudaMemcpyAsync(hdr, workspace, sizeof(hdr), cudaMemcpyDeviceToHost, st) != cudaSuccess)
        return cuda_fail("workspace status copy");
    if (cudaStreamSynchronize(st) != cudaSuccess) return cuda_fail("workspace status sync");
    if (slow_items) *slow_items = hdr[0] + hdr[4];  // full evaluations + recomputations
    if (fault) *fault = hdr[3];
    if (hdr[3]) {
        snprintf(g_last_error, sizeof(g_last_error),
                 "kernel fault 0x%x (staging barrier timed out: the tile results are incomplete)",
                 hdr[3]);
        return HDR_ERR_FAULT;
    }
    return HDR_OK;
}

int hdr_lpa_slow_items(const void *workspace, uint32_t *count, void *stream) {
    if (!workspace || !count) return HDR_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    uint32_t hdr[WS_HEADER_WORDS];
    if (cudaMemcpyAsync(hdr, workspace, sizeof(hdr), cudaMemcpyDeviceToHost, st) != cudaSuccess)
        return HDR_ERR_CUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return HDR_ERR_CUDA;
    *count = hdr[0] + hdr[4];  // full evaluations + recomputations
    return HDR_OK;
}

}  // extern "C"
