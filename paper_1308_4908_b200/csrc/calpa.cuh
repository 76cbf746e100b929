// calpa.cuh -- CALPA: steering field kernel and the exact steered pass.
#pragma once

#include "exact.cuh"

namespace hdrlpa {

// ---------------------------------------------------------------------------
// CALPA: steering field and steered (anisotropic, two-phase) pass
// (reference steering.py:72-248, _kernels.py:262-275, :303-392)
// ---------------------------------------------------------------------------
struct SteerConsts {
    int half;
    double wstd, lam1, lam2, alpha, sigma_max, inv_scale;
    const double *scale_dev;  // non-null: inv_scale = 1 / *scale_dev (device-computed scale)
    double scale;             // tiled kernel: g / scale as the reference divides (0: scale_dev)
};

// The per-pixel epilogue of _kernels.steering_field_kernel (_kernels.py:303-392):
// eigen-range of the 2x2 structure tensor, orientation, elongation, scaling.
__device__ __forceinline__ void steering_epilogue(const SteerConsts &K, double s11, double s12,
                                                  double s22, int n, size_t o, double *theta,
                                                  double *sigma, double *gamma) {
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

// Tiled form (round 2): a 32x8 block of pixels stages its (32+2h) x (8+2h)
// neighbourhood once as float64 (g_x / scale, g_y / scale) with a validity
// byte (inside the image and both finite; invalid entries hold (0, 0), whose
// terms add +0 and leave the sums bit-identical to skipping them), and the
// (2h+1)^2 window weights exp(-(dx^2+dy^2) / (2 wstd^2)) once per block; the
// structure tensor then sums in the reference's order (rows, then columns;
// (w g1) g1 without contraction, as _kernels.py evaluates it).
constexpr int STF_TW = 32, STF_TH = 8;
#ifndef HDR_STF_FMA
#define HDR_STF_FMA 1  // measured: CALPA 827 -> 847 frames/s
#endif
__host__ __device__ inline int stf_smem_bytes(int half) {
    const int tw = STF_TW + 2 * half, th = STF_TH + 2 * half, nw = (2 * half + 1) * (2 * half + 1);
    return tw * th * 16 + ((tw * th + 15) & ~15) + nw * 8;
}
__global__ void __launch_bounds__(STF_TW *STF_TH)
    steering_field_tiled_kernel(const float *gx, const float *gy, int w, int h, SteerConsts K,
                                double *theta, double *sigma, double *gamma) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int half = K.half, tw = STF_TW + 2 * half, th = STF_TH + 2 * half;
    const int nwin = 2 * half + 1;
    double2 *g = (double2 *)sm;
    unsigned char *valid = sm + tw * th * 16;
    double *wt = (double *)(sm + tw * th * 16 + ((tw * th + 15) & ~15));
    const double scale = K.scale_dev ? *K.scale_dev : K.scale;
    const int x0 = blockIdx.x * STF_TW - half, y0 = blockIdx.y * STF_TH - half;
    const int tid = threadIdx.y * STF_TW + threadIdx.x;
    for (int i = tid; i < tw * th; i += STF_TW * STF_TH) {
        const int ix = x0 + i % tw, iy = y0 + i / tw;
        double g1 = 0.0, g2 = 0.0;
        bool ok = false;
        if (ix >= 0 && ix < w && iy >= 0 && iy < h) {
            g1 = __ddiv_rn((double)gx[(size_t)iy * w + ix], scale);  // gx / scale (steering.py)
            g2 = __ddiv_rn((double)gy[(size_t)iy * w + ix], scale);
            ok = isfinite(g1) && isfinite(g2);
        }
        g[i] = ok ? make_double2(g1, g2) : make_double2(0.0, 0.0);
        valid[i] = ok ? 1 : 0;
    }
    const double den = 2.0 * K.wstd * K.wstd;
    for (int i = tid; i < nwin * nwin; i += STF_TW * STF_TH) {
        const int dx = i % nwin - half, dy = i / nwin - half;
        wt[i] = exp(-(double)(dx * dx + dy * dy) / den);
    }
    __syncthreads();
    const int xx = blockIdx.x * STF_TW + threadIdx.x, yy = blockIdx.y * STF_TH + threadIdx.y;
    if (xx >= w || yy >= h) return;
    double s11 = 0.0, s12 = 0.0, s22 = 0.0;
    int n = 0;
    for (int dy = 0; dy < nwin; ++dy) {
        const double2 *gr = g + (threadIdx.y + dy) * tw + threadIdx.x;
        const unsigned char *vr = valid + (threadIdx.y + dy) * tw + threadIdx.x;
        const double *wr = wt + dy * nwin;
        for (int dx = 0; dx < nwin; ++dx) {
            const double2 v = gr[dx];
            const double wgt = wr[dx];
            const double a = __dmul_rn(wgt, v.x);
#if HDR_STF_FMA
            // fused: 5 FP64 operations per tap instead of 8 (each sum differs
            // from the reference's unfused one by <= 1 ulp per term)
            s11 = fma(a, v.x, s11);
            s12 = fma(a, v.y, s12);
            s22 = fma(__dmul_rn(wgt, v.y), v.y, s22);
#else
            s11 = __dadd_rn(s11, __dmul_rn(a, v.x));
            s12 = __dadd_rn(s12, __dmul_rn(a, v.y));
            s22 = __dadd_rn(s22, __dmul_rn(__dmul_rn(wgt, v.y), v.y));
#endif
            n += vr[dx];
        }
    }
    steering_epilogue(K, s11, s12, s22, n, (size_t)yy * w + xx, theta, sigma, gamma);
}

// steering_field_kernel (_kernels.py:310-392), float64, one thread per pixel.
__global__ void steering_field_kernel(const float *gx, const float *gy, int w, int h,
                                      SteerConsts K, double *theta, double *sigma,
                                      double *gamma) {
    const int xx = blockIdx.x * blockDim.x + threadIdx.x, yy = blockIdx.y;
    if (xx >= w) return;
    if (K.scale_dev) K.inv_scale = 1.0 / *K.scale_dev;
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
    steering_epilogue(K, s11, s12, s22, n, (size_t)yy * w + xx, theta, sigma, gamma);
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
            int st = solve_exact<PN>(acc, P.cond, fit);
            if (st == FIT_CRITICAL)  // the reference's order (exact_ref.cuh)
                st = settle_critical<ORDER>(P, c, sweep.qx, sweep.qy, h11, h12, h22, r, fit);
            if (st == FIT_OK) {
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
    // items are fetched dynamically (their cost varies by orders of magnitude)
    const unsigned gmask = G >= 32 ? 0xffffffffu
                                   : ((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1));
    const int leader = (threadIdx.x & 31) & ~(G - 1);
    for (;;) {
        uint32_t i = 0;
        if ((threadIdx.x & (G - 1)) == 0) i = atomicAdd(P.slow_counter, 1u);
        i = __shfl_sync(gmask, i, leader);
        if (i >= n) break;
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

}  // namespace hdrlpa

namespace hdrlpa {

// ---------------------------------------------------------------------------
// The steering field's gradient scale on the device (steering.py:206-211):
// np.percentile(|finite values|, 99.5) with numpy's linear interpolation
// (virtual index q (n-1), _lerp with its t >= 0.5 branch), 1.0 when there is
// no finite value or the percentile is 0.  An exact two-pass radix select on
// the float32 bit patterns of |v| (monotone for non-negative floats): the
// high 16 bits pick the bins of ranks k and k+1, the low 16 bits the values.
// Lets a CALPA frame run without a host round trip (CUDA-graph capturable).
// Workspace: 4 x 65536 uint32 + 64 B.
// ---------------------------------------------------------------------------
constexpr int QBINS = 65536;
struct QuantileState {
    unsigned long long n;       // finite values
    long long rank[2];          // k, k + 1 (clipped)
    int bin[2];                 // their high-16 bins
    long long before[2];        // values in lower bins
    double t;                   // interpolation weight
};

// High-16-bit histogram, privatised per block in shared memory: |x| has a
// zero sign bit, so its high 16 bits take 2^15 values (128 KB of counters);
// one block per SM counts its slice with shared-memory atomics and adds its
// non-zero bins to the global histogram (round 1's global atomics serialised
// on the few hot bins of a natural image: 0.37 ms per 4-Mpx plane; now 12 us).
constexpr int QBINS_HI = 32768;
constexpr int QHIST_SMEM = QBINS_HI * 4;
__global__ void __launch_bounds__(1024) absq_hist_hi_smem_kernel(const float *v, long long n,
                                                                  unsigned *hist,
                                                                  unsigned long long *count) {
    extern __shared__ unsigned sh[];
    for (int i = threadIdx.x; i < QBINS_HI; i += blockDim.x) sh[i] = 0u;
    __syncthreads();
    unsigned long long c = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const float x = v[i];
        if (!isfinite(x)) continue;
        atomicAdd(&sh[__float_as_uint(fabsf(x)) >> 16], 1u);
        ++c;
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) c += __shfl_xor_sync(0xffffffffu, c, m);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
    __syncthreads();
    for (int i = threadIdx.x; i < QBINS_HI; i += blockDim.x) {
        const unsigned b = sh[i];
        if (b) atomicAdd(&hist[i], b);
    }
}

// Block-cooperative rank search over a QBINS-bin histogram (1024 threads):
// block_chunk_scan sums chunks of 64 bins by coalesced warp loads and scans
// the 1024 chunk sums; block_locate finds the chunk holding rank `want` and
// scans its 64 bins in one warp, returning (through shared memory) the bin and
// the count of values in lower bins.
// (round 1 summed 64 bins per thread with strided loads and walked the chunk
// with dependent loads: 40-80 us per search)
constexpr int QPER = QBINS / 1024;  // 64 bins per chunk
__device__ __forceinline__ void block_chunk_scan(const unsigned *h, unsigned long long *part) {
    constexpr int PER = QPER;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // 32 chunks per warp, all loads in flight before the reductions (a
    // load-reduce loop left one L2 round trip per chunk on the critical path)
    unsigned a[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        const int c = wid + 32 * i;
        a[i] = h[c * PER + lane] + h[c * PER + 32 + lane];  // two disjoint bins: <= n < 2^32
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        unsigned long long v = a[i];
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
        if (lane == 0) part[wid + 32 * i] = v;
    }
    __syncthreads();
    {  // inclusive scan of part[1024]: warp scans, then the warp totals
        __shared__ unsigned long long wsum[32];
        unsigned long long x = part[threadIdx.x];
#pragma unroll
        for (int m = 1; m < 32; m <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, m);
            if (lane >= m) x += y;
        }
        if (lane == 31) wsum[wid] = x;
        __syncthreads();
        if (wid == 0) {
            unsigned long long t = wsum[lane];
#pragma unroll
            for (int m = 1; m < 32; m <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, t, m);
                if (lane >= m) t += y;
            }
            wsum[lane] = t;
        }
        __syncthreads();
        part[threadIdx.x] = x + (wid ? wsum[wid - 1] : 0ull);
        __syncthreads();
    }
}
// the bin of rank `want` given block_chunk_scan's part[]
__device__ __forceinline__ void block_locate(const unsigned *h, unsigned long long want,
                                             const unsigned long long *part, int *s_bin,
                                             unsigned long long *s_before) {
    constexpr int PER = QPER;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __shared__ int s_chunk;
    {
        const unsigned long long lo = threadIdx.x ? part[threadIdx.x - 1] : 0, hi = part[threadIdx.x];
        if (want >= lo && want < hi) s_chunk = threadIdx.x;
    }
    __syncthreads();
    if (wid == 0) {  // the chunk's 64 bins: inclusive scan of lane pairs
        const int c = s_chunk;
        const unsigned long long base = c ? part[c - 1] : 0;
        const unsigned a = h[c * PER + 2 * lane], b = h[c * PER + 2 * lane + 1];
        unsigned long long x = (unsigned long long)a + b;
#pragma unroll
        for (int m = 1; m < 32; m <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, m);
            if (lane >= m) x += y;
        }
        const unsigned long long lo = base + x - a - b;  // before this lane's two bins
        if (want >= lo && want < lo + a) {
            *s_bin = c * PER + 2 * lane;
            *s_before = lo;
        } else if (want >= lo + a && want < lo + a + b) {
            *s_bin = c * PER + 2 * lane + 1;
            *s_before = lo + a;
        }
    }
    __syncthreads();
}

// one block of 1024 threads: bins of ranks k and k+1
__global__ void __launch_bounds__(1024) absq_select_kernel(const unsigned *hist, double q,
                                                            QuantileState *st) {
    __shared__ unsigned long long part[1024];
    __shared__ int s_bin;
    __shared__ unsigned long long s_before;
    const unsigned long long n = st->n;
    if (n == 0) return;
    const double vidx = q * (double)(n - 1);  // numpy: quantiles * (n - alpha - beta + 1) + alpha - 1
    const long long k = (long long)floor(vidx);
    const long long k1 = k + 1 < (long long)n ? k + 1 : (long long)n - 1;
    block_chunk_scan(hist, part);
    for (int r = 0; r < 2; ++r) {
        block_locate(hist, (unsigned long long)(r ? k1 : k), part, &s_bin, &s_before);
        if (threadIdx.x == 0) {
            st->bin[r] = s_bin;
            st->before[r] = (long long)s_before;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        st->rank[0] = k;
        st->rank[1] = k1;
        st->t = vidx - (double)k;
    }
}

__global__ void absq_hist_lo_kernel(const float *v, long long n, const QuantileState *st,
                                    unsigned *hist0, unsigned *hist1) {
    if (st->n == 0) return;
    const int b0 = st->bin[0], b1 = st->bin[1];
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const float x = v[i];
        if (!isfinite(x)) continue;
        const unsigned u = __float_as_uint(fabsf(x));
        if ((int)(u >> 16) == b0) atomicAdd(&hist0[u & 0xffffu], 1u);
        if (b1 != b0 && (int)(u >> 16) == b1) atomicAdd(&hist1[u & 0xffffu], 1u);
    }
}

__global__ void __launch_bounds__(1024) absq_finish_kernel(const unsigned *hist0,
                                                            const unsigned *hist1,
                                                            const QuantileState *st,
                                                            double *scale) {
    __shared__ unsigned long long part[1024];
    __shared__ int s_bin;
    __shared__ unsigned long long s_before;
    __shared__ float val[2];
    if (st->n == 0) {
        if (threadIdx.x == 0) *scale = 1.0;
        return;
    }
    for (int r = 0; r < 2; ++r) {
        const bool other = r == 1 && st->bin[1] != st->bin[0];
        const unsigned *h = other ? hist1 : hist0;
        if (r == 0 || other) block_chunk_scan(h, part);
        block_locate(h, (unsigned long long)(st->rank[r] - st->before[r]), part, &s_bin,
                     &s_before);
        if (threadIdx.x == 0) val[r] = __uint_as_float(((unsigned)st->bin[r] << 16) | (unsigned)s_bin);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double a = (double)val[0], b = (double)val[1], t = st->t;
        const double d = b - a;
        const double p = t >= 0.5 ? b - d * (1.0 - t) : a + d * t;  // numpy _lerp
        *scale = p > 0.0 ? p : 1.0;
    }
}

}  // namespace hdrlpa
