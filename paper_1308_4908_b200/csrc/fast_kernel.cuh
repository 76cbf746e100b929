// fast_kernel.cuh -- lpa_fast_kernel: the persistent tile kernel (tap, row-
// tap, sweep, ICI and CALPA-steered variants) and its per-pixel compute.
#pragma once

#include "exact.cuh"
#include "staging.cuh"

namespace hdrlpa {

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

// the pixel's own position in each sensor's staged phase planes (origins are
// even), computed once per pixel for all channels
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(a));
    return v;
}

// ESZ: bytes per staged phase-plane element (8: (f_hat, 1/den); 16: merged)
template <int NS, int ESZ = 8>
__device__ __forceinline__ void tap_bases(const DevParams &P, const unsigned char *sm,
                                          const int (*org)[2], int px, int py, uint32_t (&vbs)[NS]) {
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        if (s >= P.n_sensors) break;
        const DevSensor &S = P.s[s];
        const int pw = S.rw >> 1;
        vbs[s] = smem_addr(sm + S.off_vi) +
                 (uint32_t)ESZ * (uint32_t)(((py - org[s][1]) >> 1) * pw + ((px - org[s][0]) >> 1));
    }
}

// Co-sited taps (PAT 3/4): one merged sample per position, (sum 1/den,
// sum f_hat/den, sum |f_hat|/den, count) over the sensors, so one float64
// update per position instead of one per sensor sample.
template <int ORDER, bool CNT>
__device__ __forceinline__ void accumulate_merged_taps(const DevParams &P, const unsigned char *taps,
                                                       uint32_t vb, int c, int px, int py,
                                                       Acc<NC<ORDER>::P> &acc) {
    acc.zero();
    const int cls = ((py & 1) << 1) | (px & 1);
    const uint32_t txy = smem_addr(taps);
    const uint32_t tw = txy + (uint32_t)P.n_taps * (uint32_t)sizeof(TapXY);
    float count = 0.f;
    float sabs = 0.f;
    const int n = P.pat_cnt[0][c][cls];
    const int o = P.pat_off[0][c][cls];
#ifndef HDR_MRG_UNROLL
#define HDR_MRG_UNROLL 2
#endif
    constexpr int kUnroll = HDR_MRG_UNROLL;
#pragma unroll kUnroll
    for (int t = o; t < o + n; ++t) {
        const double2 X = lds_d2(txy + 16u * (uint32_t)t);
        const uint2 Q = lds_u2(tw + 8u * (uint32_t)t);
        const float4 e = lds_f4(vb + Q.y);
        const float W = __uint_as_float(Q.x);
        sabs = fmaf(W, e.z, sabs);
        const double dxx = ORDER >= 2 ? __dmul_rn(X.x, X.x) : 0.0;
        const double dyy = ORDER >= 2 ? __dmul_rn(X.y, X.y) : 0.0;
        acc.add_wy((double)(W * e.x), (double)(W * e.y), X.x, X.y, dxx, dyy);
        if constexpr (CNT) count += e.w;
    }
    acc.count = CNT ? (int)count : 1 << 20;
    acc.sabs = sabs;
}

template <int ORDER, bool CNT>
__device__ __forceinline__ void accumulate_taps(const DevParams &P, const unsigned char *taps,
                                                const uint32_t (&vbs)[PAT_MAXS], int c, int px,
                                                int py, Acc<NC<ORDER>::P> &acc) {
    acc.zero();
    const int cls = ((py & 1) << 1) | (px & 1);
    // shared-window addresses: one LDS.128 (dx, dy), one LDS.64 (W, byte
    // offset) and one LDS.64 (f_hat, 1/den) per tap
    const uint32_t txy = smem_addr(taps);
    const uint32_t tw = txy + (uint32_t)P.n_taps * (uint32_t)sizeof(TapXY);
    int count = 0;
    float sabs = 0.f;
#pragma unroll
    for (int s = 0; s < PAT_MAXS; ++s) {
        if (s >= P.n_sensors) break;
        const int n = P.pat_cnt[s][c][cls];
        const int o = P.pat_off[s][c][cls];
        const uint32_t vb = vbs[s];
#pragma unroll 4
        for (int t = o; t < o + n; ++t) {
            const double2 X = lds_d2(txy + 16u * (uint32_t)t);
            const uint2 Q = lds_u2(tw + 8u * (uint32_t)t);
            // masked samples carry (0, 0), so w and the
            // value are already zero exactly when the tap must not count
            const float2 e = lds_f2(vb + Q.y);
            const float w = __uint_as_float(Q.x) * e.y;
            sabs = fmaf(w, fabsf(e.x), sabs);
            const double dxx = ORDER >= 2 ? __dmul_rn(X.x, X.x) : 0.0;
            const double dyy = ORDER >= 2 ? __dmul_rn(X.y, X.y) : 0.0;
            acc.add((double)w, (double)e.x, X.x, X.y, dxx, dyy, 0);
            // predicated increment (setp + @p add): one instruction less than a select
            if constexpr (CNT)
                asm("{\n .reg .pred p;\n setp.gt.f32 p, %1, 0f00000000;\n @p add.s32 %0, %0, 1;\n}"
                    : "+r"(count)
                    : "f"(w));
        }
    }
    // Without the count/work planes the count is not needed: a window with
    // fewer than p weighted samples has a singular A, which the solve's
    // positive-definiteness guards reject or route to the exact path.
    acc.count = CNT ? count : 1 << 20;
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
// The channel-independent part (one cos/sin pair per pixel): the steering
// matrix C = gamma R diag(sigma, 1/sigma) R^T and sigma/gamma.
struct SteerPixel {
    double c11, c12, c22, s, g;
};
__device__ __forceinline__ SteerPixel steer_pixel(const DevParams &P, int pix) {
    const double th = P.st_theta[pix], s = P.st_sigma[pix], g = P.st_gamma[pix];
    double st, ct;
    sincos(th, &st, &ct);  // one argument reduction for both
    SteerPixel o;
    o.c11 = g * (s * ct * ct + st * st / s);
    o.c12 = g * (ct * st) * (1.0 / s - s);
    o.c22 = g * (s * st * st + ct * ct / s);
    o.s = s;
    o.g = g;
    return o;
}
// ... and per channel: H^-1 = C / h, r0 = 3 sqrt(h sigma / gamma) (same
// operation order as the one-piece form)
__device__ __forceinline__ void steer_channel(const DevParams &P, const SteerPixel &sp, int c,
                                              double *an) {
    const double h = P.h[c][0];  // channel scale
    an[0] = sp.c11 / h;
    an[1] = sp.c12 / h;
    an[2] = sp.c22 / h;
    an[3] = 3.0 * sqrt(h * sp.s / sp.g);
}
__device__ __forceinline__ void steer_inputs(const DevParams &P, int pix, int c, double *an) {
    steer_channel(P, steer_pixel(P, pix), c, an);
}

// Row-factored moments with the anisotropic window
// W = exp(-(h11 dx^2 + 2 h12 dx dy + h22 dy^2)) (_kernels.py:164-168): along a
// row dy is constant, so q = h11 dx^2 + (2 h12 dy) dx + h22 dy^2.
template <int ORDER>
struct RowAniso {
    static constexpr int PN = NC<ORDER>::P;
    RowMoments<ORDER> m;
    // pre-scaled by log2(e).  q is formed in float64: a strongly anisotropic
    // window's terms h11 dx^2, 2 h12 dx dy, h22 dy^2 cancel, and an fp32 sum
    // of them left weight errors far beyond FAST_EPS (1.4e-4 relative on a
    // sigma = 20 field in the stress fuzz); only the sum is rounded to fp32
    double h11, h12x2, h22;
    double a, b;  // per row: h22 dy^2, 2 h12 dy
    __device__ __forceinline__ void begin_row(double dy, double dyy) {
        m.begin_row(dy, dyy);
        a = h22 * dyy;
        b = h12x2 * dy;
    }
    __device__ __forceinline__ void end_row(double dy, double dyy) { m.end_row(dy, dyy); }
    __device__ __forceinline__ void sample(bool ok, double v, float iv, double dx, double dy,
                                           double dxx, double dyy, float, bool = true) {
        const float q2 = (float)fma(h11, dxx, fma(b, dx, a));
        // RowMoments' weight is ex2(-hl * d2f) * iv: feed it q2 with hl = 1
        m.sample(ok, v, iv, dx, dy, dxx, dyy, q2);
    }
    __device__ __forceinline__ void sample4(bool ok, float4 e, double dx, double dy, double dxx,
                                            double dyy, float) {
        const float q2 = (float)fma(h11, dxx, fma(b, dx, a));
        m.sample4(ok, e, dx, dxx, ex2_approx(-q2));
    }
    template <bool CNT = true>
    __device__ __forceinline__ void general(bool ok, double v, float iv, double dx, double dy,
                                            double dxx, double dyy, float, bool = true) {
        const float q2 = (float)fma(h11, dxx, fma(h12x2, dx * dy, h22 * dyy));
        m.template general<CNT>(ok, v, iv, dx, dy, dxx, dyy, q2);
    }
    __device__ __forceinline__ void count_add(int n) { m.count_add(n); }
};

template <int ORDER, class Sweep>
__device__ __forceinline__ void accumulate_aniso(const Sweep &sweep, int c, const double *an,
                                                 double r, double r2, Acc<NC<ORDER>::P> &acc) {
    constexpr double L2E = 1.4426950408889634;
    acc.zero();
    const double h11 = an[0] * L2E, h12x2 = 2.0 * an[1] * L2E, h22 = an[2] * L2E;
    if constexpr (ORDER >= 1) {
        RowAniso<ORDER> pol{RowMoments<ORDER>{acc, 1.0f}, h11, h12x2, h22, 0.0, 0.0};
        sweep.rows(c, -1, r, r2, pol);
    } else {
        sweep(c, -1, r, r2, [&](bool ok, double v, float iv, double dx, double dy, double dxx,
                                double dyy, float) {
            const float q2 = (float)fma(h11, dxx, fma(h12x2, dx * dy, h22 * dyy));
            const float w = ok ? ex2_approx(-q2) * iv : 0.f;
            const double y = ok ? v : 0.0;
            acc.sabs = fmaf(w, fabsf((float)y), acc.sabs);
            acc.add((double)w, y, dx, dy, dxx, dyy, ok ? 1 : 0);
        });
    }
}

template <int ORDER, bool ICI, int MAXC, int PAT, int RT, bool STEER, bool MRGS, bool ICISM>
__device__ __forceinline__ void tile_compute(const DevParams &P, const unsigned char *sm,
                                             const unsigned char *taps, int tcol, int trow,
                                             const int (*org)[2], bool tile_covered,
                                             int rot) {
    constexpr int PN = NC<ORDER>::P;
    // tile origin from its (column, row) index, published by the staging warp
    const int tx0 = tcol * TW, ty0 = P.row_begin + trow * TH;
    const int tx1 = min(tx0 + TW, P.out_w) - 1, ty1 = min(ty0 + TH, P.row_end) - 1;
    int px, py;
    if constexpr (PAT != 0 || RT) {
        // tap and row-tap kernels: each warp holds 32 pixels of ONE Bayer class (16
        // columns x 2 rows of equal parity), so the tap list is uniform across
        // the warp -- no padding of the shorter class list, broadcast tap
        // loads.  Two warps per class; rot swaps the x class between tiles so
        // light and heavy classes alternate per warp.
        static_assert(TW == 32 && TH == 8 && NT == 256, "class mapping assumes 32x8 tiles");
        const int lane = (int)(threadIdx.x & 31);
        if (RT && P.rt_period == 4) {
            // 2x output grid (16 classes): a warp takes one row class (py & 3)
            // and the pixel pairs of one anchor parity ((px >> 1) & 1) --
            // two classes that share their anchor, i.e. nearly the same rows
            const int slot = (int)(threadIdx.x >> 5) ^ rot;
            px = tx0 + 4 * ((lane & 15) >> 1) + 2 * (slot & 1) + (lane & 1);
            py = ty0 + (slot >> 1) + 4 * (lane >> 4);
        } else {
            const int slot = (int)(threadIdx.x >> 5) ^ (rot << 1);
            const int cl = slot >> 1;
            px = tx0 + (cl & 1) + 2 * (lane & 15);
            py = ty0 + (cl >> 1) + 4 * (slot & 1) + 2 * (lane >> 4);
        }
    } else {
        px = tx0 + (int)(threadIdx.x % TW);
        // warp w takes row w ^ rot: even and odd rows (different Bayer classes,
        // different amounts of work) alternate between tiles, so no warp is
        // systematically the slowest of its CTA
        py = ty0 + ((int)(threadIdx.x / TW) ^ rot);
    }
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
    __shared__ double2 s_q[NT];  // this thread's query point (TileSweep::qx / qy)
    // volatile store: stays ordered before TileSweep's volatile loads
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(smem_addr(&s_q[threadIdx.x])), "d"(qx),
                 "d"(qy));
    const TileSweep<MAXC, HDR_BRANCHY_O2 && (ORDER >= 2), RT, MRGS> sweep{P, sm, org,
                                                                   smem_addr(&s_q[threadIdx.x]),
                                                                   px, py, taps};
    // PAT: 1 taps (counting samples), 2 taps without the count, 3 / 4 the same
    // over co-sited merged samples
    constexpr bool MRG = PAT >= 3;
    uint32_t vbs[PAT_MAXS];
    if constexpr (PAT) tap_bases<PAT_MAXS, MRG ? 16 : 8>(P, sm, org, px, py, vbs);

    // STEER: the steering field's channel-independent part once per pixel
    SteerPixel sp{};
    if constexpr (STEER)
        if (covered) sp = steer_pixel(P, pix);
    for (int c = 0; c < 3; ++c) {
        if ((P.flags >> (2 + c)) & 1) continue;  // HDR_FLAG_SKIP_R/G/B
        PixelResult R;
        R.sidx = 0;
        int st = FIT_AMBIG;
        if (covered) {
            if constexpr (STEER) {
                double an[4];
                // the fast path rounds H^-1 to fp32 for its weights: C * (1/h)
                // instead of C / h there (the radius an[3] stays exact)
                const double ih = P.hinv[c][0];
                an[0] = sp.c11 * ih;
                an[1] = sp.c12 * ih;
                an[2] = sp.c22 * ih;
                an[3] = 3.0 * sqrt(P.h[c][0] * sp.s / sp.g);
                const double r = fmin(an[3], P.max_radius);
                Acc<PN> acc;
                accumulate_aniso<ORDER>(sweep, c, an, r, __dmul_rn(r, r), acc);
                R.work = acc.count;
                Fit fit;
                st = solve_fast<PN>(acc, P.cond, fit);
                if (st == FIT_OK && !fit_precise<PN>(fit, acc.sabs, r, P.prec_floor,
                                                     MRGS ? FAST_EPS_MERGED : FAST_EPS))
                    st = FIT_AMBIG;
                if (st == FIT_OK) {
                    R.count = acc.count;
                    R.val = fit.c0;
                    R.gx = ORDER >= 1 ? fit.c1 : qnan();
                    R.gy = ORDER >= 1 ? fit.c2 : qnan();
                    R.outcome = ORDER * 16;  // phase 0 (anisotropic), radius step 0
                }
            } else if constexpr (ICI) {
                // ICISM: the running ICI state in a per-thread shared-memory slot
                // (frees ~20 registers the order-2 sweeps spill without it; the
                // host picks it when it costs no occupancy)
                if constexpr (ICISM) {
                    __shared__ IciState s_ici[NT];
                    st = ici<ORDER, false>(P, c, sweep, R, IciSmem{&s_ici[threadIdx.x]});
                } else {
                    st = ici<ORDER, false>(P, c, sweep, R);
                }
            } else {
                Acc<PN> acc;
                if constexpr (MRG)
                    accumulate_merged_taps<ORDER, PAT == 3>(P, taps, vbs[0], c, px, py, acc);
                else if constexpr (PAT)
                    accumulate_taps<ORDER, PAT == 1>(P, taps, vbs, c, px, py, acc);
                else
                    accumulate<ORDER, false>(P, c, 0, P.r[c][0], P.r2[c][0], sweep, acc);
                R.work = acc.count;
                Fit fit;
                st = solve_fast<PN>(acc, P.cond, fit, P.grad != nullptr);
                if (st == FIT_OK && !fit_precise<PN>(fit, acc.sabs, P.r[c][0], P.prec_floor,
                                                     MRG ? FAST_EPS_MERGED : FAST_EPS)) {
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
            // kk = KK_LADDER: scale 0 certainly invalid (the ladder from step 1;
            // ICI kernels only -- the extra select cost the 64-register
            // co-sited tap kernel 1.7 %)
            const uint32_t kk = st == FIT_PREC ? (uint32_t)R.sidx + 1u
                                               : (ICI && st == FIT_FAIL ? KK_LADDER : 0u);
            const uint32_t item =
                ((uint32_t)(pix - P.row_begin * P.out_w) << 6) | (kk << 2) | (uint32_t)c;
            if (kk && kk != KK_LADDER)  // recomputations from the end of the list (lpa_precise_kernel)
                P.work_items[P.item_cap - 1u - atomicAdd(P.prec_count, 1u)] = item;
            else
                P.work_items[atomicAdd(P.work_count, 1u)] = item;
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
// co-sited tap kernels (PAT 3/4): 64 registers, 4 CTAs = 32 warps/SM (cfg2
// 0.198 -> 0.186 ms; the per-sensor tap kernel measured best at 3)
#ifndef HDR_MRG_MINBLOCKS
#define HDR_MRG_MINBLOCKS 4
#endif
// PAT: 0 no tap table, 1 taps (counting samples), 2 taps without the count
// (no count/work output planes requested), 3 / 4 the same over co-sited
// merged samples (radiance_merge_kernel)
// MRGS: CALPA's steered pass over co-sited merged planes (ORDER >= 1)
template <int ORDER, bool ICI, int MAXC, int PAT, int RT = 0, bool STEER = false,
          bool MRGS = false, bool ICISM = false>
// Per-sensor tap kernels are held to 80 registers: 3 CTAs per SM beat 2 by
// ~8% on cfg2 and 4 (64 registers) measured ~2% slower than 3.
#ifndef HDR_STEER_MINBLOCKS
#define HDR_STEER_MINBLOCKS 2
#endif
__global__ void __launch_bounds__(NT, (ORDER >= 2 ? HDR_O2_MINBLOCKS
                                               : (PAT >= 3 ? HDR_MRG_MINBLOCKS
                                                           : (PAT ? HDR_PAT_MINBLOCKS
                                                                  : (STEER ? HDR_STEER_MINBLOCKS
                                                                           : 2)))))
    lpa_fast_kernel(const __grid_constant__ DevParams P,
                    const __grid_constant__
                    typename std::conditional<(PAT != 0), TapParam, NoTaps>::type T) {
    constexpr int NBUF = nbuf_for(PAT, STEER);
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ int s_org[NBUF][MAXS][2];
    __shared__ int s_cov[NBUF];
    __shared__ unsigned s_done[NBUF];
    __shared__ int s_tile[NBUF];
    __shared__ int s_tcol[NBUF], s_trow[NBUF];  // the tile's column / row index
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
    __shared__ int s_next[NBUF];  // tile index the next refill of buffer b stages
    if (threadIdx.x == 0) {
#pragma unroll
        for (int b = 0; b < NBUF; ++b) {
            mbar_init(&bar_full[b], 1);
            s_done[b] = 0;
            s_next[b] = (int)atomicAdd(P.tile_counter, 1u);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();  // barriers initialised, taps staged
    // Tiles are handed out dynamically from a global counter (the workspace
    // header): a CTA whose tiles were cheap takes more, so all CTAs finish
    // together.  The staging warp takes the next index, publishes it in
    // s_tile[b] and releases it with the buffer's mbarrier (a plain arrive, no
    // copies, when the counter is exhausted: s_tile = -1 ends the loop).
    // The index a refill stages was taken from the counter one refill of this
    // buffer earlier (s_next), so the global atomic's latency is not on the
    // path from "buffer free" to "copy issued"; the refill takes the index for
    // the buffer's next refill after issuing its copies.
    auto refill = [&](int b) {  // one whole warp
        const int tn = s_next[b];
        if (tn < ntiles) {
            if ((threadIdx.x & 31) == 0) {
                s_tile[b] = tn;
                s_trow[b] = tn / P.tiles_x;
                s_tcol[b] = tn - s_trow[b] * P.tiles_x;
            }
            stage_tile<!PAT>(P, planes + b * P.buf_stride, tn, s_org[b], &s_cov[b], &bar_full[b]);
            if ((threadIdx.x & 31) == 0) s_next[b] = (int)atomicAdd(P.tile_counter, 1u);
        } else if ((threadIdx.x & 31) == 0) {
            s_tile[b] = -1;
            mbar_expect_tx(&bar_full[b], 0);
        }
    };
    if (threadIdx.x < 32) {
#pragma unroll
        for (int b = 0; b < NBUF; ++b) refill(b);
    }
    // No CTA-wide barrier in the loop: a warp waits only for its tile's data.
    // The LAST warp to finish the tile of buffer b refills b, so warps that
    // finish early run up to NBUF-1 tiles ahead instead of idling at a
    // __syncthreads while the slowest warp of the tile completes.
    constexpr int NWARPS = NT / 32;
    for (int i = 0;; ++i) {
        const int b = i % NBUF;
        unsigned char *pb = planes + b * P.buf_stride;
        if (!mbar_wait(&bar_full[b], (uint32_t)((i / NBUF) & 1), P.fault)) break;
        const int t = s_tile[b];
        if (t < 0) break;
        tile_compute<ORDER, ICI, MAXC, PAT, RT, STEER, MRGS, ICISM>(P, pb, taps, s_tcol[b], s_trow[b], s_org[b],
                                                       s_cov[b] != 0, HDR_ROW_ROT ? (i & 1) : 0);
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
        if (__shfl_sync(0xffffffffu, last, 0)) refill(b);
    }
}

}  // namespace hdrlpa
