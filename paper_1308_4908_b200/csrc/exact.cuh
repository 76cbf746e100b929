// exact.cuh -- the exact (slow) path: lpa_evaluate's ladder, the ICI rule,
// float64 recomputation, and lpa_slow_kernel over the fast path's work list.
#pragma once

#include "exact_ref.cuh"

namespace hdrlpa {

// ---------------------------------------------------------------------------
// Exact evaluation (slow path): lpa_evaluate's ladder (_kernels.py:257-300)
// and the ICI rule.
// ---------------------------------------------------------------------------
// skip0: the fast path decided (with certainty, solve_fast's FIT_FAIL) that
// step 0 of this order is invalid -- start at step 1 with the same radius
// sequence (r0, then min(1.5 r, max_radius))
template <int ORDER, class Sweep>
__device__ bool ladder_order(const DevParams &P, int c, const Sweep &sweep, PixelResult &R,
                             bool skip0 = false) {
    constexpr int PN = NC<ORDER>::P;
    double r = P.r[c][0];  // already min(r0, max_radius)
    int step = 0;
    if (skip0) {
        if (r >= P.max_radius * (1.0 - 1e-12)) return false;
        r = fmin(r * 1.5, P.max_radius);
        step = 1;
    }
    Acc<PN> acc;
    for (;;) {
        accumulate<ORDER, true>(P, c, 0, r, __dmul_rn(r, r), sweep, acc);
        R.work += acc.count;
        Fit fit;
        int st = solve_exact<PN>(acc, P.cond, fit);
        if (st == FIT_CRITICAL)  // the reference's closed form decides on noise: its order
            st = settle_critical<ORDER>(P, c, sweep.qx, sweep.qy, P.hinv[c][0], 0.0,
                                        P.hinv[c][0], r, fit);
        if (st == FIT_OK) {
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
__device__ void ladder(const DevParams &P, int c, const Sweep &sweep, PixelResult &R,
                       bool skip0 = false) {
    R.sidx = 0;
    if (ladder_order<ORDER>(P, c, sweep, R, skip0)) return;
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
// The running state (bounds, their error bounds, the selected estimate) lives
// across the scale loop; the fast kernel keeps it in a per-thread shared-memory
// slot (IciState) instead of registers, which the order-2 sweeps need.
struct IciState {
    double L, U;           // running intersection
    float eL, eU;          // their error bounds (rounded up)
    float val, gx, gy;     // estimate of the selected scale (the output is float32)
    float tgx, tgy;        // gradient of the scale being evaluated (until it is accepted)
    int sidx, count, precise;
};
struct IciRegs {  // the exact path: plain registers
    IciState st;
    __device__ __forceinline__ IciState &operator()() { return st; }
};
struct IciSmem {  // the fast path: volatile accesses keep it out of registers
    volatile IciState *p;
    __device__ __forceinline__ volatile IciState &operator()() { return *p; }
};
template <int ORDER, bool EXACT, class Sweep, class State = IciRegs>
__device__ int ici(const DevParams &P, int c, const Sweep &sweep, PixelResult &R,
                   State S = State()) {
    constexpr int PN = NC<ORDER>::P;
    Acc<PN> acc;
    Fit fit;
    S().precise = 1;
    // fast row sweeps: the variance sweep of scale k and the moment sweep of
    // scale k+1 share one traversal (FusedVarMom); the moments of k+1 are
    // wasted only when the search ends at k
    constexpr bool FUSED = !EXACT && ORDER >= 1 && HasRows<Sweep>::value;
    if constexpr (FUSED) accumulate<ORDER, EXACT>(P, c, 0, P.r[c][0], P.r2[c][0], sweep, acc);
    int k = 0;
    for (; k < P.n_scales; ++k) {
        if constexpr (!FUSED) accumulate<ORDER, EXACT>(P, c, k, P.r[c][k], P.r2[c][k], sweep, acc);
        R.work += acc.count;
        int st = EXACT ? solve_exact<PN>(acc, P.cond, fit) : solve_fast<PN>(acc, P.cond, fit);
        if constexpr (EXACT) {
            if (st == FIT_CRITICAL)
                st = settle_critical<ORDER>(P, c, sweep.qx, sweep.qy, P.hinv[c][k], 0.0,
                                            P.hinv[c][k], P.r[c][k], fit);
        }
        if (st == FIT_AMBIG) return FIT_AMBIG;
        if (st != FIT_OK) {
            if (k == 0) return FIT_FAIL;
            break;  // an invalid scale ends the search at k-1
        }
        const int count_k = acc.count;
        float tk = 0.f;
        double var_k;
        const double c0 = fit.c0;
        S().tgx = (float)fit.c1;  // parked in the state while the next sweep runs
        S().tgy = (float)fit.c2;
        if constexpr (FUSED) {
            RowVariance<ORDER> V{fit.g, P.hl[c][k], (bool)P.use_sigma, 0.0, 0.0, 0.0, 0.f};
            if (k + 1 < P.n_scales) {
                acc.zero();
                RowMoments<ORDER> M{acc, P.hl[c][k + 1]};
                FusedVarMom<ORDER> F{V, M};
                sweep.rows(c, k + 1, P.r[c][k + 1], P.r2[c][k + 1], F, k);
            } else {
                sweep.rows(c, k, P.r[c][k], P.r2[c][k], V);
            }
            tk = V.T;
            var_k = (double)V.v;
            if (HDR_VAR32 && !(var_k >= 1e-30 && var_k <= 1e37)) return FIT_AMBIG;
        } else {
            var_k = fit_variance<ORDER, EXACT>(P, c, k, sweep, fit.g, &tk);
        }
        const double sd = sqrt(var_k);
        const double lo = c0 - P.gamma * sd, hi = c0 + P.gamma * sd;
        // fast path: error bound of lo/hi (fp32 rounding of c0: fit_precise_sharp;
        // of sd: ICI_SD_EPS relative) -- an intersection test closer than the
        // bounds is decided by the exact path, so scale indices stay exact
        const float ek =
            EXACT ? 0.f
                  : __double2float_ru(2.0 * FAST_EPS * (double)tk +
                                      P.gamma * sd * (ICI_SD_EPS + VAR32_EPS_TERM * (count_k + 3)));
        if (k == 0) {
            S().L = lo;
            S().U = hi;
            S().eL = ek;
            S().eU = ek;
        } else {
            double L = S().L, U = S().U;
            float eL = S().eL, eU = S().eU;
            if (lo >= L) eL = lo > L ? ek : fmaxf(eL, ek);
            if (hi <= U) eU = hi < U ? ek : fmaxf(eU, ek);
            L = fmax(L, lo);
            U = fmin(U, hi);
            if (!EXACT && fabs(L - U) <= (double)eL + (double)eU) return FIT_AMBIG;
            if (L > U) break;
            S().L = L;
            S().U = U;
            S().eL = eL;
            S().eU = eU;
        }
        S().val = (float)c0;  // write_result rounds max(val, 0) to float32 anyway
        S().gx = S().tgx;
        S().gy = S().tgy;
        S().sidx = k;
        S().count = count_k;
        if constexpr (!EXACT) S().precise = fit_precise_sharp(c0, tk, P.prec_floor) ? 1 : 0;
    }
    R.val = S().val;
    R.gx = S().gx;
    R.gy = S().gy;
    R.sidx = S().sidx;
    R.count = S().count;
    if (!S().precise) return FIT_PREC;  // selected estimate too close to fp32 rounding limits
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
// (measured: cfg2 4 / 8 / 16 lanes within noise of each other, kept at 8;
// order 2 with ICI, cfg3 / cfg5: 4 lanes 1 % faster than 8)
#ifndef SLOW_LANES
#define SLOW_LANES 8
#endif
#ifndef SLOW_LANES_O2
#define SLOW_LANES_O2 4
#endif
constexpr uint32_t ITEM_DONE = 0xffffffffu;  // a recomputation that succeeded
// work-item kk code: scale 0 / the fixed scale certainly invalid (solve_fast's
// FIT_FAIL), the exact path runs the ladder from step 1
constexpr uint32_t KK_LADDER = 15u;

// The recomputations (kk > 0, from the end of the item list) in a kernel of
// their own: a small, uniform code path (one float64 fit at the selected
// scale) instead of sharing warps and the instruction cache with the full
// ladder / ICI evaluations (round 2: the mixed kernel issued 12 % of cycles,
// 10.6 of 32 lanes active, instruction-fetch stalls dominant).  A success
// writes the result and marks the slot ITEM_DONE; a failure leaves the item
// as a full evaluation (kk = 0) for lpa_slow_kernel.
template <int ORDER>
__global__ void __launch_bounds__(128) lpa_precise_kernel(const __grid_constant__ DevParams P) {
    constexpr int G = ORDER >= 2 ? SLOW_LANES_O2 : SLOW_LANES;
    const uint32_t n = *P.prec_count;
    const unsigned gmask = G >= 32 ? 0xffffffffu
                                   : ((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1));
    const int leader = (threadIdx.x & 31) & ~(G - 1);
    for (;;) {
        uint32_t i = 0;
        if ((threadIdx.x & (G - 1)) == 0) i = atomicAdd(P.prec_counter, 1u);
        i = __shfl_sync(gmask, i, leader);
        if (i >= n) break;
        const uint32_t slot = P.item_cap - 1u - i;
        const uint32_t item = P.work_items[slot];
        const int pix = P.row_begin * P.out_w + (int)(item >> 6), c = (int)(item & 3);
        const int kk = (int)((item >> 2) & 15);
        const int ox = pix % P.out_w, oy = pix / P.out_w;
        const GlobalSweep<G> sweep{P, qcoord(ox, P.sx), qcoord(oy, P.sy)};
        PixelResult R;
        const bool ok = precise_fit<ORDER>(P, c, kk - 1, sweep, R);
        if ((threadIdx.x & (G - 1)) == 0) {
            if (ok) write_result(P, pix, c, R);
            P.work_items[slot] = ok ? ITEM_DONE : (item & ~(15u << 2));
        }
    }
}

template <int ORDER>
__global__ void __launch_bounds__(128) lpa_slow_kernel(const __grid_constant__ DevParams P) {
    constexpr int G = ORDER >= 2 ? SLOW_LANES_O2 : SLOW_LANES;  // lanes per work item
    // the full evaluations, then the recomputation slots (those that failed
    // lpa_precise_kernel's float64 fit; ITEM_DONE ones are skipped)
    const uint32_t n0 = P.all_items ? P.all_items : *P.work_count;
    const uint32_t n = P.all_items ? P.all_items : n0 + *P.prec_count;
    // items are fetched dynamically (their cost varies by orders of magnitude)
    const unsigned gmask = G >= 32 ? 0xffffffffu
                                   : ((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1));
    const int leader = (threadIdx.x & 31) & ~(G - 1);
    for (;;) {
        uint32_t i = 0;
        if ((threadIdx.x & (G - 1)) == 0) i = atomicAdd(P.slow_counter, 1u);
        i = __shfl_sync(gmask, i, leader);
        if (i >= n) break;
        const uint32_t item = P.all_items ? (((i / 3u) << 6) | (i % 3u))
                                          : P.work_items[i < n0 ? i : P.item_cap - 1u - (i - n0)];
        if (item == ITEM_DONE) continue;
        const int pix = P.row_begin * P.out_w + (int)(item >> 6), c = (int)(item & 3);
        const int kk = (int)((item >> 2) & 15);
        const int ox = pix % P.out_w, oy = pix / P.out_w;
        const GlobalSweep<G> sweep{P, qcoord(ox, P.sx), qcoord(oy, P.sy)};
        PixelResult R;
        if (kk == (int)KK_LADDER) {
            ladder<ORDER>(P, c, sweep, R, true);
        } else if (kk && precise_fit<ORDER>(P, c, kk - 1, sweep, R)) {
            // the fast path's decisions stand; only the value was recomputed
        } else if (P.n_scales > 1) {
            if (ici<ORDER, true>(P, c, sweep, R) != FIT_OK) ladder<ORDER>(P, c, sweep, R);
        } else {
            ladder<ORDER>(P, c, sweep, R);
        }
        if ((threadIdx.x & (G - 1)) == 0) write_result(P, pix, c, R);
    }
}

}  // namespace hdrlpa
