// staging.cuh -- TMA / mbarrier helpers and the per-tile staging of the
// fast kernels (region origins, coverage, coordinate tables, 3-D bulk copies).
#pragma once

#include "config.cuh"

namespace hdrlpa {

// ---------------------------------------------------------------------------
// Fast path: persistent CTAs, double-buffered TMA staging of the raw tiles.
// ---------------------------------------------------------------------------
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
// Bounded wait: a barrier that never completes (a lost TMA transaction)
// must not hang the GPU.  try_wait carries a suspend-time hint, so a waiting
// warp is parked until the phase completes instead of spinning through the
// issue slots of the warps that compute (busy polling was ~10 % of the tap
// kernel's instructions).  After HDR_MBAR_TIMEOUT_NS of %globaltimer the wait
// gives up: it raises HDR_FAULT_MBAR_TIMEOUT in the workspace header's fault
// word (read back by hdr_lpa_workspace_status) and returns false, and the
// caller's warp leaves the kernel.  No __trap: preemption, time-slicing or a
// debugger can stretch a healthy wait, and a trap kills the whole context.
#ifndef HDR_MBAR_SLEEP
#define HDR_MBAR_SLEEP 0  // ns of __nanosleep between failed polls
#endif
#ifndef HDR_MBAR_TIMEOUT_NS
#define HDR_MBAR_TIMEOUT_NS 20000000000ull  // 20 s
#endif
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#ifndef HDR_MBAR_TIMER_EVERY
#define HDR_MBAR_TIMER_EVERY 64  // failed polls between %globaltimer reads (power of 2)
#endif
__device__ __forceinline__ bool mbar_wait(uint64_t *bar, uint32_t parity, uint32_t *fault) {
    uint32_t done = 0;
    uint64_t t0 = 0;
    // the clock is read only every HDR_MBAR_TIMER_EVERY failed polls: a poll
    // loop that also read %globaltimer and compared 64-bit times each time was
    // ~30 % of the co-sited tap kernel's issued instructions
    for (uint32_t it = 1;; ++it) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
            " selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity), "r"(1000000u)
            : "memory");
        if (done) return true;
#if HDR_MBAR_SLEEP > 0
        __nanosleep(HDR_MBAR_SLEEP);
#endif
        if ((it & (HDR_MBAR_TIMER_EVERY - 1)) == 0) {
            const uint64_t now = global_ns();
            if (t0 == 0) {
                t0 = now;
            } else if (now - t0 > HDR_MBAR_TIMEOUT_NS) {
                atomicOr(fault, (uint32_t)HDR_FAULT_MBAR_TIMEOUT);
                return false;
            }
        }
    }
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
    // x: a TMA tile copy must start on a 16-byte boundary of the row
    // (measured: unaligned starts raise an illegal-instruction fault;
    // scripts/probes/tma_probe.cu).  The phase planes' x coordinate is in
    // floats (float2 elements: the sensor column; float4 merged planes: twice
    // it), so 4 columns are 16 bytes.  Both even, so the Bayer phase of a
    // staged pixel equals the parity of its coordinates.
    ox = xmin & ~3;
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
            // partial products, interleaved: {fl(T00 x), fl(T10 x)} per column
            // at off_tx0, {fl(T01 y), fl(T11 y)} per row at off_ty1.
            if (S.separable) {
                double *tx0t = (double *)(pb + S.off_tx0), *ty4t = (double *)(pb + S.off_ty4);
                for (int i = lane; i < S.rw; i += 32)
                    tx0t[i] = __dadd_rn(__dmul_rn(S.T[0], (double)(ox + i)), S.T[2]);
                for (int i = lane; i < S.rh; i += 32)
                    ty4t[i] = __dadd_rn(__dmul_rn(S.T[4], (double)(oy + i)), S.T[5]);
            } else {
                double2 *txi = (double2 *)(pb + S.off_tx0), *tyi = (double2 *)(pb + S.off_ty1);
                for (int i = lane; i < S.rw; i += 32) {
                    const double xd = (double)(ox + i);
                    txi[i] = make_double2(__dmul_rn(S.T[0], xd), __dmul_rn(S.T[3], xd));
                }
                for (int i = lane; i < S.rh; i += 32) {
                    const double yd = (double)(oy + i);
                    tyi[i] = make_double2(__dmul_rn(S.T[1], yd), __dmul_rn(S.T[4], yd));
                }
            }
        }
        __syncwarp();
    }
    if (lane == 0) {
        // the buffer's previous contents were read through the generic proxy
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        uint32_t bytes = 0;
        // element: float2 (f_hat, 1/den), or float4 for co-sited merged planes
        const int esz = P.merged ? 16 : 8;
        for (int s = 0; s < P.n_sensors; ++s) bytes += (uint32_t)(P.s[s].rw * P.s[s].rh * esz);
        mbar_expect_tx(full, bytes);
        // phase-plane coords: ox/2 elements = ox (float2) or 2 ox (float4) floats, oy/2
        for (int s = 0; s < P.n_sensors; ++s)
            tma_load_3d(pb + P.s[s].off_vi, &P.tmap[s], P.merged ? 2 * org[s][0] : org[s][0],
                        org[s][1] >> 1, 0, full);
    }
}

}  // namespace hdrlpa
