// config.cuh -- tiling, workspace and tuning constants of the sm_100a kernels.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "hdr_lpa.h"
#include "lpa_device.cuh"

namespace hdrlpa {

// Debug builds (-DHDR_DEBUG_BOUNDS=1, scripts/gpu_bounds.sh): every staged
// shared-memory read of the tile sweeps is range-checked; a violation raises
// HDR_FAULT_BOUNDS in the workspace header (hdr_lpa_workspace_status) instead
// of reading out of range.  compute-sanitizer is not available on the
// measurement pool, so this is the memory-safety check the tests run.
#ifndef HDR_DEBUG_BOUNDS
#define HDR_DEBUG_BOUNDS 0
#endif
#if HDR_DEBUG_BOUNDS
#define HDR_BOUNDS(P, cond) \
    do { if (!(cond)) atomicOr((P).fault, (uint32_t)HDR_FAULT_BOUNDS); } while (0)
#else
#define HDR_BOUNDS(P, cond) do { } while (0)
#endif

constexpr int TW = 32, TH = 8, NT = TW * TH;  // NT consumer threads, one per tile pixel

// workspace layout: [header: work counter][pre-computed taps][work items]
static const size_t WS_HEADER = 256;
// header words: 0 full-evaluation items, 1 tile counter, 2 exact-path item
// counter, 3 fault bits, 4 recomputation items, 5 recomputation counter
static const int WS_HEADER_WORDS = 6;
// Order-2 tile sweeps: skip samples outside the disk with branches (1) or
// accumulate them with zero weight (0; the row-factored moments make a
// sample cheap enough that divergent branches cost more than they save)
#ifndef HDR_BRANCHY_O2
#define HDR_BRANCHY_O2 1
#endif
static_assert(sizeof(DevParams) + TAP_PARAM_BYTES <= 32764, "kernel parameter space");
// plane buffers per CTA of the fast kernel's staging pipeline (measured: 3
// buffers gain nothing on cfg2 and cost cfg3 5% through occupancy)
// alternate the row parity each warp takes per tile (fast kernel)
#ifndef HDR_ROW_ROT
#define HDR_ROW_ROT 1
#endif
// sensors of a tap-table (PAT) rig: per-pixel phase-plane bases in registers
constexpr int PAT_MAXS = 4;
#ifndef HDR_NBUF
#define HDR_NBUF 2
#endif
constexpr int NBUF = HDR_NBUF;
// tap kernels (PAT): measured 2 / 3 / 4 / 6 buffers on cfg2 -- more buffers
// only cost occupancy (4 CTAs/SM of the co-sited kernel need 2)
#ifndef HDR_NBUF_TAP
#define HDR_NBUF_TAP 2
#endif
constexpr int NBUF_TAP = HDR_NBUF_TAP;
// CALPA's steered pass: windows up to max_radius make each tile's staged
// region large and its compute short
#ifndef HDR_NBUF_STEER
#define HDR_NBUF_STEER 2
#endif
constexpr int NBUF_STEER = HDR_NBUF_STEER;
__host__ __device__ constexpr int nbuf_for(int pat, bool steer = false) {
    return steer ? NBUF_STEER : (pat ? NBUF_TAP : NBUF);
}
static const size_t LUT_BYTES = 65536 * sizeof(double2);
static const size_t RT_TABLE_BYTES = 64 * 1024;  // row-tap table (workspace, then shared memory)

template <int ORDER>
struct NC {
    static constexpr int P = (ORDER + 1) * (ORDER + 2) / 2;
};

// shared-memory helpers (32-bit shared-window addresses)
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
// 8-byte shared-memory load at a 32-bit shared address (row-tap samples)
__device__ __forceinline__ float2 lds_f2(uint32_t a) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
    return v;
}

}  // namespace hdrlpa
