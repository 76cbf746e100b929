// launch.cuh -- host-side launch helpers shared by the library's translation
// units (hdr_lpa.cu and the per-order fast_o*.cu).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <atomic>
#include <climits>
#include <type_traits>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges for nsys / ncu --nvtx

#include "hdr_lpa.h"
#include "config.cuh"
#include "fast_kernel.cuh"

namespace hdrlpa {

// scoped NVTX range around the host-side enqueue of a library stage (no-op
// unless a tool is attached)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

extern thread_local char g_last_error[256];
extern std::atomic<unsigned long long> g_launches;
#define COUNT_LAUNCH() g_launches.fetch_add(1, std::memory_order_relaxed)
int cuda_fail(const char *where);
int set_smem_attr(const void *fn, int bytes);
extern thread_local bool g_timer_on;
extern thread_local cudaEvent_t g_timer_ev[2];
extern thread_local bool g_timer_recorded;
bool timer_active(cudaStream_t st);

template <int ORDER, bool ICI, int MAXC, int PAT = 0, int RT = 0, bool STEER = false,
          bool MRGS = false, bool ICISM = false>
inline int launch_fast(const DevParams &P, const TapParam &T, int tiles, int smem_bytes,
                       cudaStream_t st) {
    const void *fn = (const void *)lpa_fast_kernel<ORDER, ICI, MAXC, PAT, RT, STEER, MRGS, ICISM>;
    if (set_smem_attr(fn, smem_bytes) != HDR_OK) return HDR_ERR_CUDA;
    int dev = 0, nsm = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT, smem_bytes) != cudaSuccess ||
        per_sm < 1)
        return cuda_fail("occupancy query");
    const int grid = min(tiles, nsm * per_sm);  // persistent: every CTA loops over tiles
    const bool timed = timer_active(st);
    if (timed) cudaEventRecord(g_timer_ev[0], st);
    COUNT_LAUNCH();
    if constexpr (PAT)
        lpa_fast_kernel<ORDER, ICI, MAXC, PAT, RT, STEER, MRGS, ICISM><<<grid, NT, smem_bytes, st>>>(P, T);
    else
        lpa_fast_kernel<ORDER, ICI, MAXC, PAT, RT, STEER, MRGS, ICISM>
            <<<grid, NT, smem_bytes, st>>>(P, NoTaps{});
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("lpa_fast_kernel launch");
    if (timed) {
        cudaEventRecord(g_timer_ev[1], st);
        g_timer_recorded = true;
    }
    return HDR_OK;
}


// CTAs per SM a fast kernel reaches with `smem_bytes` of dynamic shared memory
template <int ORDER, bool ICI, int MAXC, int PAT, int RT, bool STEER, bool MRGS, bool ICISM>
inline int fast_occupancy(int smem_bytes) {
    const void *fn = (const void *)lpa_fast_kernel<ORDER, ICI, MAXC, PAT, RT, STEER, MRGS, ICISM>;
    if (set_smem_attr(fn, smem_bytes) != HDR_OK) return 0;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT, smem_bytes) != cudaSuccess)
        return 0;
    return per_sm;
}

// ICI kernels: the variant with the ICI state in shared memory (no spills)
// whenever its extra static shared memory costs no CTA per SM, else the
// register variant (e.g. 4-sensor rigs, whose staged planes fill the SM).
template <int ORDER, int MAXC, int RT>
inline int launch_ici(const DevParams &P, const TapParam &T, int tiles, int smem_bytes,
                      cudaStream_t st) {
    const int occ_sm = fast_occupancy<ORDER, true, MAXC, 0, RT, false, false, true>(smem_bytes);
    const int occ_rg = fast_occupancy<ORDER, true, MAXC, 0, RT, false, false, false>(smem_bytes);
    if (getenv("HDR_DEBUG_RT"))
        fprintf(stderr, "ici kernel: dynamic smem %d B, CTAs/SM smem-state %d, register-state %d\n",
                smem_bytes, occ_sm, occ_rg);
    if (occ_sm > 0 && occ_sm >= occ_rg)
        return launch_fast<ORDER, true, MAXC, 0, RT, false, false, true>(P, T, tiles, smem_bytes, st);
    return launch_fast<ORDER, true, MAXC, 0, RT, false, false, false>(P, T, tiles, smem_bytes, st);
}

// Pf: the fast kernel's parameters (a one-sensor view over the merged planes
// in co-sited mode), P: the full rig for the exact path.
template <int ORDER>
int launch_all(const DevParams &Pf, const DevParams &P, const TapParam &T, int tiles,
                      int smem_bytes, int maxc, cudaStream_t st) {
    NvtxRange nv("hdr_lpa tile + exact kernels");
    int rc;
    const bool cnt = P.count || P.work;
    if (P.all_items) {  // no staged path (hdr_lpa_reconstruct): the exact path for everything
        int dev = 0, nsm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        COUNT_LAUNCH();
        lpa_slow_kernel<ORDER><<<nsm * 4, 128, 0, st>>>(P);
        return cudaPeekAtLastError() == cudaSuccess ? HDR_OK : cuda_fail("lpa_slow_kernel launch");
    }
    if (Pf.merged)
        rc = cnt ? launch_fast<ORDER, false, 4, 3>(Pf, T, tiles, smem_bytes, st)
                 : launch_fast<ORDER, false, 4, 4>(Pf, T, tiles, smem_bytes, st);
    else if (P.pat)
        rc = cnt ? launch_fast<ORDER, false, 4, 1>(P, T, tiles, smem_bytes, st)
                 : launch_fast<ORDER, false, 4, 2>(P, T, tiles, smem_bytes, st);
    // row taps (every separable sensor tapped; MAXC only sizes the column
    // sweep of separable sensors, so it is irrelevant here): RT 1 counts the
    // valid samples per tap for the count / work planes, RT 2 counts taps
    else if (P.rt && P.n_scales > 1)
        rc = cnt ? launch_ici<ORDER, 6, 1>(P, T, tiles, smem_bytes, st)
                 : launch_ici<ORDER, 6, 2>(P, T, tiles, smem_bytes, st);
    else if (P.rt)
        rc = cnt ? launch_fast<ORDER, false, 4, 0, 1>(P, T, tiles, smem_bytes, st)
                 : launch_fast<ORDER, false, 4, 0, 2>(P, T, tiles, smem_bytes, st);
    else if (P.n_scales > 1)
        rc = maxc <= 6 ? launch_ici<ORDER, 6, 0>(P, T, tiles, smem_bytes, st)
                       : launch_ici<ORDER, 8, 0>(P, T, tiles, smem_bytes, st);
    else
        rc = maxc <= 4 ? launch_fast<ORDER, false, 4>(P, T, tiles, smem_bytes, st)
                       : launch_fast<ORDER, false, 8>(P, T, tiles, smem_bytes, st);
    if (rc != HDR_OK) return rc;
    if (P.flags & HDR_FLAG_FAST_ONLY) return HDR_OK;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    COUNT_LAUNCH();
    lpa_precise_kernel<ORDER><<<nsm * 4, 128, 0, st>>>(P);
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("lpa_precise_kernel launch");
    COUNT_LAUNCH();
    lpa_slow_kernel<ORDER><<<nsm * 4, 128, 0, st>>>(P);
    if (cudaPeekAtLastError() != cudaSuccess) return cuda_fail("lpa_slow_kernel launch");
    return HDR_OK;
}


extern template int launch_all<0>(const DevParams &, const DevParams &, const TapParam &, int, int,
                                  int, cudaStream_t);
extern template int launch_all<1>(const DevParams &, const DevParams &, const TapParam &, int, int,
                                  int, cudaStream_t);
extern template int launch_all<2>(const DevParams &, const DevParams &, const TapParam &, int, int,
                                  int, cudaStream_t);

}  // namespace hdrlpa
