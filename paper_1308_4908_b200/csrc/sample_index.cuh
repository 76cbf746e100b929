// sample_index.cuh -- scattered-sample mode on the device without library
// sorts: the stable counting sort of the reference's SampleIndex
// (radiometry.py:208-242) and the order-preserving compaction of the sample
// planes into RadianceSamples columns (radiometry.py:303-349).
//
// SampleIndex: cells are unit squares over floor(x), floor(y) from the bbox
// origin of one channel's samples; samples are sorted by cell STABLY (ties in
// original order) and packed as rows [x, y, value, sigma^2].  Device steps:
//   1. sample_bbox_kernel    count and floor bounds of the channel (atomics)
//   2. cell_count_kernel     per-cell counts
//   3. exclusive scan        cell_start (int64), scan_* kernels
//   4. cell_scatter_kernel   slot = cell_start[cell] + atomic fill: original
//                            index per slot (order within a cell arbitrary)
//   5. cell_order_kernel     per cell, insertion sort of its slots by original
//                            index (cells hold a handful of samples), then
//                            the packed rows are gathered in that order
// The result equals np.argsort(cell, kind="stable") + the reference's packing.
#pragma once

#include "config.cuh"

namespace hdrlpa {

constexpr int SCAN_BLOCK = 1024;

__device__ __forceinline__ long long floor_ll(double v) { return (long long)floor(v); }

// bbox[0] = count, [1] = min floor x, [2] = min floor y, [3] = max floor x, [4] = max floor y
__global__ void sample_bbox_kernel(const double2 *pos, const uint8_t *ch, long long n, int channel,
                                   long long *bbox) {
    long long cnt = 0, xlo = LLONG_MAX, ylo = LLONG_MAX, xhi = LLONG_MIN, yhi = LLONG_MIN;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        if (ch[i] != channel) continue;
        const double2 p = pos[i];
        const long long fx = floor_ll(p.x), fy = floor_ll(p.y);
        ++cnt;
        xlo = min(xlo, fx);
        ylo = min(ylo, fy);
        xhi = max(xhi, fx);
        yhi = max(yhi, fy);
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, m);
        xlo = min(xlo, __shfl_xor_sync(0xffffffffu, xlo, m));
        ylo = min(ylo, __shfl_xor_sync(0xffffffffu, ylo, m));
        xhi = max(xhi, __shfl_xor_sync(0xffffffffu, xhi, m));
        yhi = max(yhi, __shfl_xor_sync(0xffffffffu, yhi, m));
    }
    if ((threadIdx.x & 31) == 0 && cnt) {
        atomicAdd((unsigned long long *)&bbox[0], (unsigned long long)cnt);
        atomicMin(&bbox[1], xlo);
        atomicMin(&bbox[2], ylo);
        atomicMax(&bbox[3], xhi);
        atomicMax(&bbox[4], yhi);
    }
}

__global__ void sample_bbox_init_kernel(long long *bbox) {
    bbox[0] = 0;
    bbox[1] = bbox[2] = LLONG_MAX;
    bbox[3] = bbox[4] = LLONG_MIN;
}

__device__ __forceinline__ long long cell_of(double2 p, int x0, int y0, int nx) {
    return (floor_ll(p.y) - y0) * (long long)nx + (floor_ll(p.x) - x0);  // radiometry.py:226-229
}

__global__ void cell_count_kernel(const double2 *pos, const uint8_t *ch, long long n, int channel,
                                  int x0, int y0, int nx, long long *counts) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        if (ch[i] == channel)
            atomicAdd((unsigned long long *)&counts[cell_of(pos[i], x0, y0, nx)], 1ull);
}

// Exclusive scan of int64 (block of SCAN_BLOCK): out[i] = sum in[0..i), block
// totals to sums[blockIdx] (when sums != nullptr).
__global__ void scan_block_kernel(const long long *in, long long *out, long long n,
                                  long long *sums) {
    __shared__ long long warp_tot[SCAN_BLOCK / 32];
    const long long i = blockIdx.x * (long long)SCAN_BLOCK + threadIdx.x;
    const long long v = i < n ? in[i] : 0;
    long long x = v;  // inclusive warp scan
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int m = 1; m < 32; m <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, x, m);
        if (lane >= m) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
        long long t = lane < SCAN_BLOCK / 32 ? warp_tot[lane] : 0;
#pragma unroll
        for (int m = 1; m < 32; m <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, t, m);
            if (lane >= m) t += y;
        }
        if (lane < SCAN_BLOCK / 32) warp_tot[lane] = t;  // inclusive over warps
    }
    __syncthreads();
    const long long before = w ? warp_tot[w - 1] : 0;
    if (i < n) out[i] = before + x - v;
    if (sums && threadIdx.x == SCAN_BLOCK - 1) sums[blockIdx.x] = before + x;
}

__global__ void scan_add_kernel(long long *out, long long n, const long long *offsets) {
    const long long i = blockIdx.x * (long long)SCAN_BLOCK + threadIdx.x;
    if (i < n) out[i] += offsets[blockIdx.x];
}

__global__ void cell_scatter_kernel(const double2 *pos, const uint8_t *ch, long long n, int channel,
                                    int x0, int y0, int nx, const long long *cell_start,
                                    unsigned long long *fill, long long *perm) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        if (ch[i] != channel) continue;
        const long long c = cell_of(pos[i], x0, y0, nx);
        perm[cell_start[c] + (long long)atomicAdd(&fill[c], 1ull)] = i;
    }
}

// one thread per cell: restore the original order inside the cell (the
// stable sort's tie rule), then gather the packed rows [x, y, value, var]
__global__ void cell_order_kernel(const double2 *pos, const double *values, const double *sigmas,
                                  long long ncells, const long long *cell_start, long long *perm,
                                  double4 *packed) {
    for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < ncells;
         c += (long long)gridDim.x * blockDim.x) {
        const long long a = cell_start[c], b = cell_start[c + 1];
        for (long long k = a + 1; k < b; ++k) {  // insertion sort (a few entries)
            const long long v = perm[k];
            long long j = k - 1;
            while (j >= a && perm[j] > v) {
                perm[j + 1] = perm[j];
                --j;
            }
            perm[j + 1] = v;
        }
        for (long long k = a; k < b; ++k) {
            const long long i = perm[k];
            const double2 p = pos[i];
            const double s = sigmas[i];
            packed[k] = make_double4(p.x, p.y, values[i], s * s);  // radiometry.py:240
        }
    }
}

// ---------------------------------------------------------------------------
// Order-preserving compaction of the sample planes (hdr_sample_planes) into
// the reference's sample columns: sensor pixel (x, y) with sigma > 0, raster
// order; position = apply_transform (T00*x + T01*y + T02, no contraction,
// radiometry.py:84), channel = tile[y % 2][x % 2] (bayer.py:54-59).
// ---------------------------------------------------------------------------
__global__ void row_count_kernel(const double *sigma, int w, int h, long long *rows) {
    const int y = blockIdx.x;
    if (y >= h) return;
    long long cnt = 0;
    for (int x = threadIdx.x; x < w; x += blockDim.x) cnt += sigma[(size_t)y * w + x] > 0.0;
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, m);
    __shared__ long long part[32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += part[k];
        rows[y] = t;
    }
}

// one block per row; the row's kept pixels in column order (block-wide scan)
__global__ void row_compact_kernel(const DevSensor S, int sensor_id, const double *value,
                                   const double *sigma, int w, int h, const long long *row_start,
                                   long long offset, double2 *pos, uint8_t *chan, double *vals,
                                   double *sigs, int *ids) {
    const int y = blockIdx.x;
    if (y >= h) return;
    __shared__ long long base;
    __shared__ int warp_cnt[32];
    if (threadIdx.x == 0) base = offset + row_start[y];
    __syncthreads();
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const double yd = (double)y;
    const double t1y = __dmul_rn(S.T[1], yd), t4y = __dmul_rn(S.T[4], yd);
    for (int x0 = 0; x0 < w; x0 += blockDim.x) {
        const int x = x0 + threadIdx.x;
        const size_t i = (size_t)y * w + x;
        const bool keep = x < w && sigma[i] > 0.0;
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) warp_cnt[wi] = __popc(bal);
        __syncthreads();
        int before = 0;
        for (int k = 0; k < wi; ++k) before += warp_cnt[k];
        int total = 0;
        for (int k = 0; k < nw; ++k) total += warp_cnt[k];
        if (keep) {
            const long long o = base + before + __popc(bal & ((1u << lane) - 1u));
            const double xd = (double)x;
            pos[o] = make_double2(__dadd_rn(__dadd_rn(__dmul_rn(S.T[0], xd), t1y), S.T[2]),
                                  __dadd_rn(__dadd_rn(__dmul_rn(S.T[3], xd), t4y), S.T[5]));
            int c = 0;
            const int ph = ((y & 1) << 1) | (x & 1);
            for (int q = 0; q < 3; ++q)
                if ((S.phmask[q] >> ph) & 1) c = q;
            chan[o] = (uint8_t)c;
            vals[o] = value[i];
            sigs[o] = sigma[i];
            ids[o] = sensor_id;
        }
        __syncthreads();
        if (threadIdx.x == 0) base += total;
        __syncthreads();
    }
}

}  // namespace hdrlpa
