// simulate.cuh -- the camera simulator on the device (input generator for the
// bench and the video pipeline; reference simulate.py:85-212).
//
// Per sensor pixel (x, y): position in ground-truth coordinates through the
// sensor transform (sample_scene, simulate.py:92-115: T00*x + T01*y + T02,
// edge-clamped bilinear lookup of the pixel's Bayer channel plane, float64 in
// numpy's operation order); lambda = t * a * n * max(f, 0); electrons ~
// Poisson(lambda) for lambda <= 1000, else max(round(Normal(lambda,
// sqrt(lambda))), 0) (_sample_poisson, :117-127); readout ~ Normal(bias,
// sqrt(Var[r])); y = clip(floor(g e + r + 0.5), 0, saturation) (expose,
// :130-166).  noise_free replaces the draws by their means (bit-identical to
// the reference's noise-free frames).
//
// Random numbers: a counter-based Philox4x32-10 stream keyed by (seed,
// sensor id) -- the reference's sensor_rng(seed, sensor_id) keys numpy's
// Philox the same way (simulate.py:85-88) -- with the counter = (pixel index,
// draw number), so frames are reproducible and independent of the launch
// geometry.  The draws follow the reference's distributions, not numpy's bit
// streams (numpy's normal/poisson algorithms are not restated): the tests
// compare moments against the model and the reference simulator's frames.
#pragma once

#include "config.cuh"

namespace hdrlpa {

struct Philox4 {
    uint32_t v[4];
};

__device__ __forceinline__ Philox4 philox4x32_10(uint4 ctr, uint2 key) {
    uint32_t c0 = ctr.x, c1 = ctr.y, c2 = ctr.z, c3 = ctr.w, k0 = key.x, k1 = key.y;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    Philox4 o;
    o.v[0] = c0;
    o.v[1] = c1;
    o.v[2] = c2;
    o.v[3] = c3;
    return o;
}

// a stream of uniforms in (0, 1) for one pixel: counter (pixel, block)
struct PixelRng {
    uint2 key;
    unsigned long long pix;
    uint32_t block;
    int used;
    Philox4 buf;
    __device__ __forceinline__ double uniform() {  // 53-bit, never 0 or 1
        if (used >= 4) {
            buf = philox4x32_10(make_uint4((uint32_t)pix, (uint32_t)(pix >> 32), block++, 0x5EEDu),
                                key);
            used = 0;
        }
        const uint32_t a = buf.v[used], b = buf.v[used + 1];
        used += 2;
        const unsigned long long m = ((unsigned long long)(a >> 5) << 26) | (b >> 6);
        return ((double)m + 0.5) * (1.0 / 9007199254740992.0);
    }
    __device__ __forceinline__ double normal() {  // Box-Muller (one of the pair)
        const double u1 = uniform(), u2 = uniform();
        return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
    }
    // Poisson: multiplication method below 10, else PTRS (Hoermann 1993, the
    // transformed rejection numpy's legacy and Generator samplers use)
    __device__ double poisson(double lam) {
        if (lam <= 0.0) return 0.0;
        if (lam < 10.0) {
            const double L = exp(-lam);
            double p = 1.0;
            int k = -1;
            do {
                ++k;
                p *= uniform();
            } while (p > L);
            return (double)k;
        }
        const double slam = sqrt(lam), loglam = log(lam);
        const double b = 0.931 + 2.53 * slam, a = -0.059 + 0.02483 * b;
        const double invalpha = 1.1239 + 1.1328 / (b - 3.4), vr = 0.9277 - 3.6224 / (b - 2.0);
        for (;;) {
            const double U = uniform() - 0.5, V = uniform();
            const double us = 0.5 - fabs(U);
            const double k = floor((2.0 * a / us + b) * U + lam + 0.43);
            if (us >= 0.07 && V <= vr) return k;
            if (k < 0.0 || (us < 0.013 && V > us)) continue;
            if (log(V) + log(invalpha) - log(a / (us * us) + b) <= -lam + k * loglam - lgamma(k + 1.0))
                return k;
        }
    }
};

// gt: H x W x 3 float32 (HDRImage layout); T: sensor -> ground-truth coordinates
__global__ void simulate_sensor_kernel(const float *gt, int gw, int gh, const DevSensor S,
                                       unsigned long long seed, int sensor_id, int noise_free,
                                       uint16_t *out, int pitch) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
    if (x >= S.width || y >= S.height) return;
    const double xd = (double)x, yd = (double)y;
    // sample_scene (simulate.py:92-115), numpy's operation order
    double u = __dadd_rn(__dadd_rn(__dmul_rn(S.T[0], xd), __dmul_rn(S.T[1], yd)), S.T[2]);
    double v = __dadd_rn(__dadd_rn(__dmul_rn(S.T[3], xd), __dmul_rn(S.T[4], yd)), S.T[5]);
    u = fmin(fmax(u, 0.0), (double)(gw - 1));
    v = fmin(fmax(v, 0.0), (double)(gh - 1));
    const int u0 = (int)floor(u), v0 = (int)floor(v);
    const int u1 = min(u0 + 1, gw - 1), v1 = min(v0 + 1, gh - 1);
    const double fu = __dsub_rn(u, (double)u0), fv = __dsub_rn(v, (double)v0);
    int c = 0;
    const int ph = ((y & 1) << 1) | (x & 1);
    for (int q = 0; q < 3; ++q)
        if ((S.phmask[q] >> ph) & 1) c = q;
    auto P = [&](int yy, int xx) { return (double)gt[((size_t)yy * gw + xx) * 3 + c]; };
    const double top = __dadd_rn(__dmul_rn(P(v0, u0), __dsub_rn(1.0, fu)), __dmul_rn(P(v0, u1), fu));
    const double bot = __dadd_rn(__dmul_rn(P(v1, u0), __dsub_rn(1.0, fu)), __dmul_rn(P(v1, u1), fu));
    const double f = __dadd_rn(__dmul_rn(top, __dsub_rn(1.0, fv)), __dmul_rn(bot, fv));
    // expose (simulate.py:130-166)
    const double lam = __dmul_rn(__dmul_rn(__dmul_rn(S.t, S.nonuni), S.n), f > 0.0 ? f : 0.0);
    double e, r;
    if (noise_free) {
        e = lam;
        r = S.bias;
    } else {
        PixelRng rng{make_uint2((uint32_t)seed, (uint32_t)(seed >> 32) ^ (0x9E3779B9u * (uint32_t)(sensor_id + 1))),
                     (unsigned long long)y * S.width + x, 0u, 4, {}};
        if (lam <= 1000.0) {  // _POISSON_NORMAL_CROSSOVER
            e = rng.poisson(lam);
        } else {
            e = fmax(rint(lam + sqrt(lam) * rng.normal()), 0.0);
        }
        r = S.bias + sqrt(S.readvar) * rng.normal();
    }
    double yv = floor(__dadd_rn(__dadd_rn(__dmul_rn(S.g, e), r), 0.5));  // round half-up
    yv = fmin(fmax(yv, 0.0), (double)S.sat);
    out[(size_t)y * pitch + x] = (uint16_t)yv;
}

}  // namespace hdrlpa
