"""Synthetic multi-sensor raw captures (input generator for tests and bench).

Forward camera model of the reference (pkg/src/hdrfuse/simulate.py:1-12,
:85-130): electrons ~ Poisson(t a n f), digital value
y = floor(g e + r + 0.5) with readout r ~ Normal(bias, Var[r]), clipped to
[0, saturation_level].  Ground-truth scenes are sampled bilinearly through
each sensor's transform.  This module only produces inputs; it is not on the
reconstruction path.  ``simulate_rig_device`` generates the same model on the
GPU (hdr_simulate_sensor; the multi-megapixel bench and video frames).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from .bayer import BayerPattern, ColorChannel, channel_map
from .images import CFAImage, HDRImage
from .radiometry import NoiseCalibration, SensorConfig

# Kodak KAI-04050 profile used throughout the reference's tests and configs
KODAK_GAIN = 0.27
KODAK_BIAS_DV = 72 * 0.27
KODAK_READVAR_DV2 = (0.27 * 11.8) ** 2


def identity_T():
    return np.array([[1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])


def translate_T(tx, ty):
    return np.array([[1.0, 0.0, float(tx)], [0.0, 1.0, float(ty)]])


def rotate_T(degrees, cx, cy, tx=0.0, ty=0.0):
    """Rotation by ``degrees`` about (cx, cy), then a shift (tx, ty)."""
    a = math.radians(degrees)
    c, s = math.cos(a), math.sin(a)
    return np.array([[c, -s, cx - c * cx + s * cy + tx], [s, c, cy - s * cx - c * cy + ty]])


@dataclass(frozen=True)
class SensorNoise:
    bias_dv: float = 0.0
    readout_var_dv2: float = 0.0
    nonuniformity: float = 1.0

    def calibration(self, width, height, gain=0.0) -> NoiseCalibration:
        return NoiseCalibration.uniform(width, height, self.bias_dv, self.readout_var_dv2,
                                        self.nonuniformity, gain)


@dataclass(frozen=True)
class RigSpec:
    sensors: Sequence[SensorConfig]
    noise: Sequence[SensorNoise]
    sensor_sizes: Sequence[tuple]
    seed: int = 0
    noise_free: bool = False

    def calibrations(self):
        return [n.calibration(w, h, c.gain) for n, c, (w, h) in
                zip(self.noise, self.sensors, self.sensor_sizes)]


def kodak_sensor(sensor_id, scaling, transform=None, exposure_time=0.1,
                 pattern=BayerPattern.RGGB) -> SensorConfig:
    return SensorConfig(sensor_id=sensor_id, exposure_time=exposure_time, gain=KODAK_GAIN,
                        exposure_scaling=scaling,
                        transform=identity_T() if transform is None else transform,
                        saturation_level=4095, bit_depth=12, pattern=pattern,
                        black_level=KODAK_BIAS_DV)


def kodak_noise() -> SensorNoise:
    return SensorNoise(KODAK_BIAS_DV, KODAK_READVAR_DV2, 1.0)


def _blur(img, sigma):
    r = int(math.ceil(3 * sigma))
    k = np.exp(-np.arange(-r, r + 1) ** 2 / (2 * sigma * sigma))
    k /= k.sum()
    p = np.pad(img, r, mode="edge")
    tmp = sum(k[i] * p[:, i:i + img.shape[1]] for i in range(2 * r + 1))
    return sum(k[i] * tmp[i:i + img.shape[0], :] for i in range(2 * r + 1))


def hdr_chart(width: int, height: int, top: float = 4.0e5, blur: float = 0.8) -> HDRImage:
    """Band-limited HDR test chart: radiance ramp 2e3..top e/s, a coloured bar
    target crossing the bright sensor's saturation, a checkerboard and a
    7-9e5 e/s highlight disk (the content of the reference's test chart)."""
    u = np.linspace(0.0, 1.0, width)[None, :]
    v = np.linspace(0.0, 1.0, height)[:, None]
    xi = np.arange(width)[None, :]
    yi = np.arange(height)[:, None]
    base = 2e3 + (top - 2e3) * u + 0.0 * v
    planes = [base.copy(), 0.8 * base, 1.15 * base]
    bars = (v > 0.12) & (v < 0.48)
    odd = ((xi // 5) % 2 == 1)
    for plane, a, b in zip(planes, (2.5e5, 6e4, 4e4), (4e4, 1.1e5, 2.8e5)):
        plane[bars & ~odd] = a
        plane[bars & odd] = b
    checker = (((xi // 4) + (yi // 4)) % 2 == 0) & (v > 0.55) & (v < 0.78) & (u > 0.08) & (u < 0.6)
    disk = (u - 0.80) ** 2 + (v - 0.86) ** 2 < 0.01
    for plane, cval, dval in zip(planes, (1.8e5, 3e4, 1.6e5), (8e5, 7e5, 9e5)):
        plane[np.broadcast_to(checker, plane.shape)] = cval
        plane[np.broadcast_to(disk, plane.shape)] = dval
    if blur > 0:
        planes = [_blur(p, blur) for p in planes]
    return HDRImage(np.ascontiguousarray(np.stack(planes, -1), np.float32))


def _bilinear(plane, X, Y):
    h, w = plane.shape
    X = np.clip(X, 0.0, w - 1.0)
    Y = np.clip(Y, 0.0, h - 1.0)
    x0 = np.floor(X).astype(np.int64)
    y0 = np.floor(Y).astype(np.int64)
    x1 = np.minimum(x0 + 1, w - 1)
    y1 = np.minimum(y0 + 1, h - 1)
    fx, fy = X - x0, Y - y0
    top = plane[y0, x0] * (1 - fx) + plane[y0, x1] * fx
    bot = plane[y1, x0] * (1 - fx) + plane[y1, x1] * fx
    return top * (1 - fy) + bot * fy


def sensor_rng(seed: int, sensor_id: int) -> np.random.Generator:
    """Counter-based stream per (run seed, sensor) -- reproducible frames."""
    return np.random.Generator(np.random.Philox(key=np.array([seed, sensor_id], dtype=np.uint64)))


def expose(f, cfg: SensorConfig, noise: SensorNoise, rng, noise_free=False):
    lam = cfg.exposure_time * noise.nonuniformity * cfg.exposure_scaling * np.maximum(f, 0.0)
    if noise_free:
        e, r = lam, noise.bias_dv
    else:
        big = lam > 1000.0
        e = np.empty_like(lam)
        e[~big] = rng.poisson(lam[~big])
        e[big] = np.maximum(np.round(rng.normal(lam[big], np.sqrt(lam[big]))), 0.0)
        r = rng.normal(noise.bias_dv, math.sqrt(noise.readout_var_dv2), size=lam.shape)
    y = np.floor(cfg.gain * e + r + 0.5)
    return np.clip(y, 0, cfg.saturation_level).astype(np.uint16)


def simulate_rig(gt: HDRImage, rig: RigSpec):
    """One raw frame per sensor (sensor coords mapped into gt coords by T)."""
    frames = []
    for cfg, noise, (w, h) in zip(rig.sensors, rig.noise, rig.sensor_sizes):
        ys, xs = np.mgrid[0:h, 0:w].astype(np.float64)
        X, Y = cfg.apply_transform(xs, ys)
        cmap = channel_map(cfg.pattern, w, h)
        f = np.empty((h, w))
        for c in ColorChannel:
            m = cmap == int(c)
            f[m] = _bilinear(gt.plane(c).astype(np.float64), X[m], Y[m])
        rng = None if rig.noise_free else sensor_rng(rig.seed, cfg.sensor_id)
        frames.append(CFAImage(expose(f, cfg, noise, rng, rig.noise_free), cfg.bit_depth,
                               cfg.pattern))
    return frames


def simulate_rig_device(gt: HDRImage, rig: RigSpec, device, seed: Optional[int] = None):
    """The same camera model on the GPU (hdr_simulate_sensor; reference
    simulate.py:92-212): one raw frame per sensor as an (h, w) int16 device
    tensor holding the uint16 digital values (rows padded to 16 bytes for the
    reconstruction's TMA staging).  Noise draws come from counter-based
    Philox4x32-10 streams keyed by (seed, sensor_id) like the reference's
    sensor_rng (:85-88); noise-free frames are bit-identical to
    :func:`simulate_rig`'s."""
    import ctypes

    import torch

    from . import _native as N

    device = torch.device(device)
    gtd = torch.as_tensor(np.ascontiguousarray(gt.data, dtype=np.float32), device=device)
    run_seed = rig.seed if seed is None else int(seed)
    out = []
    with torch.cuda.device(device):
        st = torch.cuda.current_stream(device)
        for cfg, noise, (w, h) in zip(rig.sensors, rig.noise, rig.sensor_sizes):
            pw = (w + 7) // 8 * 8
            buf = torch.empty((h, pw), dtype=torch.int16, device=device)
            s = N.HdrSensor()
            s.raw, s.width, s.height, s.pitch = buf.data_ptr(), w, h, pw
            s.saturation_level = int(cfg.saturation_level)
            tile = cfg.pattern.flat_tile()
            for i in range(4):
                s.tile[i] = int(tile[i])
            s.exposure_time, s.gain = float(cfg.exposure_time), float(cfg.gain)
            s.exposure_scaling = float(cfg.exposure_scaling)
            T = np.asarray(cfg.transform, dtype=np.float64).reshape(6)
            for i in range(6):
                s.transform[i] = float(T[i])
            s.bias, s.readout_variance = float(noise.bias_dv), float(noise.readout_var_dv2)
            s.nonuniformity = float(noise.nonuniformity)
            N.check(N.lib().hdr_simulate_sensor(
                gtd.data_ptr(), int(gt.width), int(gt.height), ctypes.byref(s),
                ctypes.c_ulonglong(run_seed & (2 ** 64 - 1)), int(cfg.sensor_id),
                1 if rig.noise_free else 0, st.cuda_stream), "hdr_simulate_sensor")
            out.append(buf[:, :w])
    return out


# ---------------------------------------------------------------------------
# BASELINE.json configurations
# ---------------------------------------------------------------------------
def baseline_rig(cfg: str, width: int, height: int, seed: int = 0, n_sensors: int = 3) -> RigSpec:
    """Rigs of the BASELINE configs: 3 (or 4) Kodak sensors at exposure
    scalings 1, 2^-4, 2^-8 (, 2^-12).  ``aligned``: identity transforms;
    ``misaligned``: sensor 1 translated by (0.4, 0.45) px and sensor 2
    rotated 0.3 deg about the centre plus a (0.25, -0.15) px shift."""
    scal = [1.0, 2.0 ** -4, 2.0 ** -8, 2.0 ** -12][:n_sensors]
    Ts = [identity_T() for _ in scal]
    if cfg == "misaligned":
        Ts[1] = translate_T(0.4, 0.45)
        if n_sensors > 2:
            Ts[2] = rotate_T(0.3, width / 2, height / 2, 0.25, -0.15)
        if n_sensors > 3:
            Ts[3] = translate_T(-0.3, 0.2)
    elif cfg != "aligned":
        raise ValueError(f"unknown rig {cfg!r}")
    sensors = [kodak_sensor(i, s, T) for i, (s, T) in enumerate(zip(scal, Ts))]
    return RigSpec(sensors=sensors, noise=[kodak_noise() for _ in sensors],
                   sensor_sizes=[(width, height)] * n_sensors, seed=seed)
