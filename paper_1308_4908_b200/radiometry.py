"""Sensor configuration, noise calibration and the raw-frame handle.

Reference: pkg/src/hdrfuse/radiometry.py.  The radiometric model is the
reference's:

    f_hat   = (y - b_i) / (g t a_i n)                                  (:271-279)
    sigma^2 = max((g^2 t a n max(f_hat, 0) + Var[r]) / (g t a n)^2,
                  (1/12) / (g t a n)^2)                                (:282-295, :326-328)

and a pixel contributes a sample iff ``y < saturation_level`` and it is not
listed as defective (:298-300, :315-317).  Black level only enters through
the bias; negative f_hat is kept (:14-16).

What changes: :func:`frames_to_samples` does not build a sample list.  It
returns a :class:`RawFrameSet` -- the raw uint16 frames plus per-sensor
scalars/planes -- which the CUDA kernels consume directly (mapping, masking
and the radiometric conversion happen on the fly inside the reconstruction
kernel).  :meth:`RawFrameSet.materialize` produces the reference's
``RadianceSamples`` columns (bit-exact, device-resident) when a caller needs
them.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .bayer import BayerPattern, ColorChannel
from .images import CFAImage, FloatFrame
from .validation import ShapeMismatchError, check_positive


class ConfigurationError(ValueError):
    """Invalid sensor configuration (e.g. non-positive g*t*a*n)."""


@dataclass(frozen=True)
class SensorConfig:
    """Per-sensor capture parameters (reference radiometry.py:35-92).

    ``transform`` is the 2x3 affine map from sensor pixel centres (x, y) to
    virtual reference coordinates, evaluated as ``T00*x + T01*y + T02``.
    """

    sensor_id: int
    exposure_time: float
    gain: float
    exposure_scaling: float
    transform: np.ndarray
    saturation_level: int
    bit_depth: int
    pattern: BayerPattern
    black_level: float = 0.0
    defective: Optional[np.ndarray] = None

    def __post_init__(self):
        check_positive("exposure_time", self.exposure_time)
        check_positive("gain", self.gain)
        if not 0 < self.exposure_scaling <= 1:
            raise ConfigurationError(f"exposure_scaling must be in (0, 1], got {self.exposure_scaling}")
        T = np.asarray(self.transform, dtype=np.float64)
        if T.shape != (2, 3):
            raise ConfigurationError(f"transform must be 2x3, got shape {T.shape}")
        if abs(T[0, 0] * T[1, 1] - T[0, 1] * T[1, 0]) <= 1e-9:
            raise ConfigurationError("transform is not invertible")
        object.__setattr__(self, "transform", T)
        if not 8 <= self.bit_depth <= 16:
            raise ConfigurationError(f"bit_depth must be in [8, 16], got {self.bit_depth}")
        if not 0 < self.saturation_level <= (1 << self.bit_depth) - 1:
            raise ConfigurationError(
                f"saturation_level {self.saturation_level} outside {self.bit_depth}-bit range")
        if self.defective is not None:
            object.__setattr__(self, "defective", np.asarray(self.defective, dtype=np.int64).ravel())

    def apply_transform(self, x, y):
        T = self.transform
        x = np.asarray(x, dtype=np.float64)
        y = np.asarray(y, dtype=np.float64)
        return T[0, 0] * x + T[0, 1] * y + T[0, 2], T[1, 0] * x + T[1, 1] * y + T[1, 2]

    def invert_transform(self, X, Y):
        T = self.transform
        det = T[0, 0] * T[1, 1] - T[0, 1] * T[1, 0]
        u = np.asarray(X, dtype=np.float64) - T[0, 2]
        v = np.asarray(Y, dtype=np.float64) - T[1, 2]
        return (T[1, 1] * u - T[0, 1] * v) / det, (-T[1, 0] * u + T[0, 0] * v) / det


@dataclass(frozen=True)
class NoiseCalibration:
    """Calibrated noise model of one sensor (reference radiometry.py:95-136)."""

    bias: FloatFrame
    readout_variance: FloatFrame
    nonuniformity: FloatFrame
    gain_estimate: float = 0.0

    def __post_init__(self):
        shapes = {self.bias.data.shape, self.readout_variance.data.shape,
                  self.nonuniformity.data.shape}
        if len(shapes) != 1:
            raise ShapeMismatchError(f"calibration frames disagree in shape: {shapes}")
        if (self.readout_variance.data < 0).any():
            raise ValueError("readout variance must be non-negative everywhere")
        if (self.nonuniformity.data <= 0).any():
            raise ValueError("non-uniformity must be positive everywhere")

    @property
    def shape(self):
        return self.bias.data.shape

    def scalar(self, name: str):
        """The plane's value if the plane ``name`` is uniform, else None --
        memoised (the planes are immutable), so a per-frame call does not scan
        4-Mpx planes again (the GPU path passes uniform planes as scalars)."""
        cache = self.__dict__.get("_scalars")
        if cache is None:
            cache = {}
            object.__setattr__(self, "_scalars", cache)
        if name not in cache:
            flat = np.asarray(getattr(self, name).data).ravel()
            cache[name] = float(flat[0]) if flat.size and (flat == flat[0]).all() else None
        return cache[name]

    @classmethod
    def uniform(cls, width, height, bias=0.0, readout_variance=0.0, nonuniformity=1.0,
                gain_estimate=0.0) -> "NoiseCalibration":
        cal = cls(FloatFrame.full(width, height, bias),
                  FloatFrame.full(width, height, readout_variance),
                  FloatFrame.full(width, height, nonuniformity), gain_estimate)
        object.__setattr__(cal, "_scalars", {"bias": float(cal.bias.data.flat[0]),
                                             "readout_variance": float(cal.readout_variance.data.flat[0]),
                                             "nonuniformity": float(cal.nonuniformity.data.flat[0])})
        return cal


def _denominator(cfg: SensorConfig, a):
    d = cfg.gain * cfg.exposure_time * cfg.exposure_scaling * np.asarray(a, dtype=np.float64)
    if (d <= 0).any() or not np.isfinite(d).all():
        raise ConfigurationError("non-positive conversion denominator g*t*a*n")
    return d


def estimate_radiance(y, i, cfg: SensorConfig, cal: NoiseCalibration):
    """Radiance estimate f_hat for digital value(s) y at linear pixel index i."""
    i = np.asarray(i, dtype=np.int64)
    b = cal.bias.data.ravel()[i]
    a = cal.nonuniformity.data.ravel()[i]
    return (np.asarray(y, dtype=np.float64) - b) / _denominator(cfg, a)


def estimate_variance(f_hat, i, cfg: SensorConfig, cal: NoiseCalibration):
    """Model variance of f_hat (shot term clamped at zero radiance)."""
    i = np.asarray(i, dtype=np.int64)
    a = cal.nonuniformity.data.ravel()[i]
    var_r = cal.readout_variance.data.ravel()[i]
    g, t, n = cfg.gain, cfg.exposure_time, cfg.exposure_scaling
    shot = g * g * t * a * n * np.maximum(np.asarray(f_hat, dtype=np.float64), 0.0)
    return (shot + var_r) / _denominator(cfg, a) ** 2


def saturation_mask(img: CFAImage, cfg: SensorConfig) -> np.ndarray:
    """True where the digital value reached saturation (reference :298-300).

    Host convenience; the GPU path applies the same predicate inside the
    kernels and exports bit-planes through ``hdr_saturation_mask``
    (:meth:`RawFrameSet.saturation_masks`).
    """
    return img.data >= cfg.saturation_level


class RawFrameSet:
    """All sensors' raw frames + configs + calibrations, validated.

    This is what :func:`frames_to_samples` returns.  It is accepted by
    :func:`paper_1308_4908_b200.lpa.reconstruct_frame` in place of the
    reference's ``RadianceSamples``; nothing is materialised per sample.
    """

    def __init__(self, frames, configs, cals):
        if not (len(frames) == len(configs) == len(cals)):
            raise ShapeMismatchError(
                f"count mismatch: {len(frames)} frames, {len(configs)} configs, {len(cals)} calibrations")
        if not len(frames):
            raise ValueError("at least one sensor is required")
        self.frames = list(frames)
        self.configs = list(configs)
        self.cals = list(cals)
        for f, cfg, cal in zip(self.frames, self.configs, self.cals):
            if cal.shape != f.data.shape:
                raise ShapeMismatchError(
                    f"dimension mismatch: calibration {cal.shape} vs frame {f.data.shape}")
            a = cal.scalar("nonuniformity") if hasattr(cal, "scalar") else None
            _denominator(cfg, cal.nonuniformity.data if a is None else a)
        self._device_cache = {}

    def __len__(self) -> int:
        return len(self.frames)

    @property
    def reference_size(self):
        """(width, height) of the first sensor (the CLI's default ref size)."""
        return self.frames[0].width, self.frames[0].height

    def device(self, device=None):
        """Device-resident copy (cached): see :class:`~.engine.DeviceRig`."""
        from .engine import DeviceRig

        key = str(device)
        if key not in self._device_cache:
            self._device_cache[key] = DeviceRig.from_host(self.frames, self.configs, self.cals,
                                                          device=device)
        return self._device_cache[key]

    def saturation_masks(self, device=None):
        """Per-sensor boolean (h, w) masks computed by the GPU kernel."""
        return self.device(device).saturation_masks()

    def materialize(self, device=None):
        """The reference's ``RadianceSamples`` (sensor-major, raster order),
        computed and compacted on the GPU from the raw frames: values and
        sigmas bit-identical to the reference's float64 columns
        (``hdr_sample_planes``); the columns stay device-resident."""
        from .samples import RadianceSamples

        return RadianceSamples(*self.device(device).materialize_samples())


def frames_to_samples(frames, configs, cals) -> RawFrameSet:
    """Validated raw-frame handle (replaces reference radiometry.py:339-349)."""
    return RawFrameSet(frames, configs, cals)


def frame_to_samples(img: CFAImage, cfg: SensorConfig, cal: NoiseCalibration) -> RawFrameSet:
    return RawFrameSet([img], [cfg], [cal])


__all__ = [
    "ColorChannel", "ConfigurationError", "NoiseCalibration", "RawFrameSet", "SensorConfig",
    "estimate_radiance", "estimate_variance", "frame_to_samples", "frames_to_samples",
    "saturation_mask",
]
