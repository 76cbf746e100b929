"""Scattered-sample mode: RadianceSamples, SampleIndex, LocalPolynomialRegressor.

Reference: pkg/src/hdrfuse/radiometry.py:140-261 (RadianceSample(s),
SampleIndex) and lpa.py:227-376 (LocalPolynomialRegressor, smoothing inputs,
_evaluate_index).  The unit-cell CSR index is built on the GPU (stable sort
by cell, torch as the device-memory/sort provider) and queries run in
``hdr_lpa_evaluate_samples`` -- a CUDA restatement of the reference's own
kernel boundary ``_kernels.lpa_evaluate`` in its exact operation order.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch
from sklearn.base import BaseEstimator, RegressorMixin

from . import _native as N
from .bayer import ColorChannel
from .lpa import SUPPORT_SIGMAS, grid_coordinates
from .validation import check_positions


def _device():
    return torch.device("cuda", torch.cuda.current_device())


@dataclass(frozen=True)
class RadianceSample:
    position: tuple
    channel: ColorChannel
    value: float
    sigma: float
    sensor_id: int


class RadianceSamples:
    """Column-oriented samples (reference radiometry.py:150-205)."""

    def __init__(self, positions, channels, values, sigmas, sensor_ids):
        self.positions = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 2)
        n = len(self.positions)
        self.channels = np.ascontiguousarray(channels, dtype=np.uint8).reshape(n)
        self.values = np.ascontiguousarray(values, dtype=np.float64).reshape(n)
        self.sigmas = np.ascontiguousarray(sigmas, dtype=np.float64).reshape(n)
        self.sensor_ids = np.ascontiguousarray(sensor_ids, dtype=np.int32).reshape(n)
        if (self.sigmas <= 0).any():
            raise ValueError("sample sigmas must be positive")
        if not np.isfinite(self.positions).all():
            raise ValueError("sample positions must be finite")
        self._indexes = {}

    def __len__(self) -> int:
        return len(self.values)

    def __getitem__(self, k: int) -> RadianceSample:
        return RadianceSample((float(self.positions[k, 0]), float(self.positions[k, 1])),
                              ColorChannel(int(self.channels[k])), float(self.values[k]),
                              float(self.sigmas[k]), int(self.sensor_ids[k]))

    @classmethod
    def empty(cls) -> "RadianceSamples":
        z = np.empty(0)
        return cls(np.empty((0, 2)), z, z, z, z)

    @classmethod
    def concatenate(cls, parts) -> "RadianceSamples":
        parts = [p for p in parts if len(p)]
        if not parts:
            return cls.empty()
        return cls(*(np.concatenate([getattr(p, a) for p in parts]) for a in
                     ("positions", "channels", "values", "sigmas", "sensor_ids")))

    def index(self, channel) -> "SampleIndex":
        key = int(channel)
        if key not in self._indexes:
            self._indexes[key] = SampleIndex(self, ColorChannel(key))
        return self._indexes[key]


class SampleIndex:
    """Unit-cell CSR grid over one channel's samples, on the GPU (reference
    radiometry.py:208-242): cells over floor(x), floor(y) from the bbox origin,
    samples stable-sorted by cell, packed rows [x, y, value, sigma^2]."""

    def __init__(self, samples: RadianceSamples, channel: ColorChannel, device=None):
        dev = torch.device(device) if device is not None else _device()
        sel = np.flatnonzero(samples.channels == int(channel))
        self.n = int(len(sel))
        x = torch.from_numpy(samples.positions[sel, 0].copy()).to(dev)
        y = torch.from_numpy(samples.positions[sel, 1].copy()).to(dev)
        if self.n:
            self.x0 = int(math.floor(float(x.min())))
            self.y0 = int(math.floor(float(y.min())))
            self.nx = int(math.floor(float(x.max()))) - self.x0 + 1
            self.ny = int(math.floor(float(y.max()))) - self.y0 + 1
        else:
            self.x0 = self.y0 = 0
            self.nx = self.ny = 1
        cell = (torch.floor(y).long() - self.y0) * self.nx + (torch.floor(x).long() - self.x0)
        order = torch.sort(cell, stable=True).indices
        counts = torch.bincount(cell, minlength=self.nx * self.ny)
        self.cell_start = torch.zeros(self.nx * self.ny + 1, dtype=torch.int64, device=dev)
        self.cell_start[1:] = torch.cumsum(counts, 0)
        v = torch.from_numpy(samples.values[sel].copy()).to(dev)
        s = torch.from_numpy(samples.sigmas[sel].copy()).to(dev)
        self.packed = torch.stack([x[order], y[order], v[order], (s * s)[order]], 1).contiguous()
        self.device = dev

    def __len__(self) -> int:
        return self.n

    def c_struct(self) -> N.HdrSampleIndex:
        return N.HdrSampleIndex(self.packed.data_ptr(), self.cell_start.data_ptr(), self.n,
                                self.x0, self.y0, self.nx, self.ny)


def evaluate_index(index: SampleIndex, qx, qy, order: int, scale: float, max_radius: float,
                   cond_threshold: float, weight_mode: str = "variance", steering=None):
    """_evaluate_index (lpa.py:322-376): (value, gx, gy) float64 numpy arrays."""
    qx = np.ascontiguousarray(qx, dtype=np.float64).ravel()
    qy = np.ascontiguousarray(qy, dtype=np.float64).ravel()
    m = len(qx)
    if len(index) == 0:
        nan = np.full(m, np.nan)
        return nan, nan.copy(), nan.copy()
    dev = index.device
    tqx, tqy = torch.from_numpy(qx).to(dev), torch.from_numpy(qy).to(dev)
    out = [torch.empty(m, dtype=torch.float64, device=dev) for _ in range(3)]
    an = [None] * 4
    if steering is not None:
        an = [torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).ravel()).to(dev)
              for a in steering]
    ix = index.c_struct()
    st = torch.cuda.current_stream(dev)
    N.check(N.lib().hdr_lpa_evaluate_samples(
        ctypes.byref(ix), tqx.data_ptr(), tqy.data_ptr(), m,
        *[a.data_ptr() if a is not None else None for a in an],
        1.0 / scale, SUPPORT_SIGMAS * math.sqrt(scale), int(order), float(max_radius),
        float(cond_threshold), N.HDR_WEIGHT_SIGMA if weight_mode == "sigma" else
        N.HDR_WEIGHT_VARIANCE, out[0].data_ptr(), out[1].data_ptr(), out[2].data_ptr(),
        st.cuda_stream), "hdr_lpa_evaluate_samples")
    return tuple(o.cpu().numpy() for o in out)


def smoothing_to_kernel_inputs(smoothing, n_queries: int):
    """Per-query SPD smoothing -> (Hinv entries, base radii) (lpa.py:296-319)."""
    H = np.asarray(smoothing, dtype=np.float64)
    if H.shape == (2, 2):
        H = np.broadcast_to(H, (n_queries, 2, 2))
    if H.shape != (n_queries, 2, 2):
        raise ValueError(f"smoothing must be 2x2 or ({n_queries}, 2, 2), got shape {H.shape}")
    a, b, d = H[:, 0, 0], H[:, 0, 1], H[:, 1, 1]
    if np.max(np.abs(b - H[:, 1, 0])) > 1e-12:
        raise ValueError("smoothing matrices must be symmetric")
    det = a * d - b * b
    if np.any(det <= 0) or np.any(a <= 0):
        raise ValueError("smoothing matrices must be positive definite")
    mean = 0.5 * (a + d)
    disc = np.hypot(0.5 * (a - d), b)
    radius = SUPPORT_SIGMAS * np.sqrt(mean + disc)
    return d / det, -b / det, a / det, radius


def reconstruct_channel_samples(samples: RadianceSamples, out_size, params, channel,
                                ref_size=None, steering=None):
    """reconstruct_channel on scattered samples (lpa.py:379-408)."""
    out_w, out_h = out_size
    xs, ys = grid_coordinates(out_size, ref_size or out_size)
    qx, qy = np.meshgrid(xs, ys)
    val, gx, gy = evaluate_index(samples.index(channel), qx, qy, params.order,
                                 params.channel_scale(channel), params.resolved_max_radius(),
                                 params.cond_threshold, params.weight_mode, steering)
    return val.reshape(out_h, out_w), gx.reshape(out_h, out_w), gy.reshape(out_h, out_w)


class LocalPolynomialRegressor(BaseEstimator, RegressorMixin):
    """Heteroscedastic local polynomial regression over scattered 2-D samples
    (reference lpa.py:227-293), evaluated on the GPU."""

    def __init__(self, order: int = 1, scale: float = 0.7, max_radius: Optional[float] = None,
                 cond_threshold: float = 1e8, weight_mode: str = "variance"):
        self.order = order
        self.scale = scale
        self.max_radius = max_radius
        self.cond_threshold = cond_threshold
        self.weight_mode = weight_mode

    def fit(self, X, y, sigma=None):
        X = check_positions(X)
        y = np.asarray(y, dtype=np.float64).ravel()
        if len(y) != len(X):
            raise ValueError(f"X has {len(X)} rows but y has {len(y)} values")
        if sigma is None:
            sigma = np.ones_like(y)
        else:
            sigma = np.broadcast_to(np.asarray(sigma, dtype=np.float64), y.shape).copy()
        if np.any(sigma <= 0):
            raise ValueError("sigma must be positive")
        samples = RadianceSamples(X, np.zeros(len(y)), y, sigma, np.zeros(len(y)))
        self.index_ = samples.index(ColorChannel.R)
        self.n_samples_ = len(y)
        return self

    def predict(self, X, return_gradients: bool = False, smoothing=None):
        if not hasattr(self, "index_"):
            raise RuntimeError("regressor is not fitted")
        X = check_positions(X)
        steering = None if smoothing is None else smoothing_to_kernel_inputs(smoothing, len(X))
        value, gx, gy = evaluate_index(
            self.index_, X[:, 0], X[:, 1], order=self.order, scale=self.scale,
            max_radius=self.max_radius if self.max_radius is not None else 10.0 * math.sqrt(self.scale),
            cond_threshold=self.cond_threshold, weight_mode=self.weight_mode, steering=steering)
        if return_gradients:
            return value, np.column_stack([gx, gy])
        return value
