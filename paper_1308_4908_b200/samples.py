"""Scattered-sample mode: RadianceSamples, SampleIndex, LocalPolynomialRegressor.

Reference: pkg/src/hdrfuse/radiometry.py:140-261 (RadianceSample(s),
SampleIndex) and lpa.py:227-376 (LocalPolynomialRegressor, smoothing inputs,
_evaluate_index).  The unit-cell CSR index is built on the GPU (stable sort
by cell, torch as the device-memory/sort provider) and queries run in
``hdr_lpa_evaluate_samples`` -- a CUDA restatement of the reference's own
kernel boundary ``_kernels.lpa_evaluate`` in its exact operation order.
The index is a stable counting sort in the library (hdr_sample_index_*).
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


def _as_numpy(a):
    return a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a


def _device():
    return torch.device("cuda", torch.cuda.current_device())


@dataclass(frozen=True)
class RadianceSample:
    position: tuple
    channel: ColorChannel
    value: float
    sigma: float
    sensor_id: int


_COLUMNS = ("positions", "channels", "values", "sigmas", "sensor_ids")
_DTYPES = {"positions": np.float64, "channels": np.uint8, "values": np.float64,
           "sigmas": np.float64, "sensor_ids": np.int32}


class RadianceSamples:
    """Column-oriented samples (reference radiometry.py:150-205).

    Columns may be host numpy arrays or device torch tensors (as produced by
    ``RawFrameSet.materialize()``): device columns stay on the GPU for the
    index build and the evaluation, and the numpy attributes are filled on
    first access."""

    def __init__(self, positions, channels, values, sigmas, sensor_ids):
        cols = dict(zip(_COLUMNS, (positions, channels, values, sigmas, sensor_ids)))
        self._dev = None
        if all(isinstance(v, torch.Tensor) and v.is_cuda for v in cols.values()):
            tdt = {"positions": torch.float64, "channels": torch.uint8, "values": torch.float64,
                   "sigmas": torch.float64, "sensor_ids": torch.int32}
            dev = {k: v.to(tdt[k]).contiguous() for k, v in cols.items()}
            n = dev["values"].numel()
            dev["positions"] = dev["positions"].reshape(n, 2)
            if bool((dev["sigmas"] <= 0).any()):
                raise ValueError("sample sigmas must be positive")
            if not bool(torch.isfinite(dev["positions"]).all()):
                raise ValueError("sample positions must be finite")
            self._dev, self._host, self._n = dev, {}, n
        else:
            host = {}
            host["positions"] = np.ascontiguousarray(
                _as_numpy(positions), dtype=np.float64).reshape(-1, 2)
            n = len(host["positions"])
            for k in _COLUMNS[1:]:
                host[k] = np.ascontiguousarray(_as_numpy(cols[k]), dtype=_DTYPES[k]).reshape(n)
            if (host["sigmas"] <= 0).any():
                raise ValueError("sample sigmas must be positive")
            if not np.isfinite(host["positions"]).all():
                raise ValueError("sample positions must be finite")
            self._host, self._n = host, n
        self._indexes = {}
        self._uploads = {}

    def _column(self, name):
        if name not in self._host:
            self._host[name] = self._dev[name].cpu().numpy()
        return self._host[name]

    positions = property(lambda self: self._column("positions"))
    channels = property(lambda self: self._column("channels"))
    values = property(lambda self: self._column("values"))
    sigmas = property(lambda self: self._column("sigmas"))
    sensor_ids = property(lambda self: self._column("sensor_ids"))

    @property
    def on_device(self) -> bool:
        return self._dev is not None

    def device_column(self, name, device):
        """Column ``name`` as a device tensor (uploaded once if host-backed)."""
        device = torch.device(device)
        if self._dev is not None and self._dev[name].device == device:
            return self._dev[name]
        key = (name, str(device))
        if key not in self._uploads:
            self._uploads[key] = torch.from_numpy(self._column(name)).to(device)
        return self._uploads[key]

    def __len__(self) -> int:
        return self._n

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
        return cls(*(np.concatenate([getattr(p, a) for p in parts]) for a in _COLUMNS))

    def index(self, channel) -> "SampleIndex":
        key = int(channel)
        if key not in self._indexes:
            self._indexes[key] = SampleIndex(self, ColorChannel(key))
        return self._indexes[key]


class SampleIndex:
    """Unit-cell CSR grid over one channel's samples, on the GPU (reference
    radiometry.py:208-242): cells over floor(x), floor(y) from the bbox origin,
    samples stable-sorted by cell, packed rows [x, y, value, sigma^2].  Built
    by the library's stable counting sort (hdr_sample_index_bbox / _build):
    per-cell counts, a device scan, an atomic scatter and a per-cell restore
    of the original order -- no library sort."""

    def __init__(self, samples: RadianceSamples, channel: ColorChannel, device=None):
        dev = torch.device(device) if device is not None else _device()
        pos = samples.device_column("positions", dev)
        ch = samples.device_column("channels", dev)
        val = samples.device_column("values", dev)
        sig = samples.device_column("sigmas", dev)
        n = len(samples)
        lib = N.lib()
        st = torch.cuda.current_stream(dev)
        hdr = torch.empty(64, dtype=torch.uint8, device=dev)
        cnt, x0, y0, nx, ny = (ctypes.c_longlong(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int(),
                               ctypes.c_int())
        with torch.cuda.device(dev):
            N.check(lib.hdr_sample_index_bbox(pos.data_ptr(), ch.data_ptr(), n, int(channel),
                                              ctypes.byref(cnt), ctypes.byref(x0),
                                              ctypes.byref(y0), ctypes.byref(nx), ctypes.byref(ny),
                                              hdr.data_ptr(), st.cuda_stream),
                    "hdr_sample_index_bbox")
            self.n = int(cnt.value)
            self.x0, self.y0, self.nx, self.ny = int(x0.value), int(y0.value), int(nx.value), int(ny.value)
            ncells = self.nx * self.ny
            wsb = ctypes.c_size_t()
            N.check(lib.hdr_sample_index_workspace_bytes(n, ncells, ctypes.byref(wsb)),
                    "hdr_sample_index_workspace_bytes")
            ws = torch.empty(int(wsb.value), dtype=torch.uint8, device=dev)
            self.cell_start = torch.empty(ncells + 1, dtype=torch.int64, device=dev)
            self.packed = torch.empty((self.n, 4), dtype=torch.float64, device=dev)
            N.check(lib.hdr_sample_index_build(
                pos.data_ptr(), ch.data_ptr(), val.data_ptr(), sig.data_ptr(), n, int(channel),
                self.x0, self.y0, self.nx, self.ny, self.cell_start.data_ptr(),
                self.packed.data_ptr() if self.n else None, ws.data_ptr(), ws.numel(),
                st.cuda_stream), "hdr_sample_index_build")
        self.device = dev

    def __len__(self) -> int:
        return self.n

    def c_struct(self) -> N.HdrSampleIndex:
        return N.HdrSampleIndex(self.packed.data_ptr(), self.cell_start.data_ptr(), self.n,
                                self.x0, self.y0, self.nx, self.ny)


def evaluate_index(index: SampleIndex, qx, qy, order: int, scale: float, max_radius: float,
                   cond_threshold: float, weight_mode: str = "variance", steering=None):
    """_evaluate_index (lpa.py:322-376): (value, gx, gy) float64 -- numpy arrays
    for numpy queries, device tensors (no host round trip) for device queries."""
    on_dev = isinstance(qx, torch.Tensor)
    dev = index.device
    if on_dev:
        tqx = qx.to(dev, torch.float64).contiguous().reshape(-1)
        tqy = qy.to(dev, torch.float64).contiguous().reshape(-1)
    else:
        tqx = torch.from_numpy(np.ascontiguousarray(qx, dtype=np.float64).ravel()).to(dev)
        tqy = torch.from_numpy(np.ascontiguousarray(qy, dtype=np.float64).ravel()).to(dev)
    m = tqx.numel()
    if len(index) == 0:
        nan = torch.full((m,), float("nan"), dtype=torch.float64, device=dev)
        out = (nan, nan.clone(), nan.clone())
        return out if on_dev else tuple(o.cpu().numpy() for o in out)
    out = [torch.empty(m, dtype=torch.float64, device=dev) for _ in range(3)]
    an = [None] * 4
    if steering is not None:
        an = [a.to(dev, torch.float64).contiguous().reshape(-1) if isinstance(a, torch.Tensor)
              else torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).ravel()).to(dev)
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
    return tuple(out) if on_dev else tuple(o.cpu().numpy() for o in out)


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


def _grid_queries(out_size, ref_size, device):
    """lpa.py:393-396 meshgrid of the output pixel centres, built on the device."""
    xs, ys = grid_coordinates(out_size, ref_size or out_size)
    tx = torch.from_numpy(np.ascontiguousarray(xs)).to(device)
    ty = torch.from_numpy(np.ascontiguousarray(ys)).to(device)
    qy, qx = torch.meshgrid(ty, tx, indexing="ij")
    return qx.reshape(-1), qy.reshape(-1)


def reconstruct_channel_device(samples: RadianceSamples, out_size, params, channel,
                               ref_size=None, steering=None):
    """(value, gx, gy) (out_h, out_w) float64 device tensors of one channel."""
    out_w, out_h = out_size
    index = samples.index(channel)
    qx, qy = _grid_queries(out_size, ref_size, index.device)
    val, gx, gy = evaluate_index(index, qx, qy, params.order, params.channel_scale(channel),
                                 params.resolved_max_radius(), params.cond_threshold,
                                 params.weight_mode, steering)
    return val.reshape(out_h, out_w), gx.reshape(out_h, out_w), gy.reshape(out_h, out_w)


def reconstruct_channel_samples(samples: RadianceSamples, out_size, params, channel,
                                ref_size=None, steering=None):
    """reconstruct_channel on scattered samples (lpa.py:379-408): numpy planes."""
    return tuple(t.cpu().numpy() for t in reconstruct_channel_device(
        samples, out_size, params, channel, ref_size, steering))


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
