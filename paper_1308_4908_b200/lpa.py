"""Local polynomial approximation (LPA) reconstruction -- public API.

Mirrors the reference's reconstruction API (pkg/src/hdrfuse/lpa.py):

* :class:`ReconstructionParams` -- same fields, defaults and validation as
  lpa.py:40-74, plus the ICI extension (``ici_scales``, ``ici_ratio``,
  ``ici_gamma``).  ``ici_scales=1`` is the reference's
  fixed-scale behaviour.
* :func:`reconstruct_frame` / :func:`reconstruct_channel` -- same signatures
  and return types as lpa.py:379-433, computed by the sm_100a kernels behind
  the C ABI (``hdr_lpa_reconstruct``).  The ``samples`` argument is the
  :class:`~.radiometry.RawFrameSet` returned by
  :func:`~.radiometry.frames_to_samples` (or a device-resident
  :class:`~.engine.DeviceRig`).

Per-pixel semantics (window, weights, basis, fallback ladder, NaN policy,
clamping) are the reference's; see DESIGN.md "Numerics" for the precision.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .bayer import ColorChannel
from .images import HDRImage
from .validation import check_positive

# support truncation radius = 3 length-scales (reference lpa.py:37)
SUPPORT_SIGMAS = 3.0


@dataclass(frozen=True)
class ReconstructionParams:
    """Reconstruction knobs (reference lpa.py:40-74) + ICI extension."""

    order: int = 1
    scale: float = 0.7
    per_channel_scale: bool = True
    max_support_radius: Optional[float] = None
    cond_threshold: float = 1e8
    weight_mode: str = "variance"
    ici_scales: int = 1
    ici_ratio: float = math.sqrt(2.0)
    ici_gamma: float = 1.5

    def __post_init__(self):
        if self.order not in (0, 1, 2):
            raise ValueError(f"order must be 0, 1 or 2, got {self.order}")
        check_positive("scale", self.scale)
        if self.weight_mode not in ("variance", "sigma"):
            raise ValueError(f"unknown weight_mode {self.weight_mode!r}")
        if self.max_support_radius is not None:
            if self.max_support_radius < math.sqrt(self.scale):
                raise ValueError("max_support_radius must be at least sqrt(scale)")
        if not 1 <= int(self.ici_scales) <= 8:
            raise ValueError(f"ici_scales must be in [1, 8], got {self.ici_scales}")
        if int(self.ici_scales) > 1 and not self.ici_ratio > 1.0:
            raise ValueError(f"ici_ratio must exceed 1, got {self.ici_ratio}")
        if not (self.ici_gamma >= 0 and math.isfinite(self.ici_gamma)):
            raise ValueError(f"ici_gamma must be finite and >= 0, got {self.ici_gamma}")
        check_positive("cond_threshold", self.cond_threshold)

    def channel_scale(self, channel) -> float:
        """h of a channel; green is sampled twice as densely (lpa.py:66-69)."""
        if self.per_channel_scale and int(channel) == int(ColorChannel.G):
            return self.scale / math.sqrt(2.0)
        return self.scale

    def resolved_max_radius(self) -> float:
        """Largest support radius of the fallback ladder (lpa.py:71-74).
        Always derived from ``scale``, never from the channel scale."""
        if self.max_support_radius is not None:
            return float(self.max_support_radius)
        return 10.0 * math.sqrt(self.scale)

    def channel_scales(self, channel) -> list:
        """ICI scale set h_k = channel_scale * ici_ratio**k, k < ici_scales."""
        h = self.channel_scale(channel)
        return [h * self.ici_ratio ** k for k in range(int(self.ici_scales))]


def n_coefficients(order: int) -> int:
    return (order + 1) * (order + 2) // 2


def basis_row(delta, order: int) -> np.ndarray:
    """Polynomial basis at offset (dx, dy): [1, dx, dy, dx^2, dx dy, dy^2][:p]
    (reference lpa.py:104-118)."""
    if order not in (0, 1, 2):
        raise ValueError(f"order must be 0, 1 or 2, got {order}")
    dx, dy = float(delta[0]), float(delta[1])
    full = [1.0, dx, dy, dx * dx, dx * dy, dy * dy]
    return np.array(full[: n_coefficients(order)])


def grid_coordinates(out_size, ref_size):
    """Output pixel centres in reference coordinates (lpa.py:213-224)."""
    out_w, out_h = out_size
    ref_w, ref_h = ref_size
    xs = (np.arange(out_w) + 0.5) * (ref_w / out_w) - 0.5
    ys = (np.arange(out_h) + 0.5) * (ref_h / out_h) - 0.5
    return xs, ys


def _device_rig(samples):
    from .engine import DeviceRig
    from .radiometry import RawFrameSet

    if isinstance(samples, DeviceRig):
        return samples
    if isinstance(samples, RawFrameSet):
        return samples.device()
    raise TypeError(
        "reconstruct_frame expects the RawFrameSet returned by frames_to_samples, a "
        f"DeviceRig or RadianceSamples, got {type(samples).__name__}")


def _is_scattered(samples) -> bool:
    from .samples import RadianceSamples

    return isinstance(samples, RadianceSamples)


def reconstruct_frame(samples, out_size, params: ReconstructionParams, ref_size=None,
                      return_gradients: bool = False):
    """LPA reconstruction of R, G and B into an :class:`HDRImage`
    (reference lpa.py:411-433): radiance clamped at zero, NaN where no order
    succeeds; gradients (when requested) unclamped, per channel.

    ``samples`` is the RawFrameSet of :func:`frames_to_samples` (fused raw
    path) or scattered :class:`~.samples.RadianceSamples` (CSR index path)."""
    from .engine import to_host

    if _is_scattered(samples):
        import torch

        from .samples import reconstruct_channel_device

        planes, grads = [], {}
        for ch in ColorChannel:
            val, gx, gy = reconstruct_channel_device(samples, out_size, params, ch, ref_size)
            planes.append(torch.clamp_min(val, 0.0).to(torch.float32))  # keeps NaN (lpa.py:428)
            if return_gradients:
                grads[ch] = (to_host(gx), to_host(gy))
        img = HDRImage._from_device_output(to_host(torch.stack(planes, 2)))
        return (img, grads) if return_gradients else img
    rig = _device_rig(samples)
    out = rig.reconstruct(out_size, params, ref_size=ref_size, want_grad=return_gradients)
    img = HDRImage._from_device_output(to_host(out["rgb"]))
    rig.status(out_size)  # synchronous API: surface a kernel fault (after the sync above)
    if not return_gradients:
        return img
    g = to_host(out["grad"].double())
    grads = {ch: (g[int(ch), 0], g[int(ch), 1]) for ch in ColorChannel}
    return img, grads


def reconstruct_channel(samples, out_size, params: ReconstructionParams, channel,
                        ref_size=None, steering=None):
    """(value, grad_x, grad_y) planes of one channel (reference lpa.py:379-408).
    ``value`` is unclamped like the reference's; NaN where no fit exists."""
    from .engine import to_host

    if _is_scattered(samples):
        from .samples import reconstruct_channel_samples

        return reconstruct_channel_samples(samples, out_size, params, channel, ref_size, steering)
    if steering is not None:
        raise ValueError("per-query steering arrays need scattered RadianceSamples; use "
                         "calpa_reconstruct for raw frames")
    rig = _device_rig(samples)
    out = rig.reconstruct(out_size, params, ref_size=ref_size, want_grad=True, raw_value=True)
    c = int(channel)
    val = to_host(out["value"][c].double())
    g = to_host(out["grad"][c].double())
    return val, g[0], g[1]
