"""Structure-adaptive second pass (CALPA) -- reference pkg/src/hdrfuse/steering.py.

An isotropic first pass (order >= 1) gives the gradient field of the G
channel on the output grid; a 9x9 weighted structure tensor per pixel gives
an orientation theta, an elongation sigma and a scaling gamma
(``hdr_steering_field``); the second pass then fits every channel with the
per-pixel anisotropic window H^{-1} = C/h, C = gamma U_theta diag(sigma,
1/sigma) U_theta^T, falling back per pixel to the isotropic window before
the radius/order ladder (``hdr_lpa_reconstruct_steered``).  Same API, fields
and validation as the reference; everything runs on the GPU.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _native as N
from .bayer import ColorChannel
from .images import HDRImage
from .lpa import SUPPORT_SIGMAS, ReconstructionParams, _device_rig
from .engine import to_host
from .validation import check_positive


@dataclass(frozen=True)
class AdaptiveParams:
    """Steering knobs on top of a base reconstruction (reference steering.py:38-69)."""

    alpha: float = 0.005
    lambda1: float = 1.0
    lambda2: float = 0.001
    gradient_window: int = 9
    sigma_max: float = 50.0
    share_steering: bool = True
    gradient_scale: Optional[float] = None
    base: ReconstructionParams = field(default_factory=ReconstructionParams)

    def __post_init__(self):
        if self.alpha < 0:
            raise ValueError(f"alpha must be >= 0, got {self.alpha}")
        if self.lambda1 < 0:
            raise ValueError(f"lambda1 must be >= 0, got {self.lambda1}")
        check_positive("lambda2", self.lambda2)
        if self.gradient_window < 3 or self.gradient_window % 2 == 0:
            raise ValueError(f"gradient_window must be odd and >= 3, got {self.gradient_window}")
        if self.base.order < 1:
            raise ValueError("steering needs a base reconstruction of order >= 1")
        if self.base.ici_scales != 1:
            raise ValueError("the steered pass is fixed-scale (ici_scales must be 1)")


@dataclass(frozen=True)
class SteeringField:
    """Per output pixel theta (rad), sigma >= 1, gamma > 0 (float64 device tensors)."""

    theta: torch.Tensor
    sigma: torch.Tensor
    gamma: torch.Tensor

    def numpy(self):
        return tuple(t.cpu().numpy() for t in (self.theta, self.sigma, self.gamma))

    def covariance_entries(self):
        """(C11, C12, C22) of C = gamma U diag(sigma, 1/sigma) U^T (steering.py:80-87)."""
        ct, st, s, g = torch.cos(self.theta), torch.sin(self.theta), self.sigma, self.gamma
        return (g * (s * ct * ct + st * st / s), g * (ct * st) * (1.0 / s - s),
                g * (s * st * st + ct * ct / s))

    def kernel_inputs(self, scale: float):
        """Per-pixel H^{-1} entries and base radii (steering.py:94-107)."""
        c11, c12, c22 = self.covariance_entries()
        r0 = SUPPORT_SIGMAS * torch.sqrt(scale * self.sigma / self.gamma)
        return c11 / scale, c12 / scale, c22 / scale, r0


def gradient_field(samples, out_size, params: ReconstructionParams, channel=ColorChannel.G,
                   ref_size=None):
    """Isotropic first pass: (value, grad_x, grad_y) device float32 planes."""
    if params.order < 1:
        raise ValueError("gradient estimation needs order >= 1")
    rig = _device_rig(samples)
    out = rig.reconstruct(out_size, params, ref_size=ref_size, want_grad=True, raw_value=True)
    c = int(channel)
    return out["value"][c], out["grad"][c, 0], out["grad"][c, 1]


def auto_gradient_scale(values: torch.Tensor) -> float:
    """99.5th percentile of |finite values| (steering.py:206-211)."""
    v = values[torch.isfinite(values)].abs().double()
    if v.numel() == 0:
        return 1.0
    s = float(torch.quantile(v.flatten()[: 1 << 24], 0.995))
    return s if s > 0 else 1.0


def gradient_scale_device(values: torch.Tensor, out: Optional[torch.Tensor] = None,
                          workspace: Optional[torch.Tensor] = None) -> torch.Tensor:
    """The gradient scale (steering.py:206-211) as a one-element float64 device
    tensor, computed without a host round trip (hdr_gradient_scale: numpy's
    linear 99.5th percentile of |finite values|, 1.0 if none or 0)."""
    v = values.contiguous().float().reshape(-1)
    dev = v.device
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=dev)
    if workspace is None:
        nb = ctypes.c_size_t()
        N.check(N.lib().hdr_gradient_scale_workspace_bytes(ctypes.byref(nb)),
                "hdr_gradient_scale_workspace_bytes")
        workspace = torch.empty(int(nb.value), dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream(dev)
    N.check(N.lib().hdr_gradient_scale(v.data_ptr(), v.numel(), 0.995, out.data_ptr(),
                                       workspace.data_ptr(), workspace.numel(), st.cuda_stream),
            "hdr_gradient_scale")
    return out


def compute_steering_field(grads, params: AdaptiveParams, gradient_scale=1.0,
                           out: Optional[SteeringField] = None) -> SteeringField:
    """Steering field for every output pixel (hdr_steering_field); the scale
    may be a float or a one-element device tensor (no host round trip)."""
    gx, gy = (g.contiguous().float() for g in grads)
    h, w = gx.shape
    if out is None:
        out = SteeringField(*(torch.empty((h, w), dtype=torch.float64, device=gx.device)
                              for _ in range(3)))
    theta, sigma, gamma = out.theta, out.sigma, out.gamma
    st = torch.cuda.current_stream(gx.device)
    if isinstance(gradient_scale, torch.Tensor):
        N.check(N.lib().hdr_steering_field_devscale(
            gx.data_ptr(), gy.data_ptr(), w, h, params.gradient_window, float(params.lambda1),
            float(params.lambda2), float(params.alpha), float(params.sigma_max),
            gradient_scale.data_ptr(), theta.data_ptr(), sigma.data_ptr(), gamma.data_ptr(),
            st.cuda_stream), "hdr_steering_field_devscale")
        return out
    scale = float(gradient_scale)
    if scale <= 0 or not math.isfinite(scale):
        raise ValueError(f"gradient_scale must be positive, got {gradient_scale}")
    N.check(N.lib().hdr_steering_field(
        gx.data_ptr(), gy.data_ptr(), w, h, params.gradient_window, float(params.lambda1),
        float(params.lambda2), float(params.alpha), float(params.sigma_max), scale,
        theta.data_ptr(), sigma.data_ptr(), gamma.data_ptr(), st.cuda_stream),
        "hdr_steering_field")
    return out


class CalpaScratch:
    """Preallocated device buffers of one all-device CALPA frame (first-pass
    outputs, steering field, scale, quantile workspace): calpa_device needs
    no allocation, so it can be captured in a CUDA graph."""

    def __init__(self, rig, out_size):
        out_w, out_h = int(out_size[0]), int(out_size[1])
        dev = rig.device
        self.first = rig.allocate_outputs((out_w, out_h), want_grad=True, raw_value=True)
        self.field = SteeringField(*(torch.empty((out_h, out_w), dtype=torch.float64, device=dev)
                                     for _ in range(3)))
        self.scale = torch.empty(1, dtype=torch.float64, device=dev)
        nb = ctypes.c_size_t()
        N.check(N.lib().hdr_gradient_scale_workspace_bytes(ctypes.byref(nb)),
                "hdr_gradient_scale_workspace_bytes")
        self.qws = torch.empty(int(nb.value), dtype=torch.uint8, device=dev)


def calpa_device(rig, out_size, params: AdaptiveParams, ref_size=None, out=None,
                 scratch: Optional[CalpaScratch] = None):
    """calpa_reconstruct (steering.py:214-248, shared steering) entirely on the
    device and stream-ordered: isotropic G pass, device gradient scale,
    steering field, steered pass.  Returns the output dict (``rgb``)."""
    if not params.share_steering:
        raise ValueError("calpa_device implements the shared-steering mode")
    base = params.base
    sc = scratch if scratch is not None else CalpaScratch(rig, out_size)
    # the isotropic pass of the G channel only (steering.py:214-248 steers every
    # channel with the G field): R and B left out of the tile kernel
    rig.reconstruct(out_size, base, ref_size=ref_size, out=sc.first,
                    flags=N.HDR_FLAG_SKIP_R | N.HDR_FLAG_SKIP_B)
    g = int(ColorChannel.G)
    grads = (sc.first["grad"][g, 0], sc.first["grad"][g, 1])
    if params.gradient_scale:
        scale = params.gradient_scale
    else:
        scale = gradient_scale_device(sc.first["value"][g], out=sc.scale, workspace=sc.qws)
    fld = compute_steering_field(grads, params, scale, out=sc.field)
    return rig.reconstruct_steered(out_size, base, (fld.theta, fld.sigma, fld.gamma),
                                   ref_size=ref_size, out=out)


def calpa_reconstruct(samples, out_size, params: AdaptiveParams, ref_size=None,
                      return_field: bool = False):
    """Colour-adaptive reconstruction: isotropic G pass, steering, steered RGB
    pass (reference steering.py:214-248)."""
    rig = _device_rig(samples)
    base = params.base

    def field_for(channel):
        val, gx, gy = gradient_field(rig, out_size, base, channel, ref_size)
        scale = params.gradient_scale or auto_gradient_scale(val)
        return compute_steering_field((gx, gy), params, scale)

    if params.share_steering:
        sc = CalpaScratch(rig, out_size)
        out = calpa_device(rig, out_size, params, ref_size=ref_size, scratch=sc)
        img = HDRImage._from_device_output(to_host(out["rgb"]))
        fld = sc.field
    else:
        out_w, out_h = out_size
        planes = np.empty((out_h, out_w, 3), np.float32)
        fld = None
        for ch in ColorChannel:
            f = field_for(ch)
            o = rig.reconstruct_steered(out_size, base, (f.theta, f.sigma, f.gamma),
                                        ref_size=ref_size)
            planes[:, :, int(ch)] = to_host(o["rgb"][:, :, int(ch)])
        img = HDRImage._from_device_output(planes)
    if return_field:
        return img, fld
    return img
