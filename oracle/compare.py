"""Parity metrics between the CUDA path and the oracle -- TEST INFRASTRUCTURE.

Radiance tolerance (north star: "within 1e-4 relative error (fp32)"):
    |gpu - ref| <= 1e-4 * max(|ref|, FLOOR)
with FLOOR = 10 e/s (the charts span 2e3..9e5 e/s; the floor only matters for
pixels clamped to ~0).  NaN maps must be identical.
"""

from __future__ import annotations

import numpy as np

FLOOR = 10.0
REL_TOL = 1e-4


def rel_err(gpu, ref, floor=FLOOR):
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    both = np.isfinite(gpu) & np.isfinite(ref)
    err = np.zeros(ref.shape)
    err[both] = np.abs(gpu[both] - ref[both]) / np.maximum(np.abs(ref[both]), floor)
    return err, both


def summary(gpu, ref, floor=FLOOR):
    """dict: nan_map_equal, n, frac_over (>1e-4), max, p99, p999."""
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    nan_eq = bool(np.array_equal(np.isnan(gpu), np.isnan(ref)))
    err, both = rel_err(gpu, ref, floor)
    e = err[both]
    if e.size == 0:
        return {"nan_map_equal": nan_eq, "n": 0, "frac_over": 0.0, "max": 0.0,
                "p99": 0.0, "p999": 0.0}
    return {
        "nan_map_equal": nan_eq,
        "n": int(e.size),
        "frac_over": float((e > REL_TOL).mean()),
        "max": float(e.max()),
        "p99": float(np.quantile(e, 0.99)),
        "p999": float(np.quantile(e, 0.999)),
    }


def grad_summary(gpu, ref, val_ref, floor=FLOOR):
    """Gradient parity: |gpu - ref| <= 1e-4 * max(|ref|, |value|, FLOOR) (per
    pixel; gradients in e/s per pixel, scaled against the pixel's own radiance
    where the gradient is small -- a flat region's gradient has no relative
    precision of its own).  Same dict as summary()."""
    gpu = np.asarray(gpu, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    v = np.abs(np.asarray(val_ref, dtype=np.float64))
    nan_eq = bool(np.array_equal(np.isnan(gpu), np.isnan(ref)))
    both = np.isfinite(gpu) & np.isfinite(ref) & np.isfinite(v)
    den = np.maximum(np.maximum(np.abs(ref), v), floor)
    e = (np.abs(gpu - ref) / den)[both]
    if e.size == 0:
        return {"nan_map_equal": nan_eq, "n": 0, "frac_over": 0.0, "max": 0.0,
                "p99": 0.0, "p999": 0.0}
    return {"nan_map_equal": nan_eq, "n": int(e.size), "frac_over": float((e > REL_TOL).mean()),
            "max": float(e.max()), "p99": float(np.quantile(e, 0.99)),
            "p999": float(np.quantile(e, 0.999))}
