"""Generate the ICI golden vectors from the REFERENCE's own fits -- test infrastructure.

The reference has no ICI; this script pins the repo's ICI
 to the reference's arithmetic for
everything the rule is built from.  Per output pixel, channel and scale
h_k = h_ch * ratio^k it calls the reference's own

  * ``gather(samples, q, r_k, channel)``   (lpa.py:134-165; r_k = min(3 sqrt(h_k), max_radius))
  * ``wls_fit(nb, q, order, h_k I, cond, weight_mode)``   (lpa.py:168-210)

on the reference's ``frames_to_samples`` output, so the estimate y_k and the
validity of every scale are the reference's.  Only the variance
v_k = g^T B_k g (g = A_k^{-1} e1 from the same normal matrix wls_fit builds,
B_k = sum w^2 sigma^2 phi phi^T, the sandwich form) and the Appendix-A
selection (running intersection of [y_k -/+ Gamma sqrt(v_k)], largest k with
a non-empty intersection, an invalid k > 0 ends the search, an invalid k = 0
takes the reference ladder at h_0 with index 0) are computed here in numpy.
For k = 0-invalid pixels the value is the reference's own fixed-scale
``reconstruct_frame`` output at h_0 (its ladder).

Writes tests/golden/ici_<case>.npz (raw frames, scale_idx (3, H, W) u8, rgb
(H, W, 3) f32, the smallest relative intersection margin per pixel) and
tests/golden/ici_golden.json (sensors, calibration, params).

Usage (dev container only, where /root/reference exists):
    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/gen_ici_golden.py
"""

from __future__ import annotations

import json
import math
import os
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def ici_pixel(hf, samples, q, channel, order, hs, radii, cond, weight_mode, gamma):
    """(value, index, margin) of one pixel-channel, or None if scale 0 is invalid."""
    from hdrfuse.lpa import basis_row, gather, isotropic_smoothing, wls_fit

    L = U = None
    sel = None
    margin = math.inf
    for k, (h, r) in enumerate(zip(hs, radii)):
        nb = gather(samples, q, r, channel)
        fit = None
        if len(nb.values):
            fit = wls_fit(nb, q, order, isotropic_smoothing(h), cond, weight_mode)
        if fit is None:
            if k == 0:
                return None
            break
        # the normal matrix exactly as wls_fit forms it (lpa.py:193-201)
        H = isotropic_smoothing(h)
        deltas = nb.positions - np.asarray(q, dtype=np.float64)[None, :]
        Hinv = np.linalg.inv(H)
        qq = np.einsum("ki,ij,kj->k", deltas, Hinv, deltas)
        det = H[0, 0] * H[1, 1] - H[0, 1] * H[1, 0]
        win = np.exp(-qq) / (2.0 * math.pi * det)
        denom = nb.sigmas ** 2 if weight_mode == "variance" else nb.sigmas
        w = win / denom
        Phi = np.stack([basis_row(d, order) for d in deltas])
        A = (Phi * w[:, None]).T @ Phi
        Lc = np.linalg.cholesky(A)
        e1 = np.zeros(len(A))
        e1[0] = 1.0
        g = np.linalg.solve(Lc.T, np.linalg.solve(Lc, e1))
        var_y = nb.sigmas ** 2  # Var(y) of each sample
        v = float(np.sum(w * w * var_y * (Phi @ g) ** 2))
        yk = float(fit.coefficients[0])
        sd = math.sqrt(v)
        lo, hi = yk - gamma * sd, yk + gamma * sd
        if k == 0:
            L, U = lo, hi
        else:
            L, U = max(L, lo), min(U, hi)
            margin = min(margin, abs(L - U) / max(abs(L), abs(U), 1e-300))
            if L > U:
                break
        sel = (yk, k)
    return sel[0], sel[1], margin


def run_case(hf, name, frames, configs, cals, out_size, order, scale, n_scales, ratio, gamma,
             weight_mode="variance", note=""):
    from hdrfuse.lpa import ReconstructionParams, reconstruct_frame

    samples = hf.frames_to_samples(frames, configs, cals)
    base = ReconstructionParams(order=order, scale=scale, weight_mode=weight_mode)
    fixed = reconstruct_frame(samples, out_size, base)  # the reference ladder at h_0
    W, H = out_size
    max_r = base.max_support_radius if base.max_support_radius is not None else 10 * math.sqrt(scale)
    sidx = np.zeros((3, H, W), np.uint8)
    rgb = np.empty((H, W, 3), np.float32)
    margin = np.full((3, H, W), np.inf)
    for c in range(3):
        h_ch = scale / math.sqrt(2.0) if (base.per_channel_scale and c == 1) else scale
        hs = [h_ch * ratio ** k for k in range(n_scales)]
        radii = [min(3.0 * math.sqrt(h), max_r) for h in hs]
        ch = hf.ColorChannel(c)
        for y in range(H):
            for x in range(W):
                res = ici_pixel(hf, samples, (float(x), float(y)), ch, order, hs, radii,
                                base.cond_threshold, weight_mode, gamma)
                if res is None:
                    rgb[y, x, c] = fixed.data[y, x, c]
                    sidx[c, y, x] = 0
                else:
                    val, k, m = res
                    rgb[y, x, c] = np.float32(max(val, 0.0))
                    sidx[c, y, x] = k
                    margin[c, y, x] = m
    arrays = {f"raw{k}": f.data for k, f in enumerate(frames)}
    np.savez_compressed(OUT / f"{name}.npz", **arrays, scale_idx=sidx, rgb=rgb,
                        margin=margin.astype(np.float32))
    hist = np.bincount(sidx.ravel(), minlength=n_scales).tolist()
    print(name, "index histogram", hist, "min margin", float(margin.min()))
    return {
        "note": note,
        "sensors": [{
            "sensor_id": int(c.sensor_id), "exposure_time": c.exposure_time, "gain": c.gain,
            "exposure_scaling": c.exposure_scaling, "transform": c.transform.ravel().tolist(),
            "saturation_level": int(c.saturation_level), "bit_depth": int(c.bit_depth),
            "pattern": c.pattern.value, "black_level": c.black_level, "defective": None,
        } for c in configs],
        "calibration": [{"bias": float(k.bias.data.flat[0]),
                         "readout_variance": float(k.readout_variance.data.flat[0]),
                         "nonuniformity": float(k.nonuniformity.data.flat[0])} for k in cals],
        "out_size": [W, H], "ref_size": None,
        "params": {"order": order, "scale": scale, "per_channel_scale": True,
                   "max_support_radius": None, "cond_threshold": 1e8,
                   "weight_mode": weight_mode},
        "ici": {"scales": n_scales, "ratio": ratio, "gamma": gamma},
        "index_histogram": hist,
        "min_margin": float(margin.min()),
    }


def main():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path[:0] = [str(REF / "src"), str(REF / "tests")]
    import hdrfuse as hf
    from fixtures import hdr_test_scene, kodak_noise, make_config, rotate_T, simulate_and_sample, \
        translate_T

    OUT.mkdir(parents=True, exist_ok=True)
    cases = {}

    def rig(W, H, seed, pattern=None):
        kw = {} if pattern is None else {"pattern": pattern}
        cfgs = [make_config(0, 1.0, **kw), make_config(1, 2 ** -4, translate_T(0.4, 0.45), **kw),
                make_config(2, 2 ** -8, rotate_T(0.3, W / 2, H / 2), **kw)]
        return hf.RigSpec(sensors=cfgs, noise=[kodak_noise() for _ in cfgs],
                          sensor_sizes=[(W, H)] * 3, seed=seed), cfgs

    # 1. the north-star configuration in miniature: cfg3's rig, order 2, J = 4
    W, H = 56, 40
    r, cfgs = rig(W, H, seed=12)
    frames, cals, _ = simulate_and_sample(hdr_test_scene(W, H), r)
    cases["ici_misaligned_56x40_o2_J4"] = run_case(
        hf, "ici_misaligned_56x40_o2_J4", frames, cfgs, cals, (W, H), 2, 0.7, 4, math.sqrt(2.0),
        1.5, note="cfg3 rig (translation + 0.3 deg rotation), order 2, J=4, Gamma=1.5")
    # 2. order 1, three scales, tighter Gamma
    W, H = 48, 36
    r, cfgs = rig(W, H, seed=13)
    frames, cals, _ = simulate_and_sample(hdr_test_scene(W, H), r)
    cases["ici_misaligned_48x36_o1_J3_g1"] = run_case(
        hf, "ici_misaligned_48x36_o1_J3_g1", frames, cfgs, cals, (W, H), 1, 0.7, 3,
        math.sqrt(2.0), 1.0, note="order 1, J=3, Gamma=1.0")
    # 3. sigma weights, ratio 2, Gamma 2, BGGR
    W, H = 40, 32
    r, cfgs = rig(W, H, seed=14, pattern=hf.BayerPattern.BGGR)
    frames, cals, _ = simulate_and_sample(hdr_test_scene(W, H), r)
    cases["ici_sigma_40x32_o2_J3_r2"] = run_case(
        hf, "ici_sigma_40x32_o2_J3_r2", frames, cfgs, cals, (W, H), 2, 0.7, 3, 2.0, 2.0,
        weight_mode="sigma", note="sigma weights, ratio 2, Gamma 2, BGGR")
    (OUT / "ici_golden.json").write_text(json.dumps({
        "generator": "oracle/gen_ici_golden.py (reference gather + wls_fit per scale, "
                     "Appendix-A selection in numpy)",
        "cases": cases}, indent=1))


if __name__ == "__main__":
    main()
