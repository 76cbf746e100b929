"""Generate tests/golden/ from the REFERENCE implementation -- test infrastructure.

Runs only in the dev container, where the reference package is importable
read-only from /root/reference/pkg/src (its test fixtures from
/root/reference/pkg/tests).  For each case it simulates raw frames with the
reference's own simulator, runs the reference's
``frames_to_samples`` + ``reconstruct_frame`` and stores:

  tests/golden/<case>.npz   raw frames (+ calibration planes when non-uniform),
                            the reference's float32 output, its gradients
                            (float64) and sample columns
  tests/golden/golden.json  per case: sensor configs, calibration scalars,
                            reconstruction params, SHA-256 of the reference's
                            float32 output and of its sample columns

The committed fixtures are what tests/test_oracle_golden.py checks the C
oracle against (bit-exact), and what the GPU tests use as inputs.

Usage:  NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/gen_golden.py
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path[:0] = [str(REF / "src"), str(REF / "tests")]
    import hdrfuse as hf
    from fixtures import (constant_scene, fig6_rig, hdr_test_scene, kodak_noise, make_config,
                          rotate_T, rotation_rig, simulate_and_sample, translate_T)
    from hdrfuse.lpa import ReconstructionParams, reconstruct_frame

    OUT.mkdir(parents=True, exist_ok=True)
    cases = {}

    def record(name, frames, configs, cals, out_size, params, ref_size=None, note=""):
        samples = hf.frames_to_samples(frames, configs, cals)
        img, grads = reconstruct_frame(samples, out_size, params, ref_size, return_gradients=True)
        arrays = {f"raw{k}": f.data for k, f in enumerate(frames)}
        cal_json = []
        for k, cal in enumerate(cals):
            entry = {}
            for name_, attr in (("bias", "bias"), ("readout_variance", "readout_variance"),
                                ("nonuniformity", "nonuniformity")):
                plane = getattr(cal, attr).data
                if np.all(plane == plane.flat[0]):
                    entry[name_] = float(plane.flat[0])
                else:
                    arrays[f"{name_}{k}"] = plane
                    entry[name_] = f"{name_}{k}"
            cal_json.append(entry)
        if img.data.size <= 64 * 1024:  # small cases: full arrays; large ones: SHA only
            arrays["rgb"] = img.data
            arrays["grad"] = np.stack([np.stack(grads[c]) for c in hf.ColorChannel])
        np.savez_compressed(OUT / f"{name}.npz", **arrays)
        cases[name] = {
            "note": note,
            "sensors": [{
                "sensor_id": int(c.sensor_id), "exposure_time": c.exposure_time, "gain": c.gain,
                "exposure_scaling": c.exposure_scaling, "transform": c.transform.ravel().tolist(),
                "saturation_level": int(c.saturation_level), "bit_depth": int(c.bit_depth),
                "pattern": c.pattern.value, "black_level": c.black_level,
                "defective": None if c.defective is None else c.defective.tolist(),
            } for c in configs],
            "calibration": cal_json,
            "out_size": list(out_size),
            "ref_size": None if ref_size is None else list(ref_size),
            "params": {"order": params.order, "scale": params.scale,
                       "per_channel_scale": params.per_channel_scale,
                       "max_support_radius": params.max_support_radius,
                       "cond_threshold": params.cond_threshold, "weight_mode": params.weight_mode},
            "sha256_rgb": sha(img.data),
            "sha256_grad": sha(np.stack([np.stack(grads[c]) for c in hf.ColorChannel])),
            "sha256_samples": {"positions": sha(samples.positions), "values": sha(samples.values),
                               "sigmas": sha(samples.sigmas), "channels": sha(samples.channels)},
            "nan_fraction": float(np.isnan(img.data).mean()),
        }
        print(name, cases[name]["sha256_rgb"][:16], cases[name]["nan_fraction"])

    # 1. the reference's pinned golden (pkg/tests/test_acceptance.py:334-357)
    W, H = 256, 192
    x = np.linspace(0, 1, W)[None, :].repeat(H, 0)
    lum = 1e4 + 2e5 * x ** 2
    gt = hf.HDRImage(np.ascontiguousarray(np.stack([lum, 0.85 * lum, 1.1 * lum], -1), np.float32))
    rig = rotation_rig(W, H, seed=4)
    frames, cals, _ = simulate_and_sample(gt, rig)
    record("pin9_rotation_256x192_o1", frames, list(rig.sensors), cals, (W, H),
           ReconstructionParams(order=1, scale=0.7),
           note="reference test_acceptance.py:334-357 (PIN9 golden SHA-256)")

    # 2. BASELINE config 1: 256x256, 3 sensors, order 0, identity
    W = H = 256
    gt = hdr_test_scene(W, H)
    cfgs = [make_config(i, s) for i, s in enumerate([1.0, 2 ** -4, 2 ** -8])]
    rig = hf.RigSpec(sensors=cfgs, noise=[kodak_noise() for _ in cfgs],
                     sensor_sizes=[(W, H)] * 3, seed=21)
    frames, cals, _ = simulate_and_sample(gt, rig)
    record("cfg1_256_o0_identity", frames, cfgs, cals, (W, H),
           ReconstructionParams(order=0, scale=0.7), note="BASELINE configs[0]")

    # 3. order 2 on the fig6 rig (translated middle sensor), 96x64 crop of the chart
    W, H = 96, 64
    gt = hdr_test_scene(W, H)
    rig = fig6_rig(W, H, seed=11)
    frames, cals, _ = simulate_and_sample(gt, rig)
    record("fig6_96x64_o2", frames, list(rig.sensors), cals, (W, H),
           ReconstructionParams(order=2, scale=0.7), note="fig6 rig, order 2 (LAPACK condition test)")

    # 4. 2x upsampled output, misaligned rig (translation + small rotation)
    W, H = 64, 48
    gt = hdr_test_scene(W, H)
    cfgs = [make_config(0, 1.0), make_config(1, 2 ** -4, translate_T(0.4, 0.45)),
            make_config(2, 2 ** -8, rotate_T(0.3, W / 2, H / 2))]
    rig = hf.RigSpec(sensors=cfgs, noise=[kodak_noise() for _ in cfgs],
                     sensor_sizes=[(W, H)] * 3, seed=5)
    frames, cals, _ = simulate_and_sample(gt, rig)
    record("upsample2x_64x48_o2", frames, cfgs, cals, (2 * W, 2 * H),
           ReconstructionParams(order=2, scale=0.7), ref_size=(W, H),
           note="2x upsampled output grid (lpa.py:213-224), affine rig")

    # 5. sigma weights, per-pixel calibration planes, defective pixels, BGGR
    W, H = 64, 48
    gt = hdr_test_scene(W, H)
    cfgs = [make_config(0, 1.0, pattern=hf.BayerPattern.BGGR),
            make_config(1, 2 ** -4, translate_T(-0.3, 0.2), pattern=hf.BayerPattern.BGGR),
            make_config(2, 2 ** -8, pattern=hf.BayerPattern.BGGR)]
    import dataclasses
    cfgs[0] = dataclasses.replace(cfgs[0], defective=np.array([7, 300, 1234, 2000]))
    rig = hf.RigSpec(sensors=cfgs, noise=[kodak_noise() for _ in cfgs],
                     sensor_sizes=[(W, H)] * 3, seed=6)
    frames, cals, _ = simulate_and_sample(gt, rig)
    rng = np.random.default_rng(3)
    cals = [hf.NoiseCalibration(
        bias=hf.FloatFrame(c.bias.data + rng.uniform(-1, 1, c.shape)),
        readout_variance=hf.FloatFrame(c.readout_variance.data * rng.uniform(0.8, 1.2, c.shape)),
        nonuniformity=hf.FloatFrame(rng.uniform(0.95, 1.05, c.shape)), gain_estimate=0.27)
        for c in cals]
    record("sigma_planes_defects_bggr_o1", frames, cfgs, cals, (W, H),
           ReconstructionParams(order=1, scale=0.8, weight_mode="sigma"),
           note="sigma weight mode, PRNU/bias planes, defective list, BGGR")

    # 6. sparse/saturated: radius ladder, order fallback and NaN
    W, H = 48, 40
    gt = hdr_test_scene(W, H, top=4e7)
    cfgs = [make_config(i, s) for i, s in enumerate([1.0, 2 ** -4, 2 ** -8])]
    rig = hf.RigSpec(sensors=cfgs, noise=[kodak_noise() for _ in cfgs],
                     sensor_sizes=[(W, H)] * 3, seed=8)
    frames, cals, _ = simulate_and_sample(gt, rig)
    record("ladder_48x40_o2", frames, cfgs, cals, (W, H),
           ReconstructionParams(order=2, scale=0.5),
           note="saturated scene: radius ladder, order fallback, NaN pixels")

    # 7. CALPA (structure-adaptive second pass): fig6 rig, 96x64, order 1, alpha 0.005
    from hdrfuse.steering import AdaptiveParams, calpa_reconstruct
    W, H = 96, 64
    gt = hdr_test_scene(W, H)
    rig = fig6_rig(W, H, seed=11)
    frames, cals, _ = simulate_and_sample(gt, rig)
    samples = hf.frames_to_samples(frames, list(rig.sensors), cals)
    ap = AdaptiveParams(alpha=0.005, base=ReconstructionParams(order=1, scale=0.7))
    img, fld = calpa_reconstruct(samples, (W, H), ap, return_field=True)
    np.savez_compressed(OUT / "calpa_fig6_96x64_o1.npz",
                        **{f"raw{k}": f.data for k, f in enumerate(frames)}, rgb=img.data,
                        theta=fld.theta, sigma=fld.sigma, gamma=fld.gamma)
    calpa_case = {
        "note": "calpa_reconstruct (steering.py:214-248), fig6 rig",
        "sensors": [{
            "sensor_id": int(c.sensor_id), "exposure_time": c.exposure_time, "gain": c.gain,
            "exposure_scaling": c.exposure_scaling, "transform": c.transform.ravel().tolist(),
            "saturation_level": int(c.saturation_level), "bit_depth": int(c.bit_depth),
            "pattern": c.pattern.value, "black_level": c.black_level, "defective": None,
        } for c in rig.sensors],
        "calibration": [{"bias": float(c.bias.data.flat[0]),
                         "readout_variance": float(c.readout_variance.data.flat[0]),
                         "nonuniformity": float(c.nonuniformity.data.flat[0])} for c in cals],
        "out_size": [W, H], "ref_size": None,
        "params": {"order": 1, "scale": 0.7, "per_channel_scale": True,
                   "max_support_radius": None, "cond_threshold": 1e8, "weight_mode": "variance"},
        "adaptive": {"alpha": 0.005, "lambda1": 1.0, "lambda2": 0.001, "gradient_window": 9,
                     "sigma_max": 50.0, "share_steering": True, "gradient_scale": None},
        "sha256_rgb": sha(img.data), "sha256_theta": sha(fld.theta),
        "sha256_sigma": sha(fld.sigma), "sha256_gamma": sha(fld.gamma),
    }
    print("calpa_fig6_96x64_o1", calpa_case["sha256_rgb"][:16])

    (OUT / "golden.json").write_text(json.dumps({
        "calpa_cases": {"calpa_fig6_96x64_o1": calpa_case},
        "generator": "oracle/gen_golden.py (reference hdrfuse imported from /root/reference)",
        "pin9_sha256_reference_test": "ea1f273c7f4269a32d447bf53aede42b63b0c9f9ef74f9a0d044d5a75b8849af",
        "cases": cases}, indent=1))


if __name__ == "__main__":
    main()
