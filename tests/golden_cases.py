"""Load the reference-generated fixtures in tests/golden/ (see oracle/gen_golden.py)
as this package's host objects."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

import paper_1308_4908_b200 as hl

GOLDEN = Path(__file__).resolve().parent / "golden"


def manifest():
    return json.loads((GOLDEN / "golden.json").read_text())


def names():
    return sorted(manifest()["cases"])


def calpa_names():
    return sorted(manifest().get("calpa_cases", {}))


def ici_manifest():
    return json.loads((GOLDEN / "ici_golden.json").read_text())


def ici_names():
    return sorted(ici_manifest()["cases"])


def load(name):
    """(frames, configs, cals, out_size, params, ref_size, case_json, arrays)."""
    m = manifest()
    if name.startswith("ici_"):
        case = ici_manifest()["cases"][name]
    else:
        case = m["cases"][name] if name in m["cases"] else m["calpa_cases"][name]
    arrays = dict(np.load(GOLDEN / f"{name}.npz"))
    frames, configs, cals = [], [], []
    for k, s in enumerate(case["sensors"]):
        pat = hl.BayerPattern(s["pattern"])
        raw = arrays[f"raw{k}"]
        frames.append(hl.CFAImage(raw, s["bit_depth"], pat))
        configs.append(hl.SensorConfig(
            sensor_id=s["sensor_id"], exposure_time=s["exposure_time"], gain=s["gain"],
            exposure_scaling=s["exposure_scaling"],
            transform=np.array(s["transform"], dtype=np.float64).reshape(2, 3),
            saturation_level=s["saturation_level"], bit_depth=s["bit_depth"], pattern=pat,
            black_level=s["black_level"],
            defective=None if s["defective"] is None else np.array(s["defective"])))
        h, w = raw.shape
        planes = {}
        for key, v in case["calibration"][k].items():
            planes[key] = arrays[v] if isinstance(v, str) else np.full((h, w), float(v))
        cals.append(hl.NoiseCalibration(
            bias=hl.FloatFrame(planes["bias"]),
            readout_variance=hl.FloatFrame(planes["readout_variance"]),
            nonuniformity=hl.FloatFrame(planes["nonuniformity"])))
    p = case["params"]
    params = hl.ReconstructionParams(order=p["order"], scale=p["scale"],
                                     per_channel_scale=p["per_channel_scale"],
                                     max_support_radius=p["max_support_radius"],
                                     cond_threshold=p["cond_threshold"],
                                     weight_mode=p["weight_mode"],
                                     **({"ici_scales": case["ici"]["scales"],
                                         "ici_ratio": case["ici"]["ratio"],
                                         "ici_gamma": case["ici"]["gamma"]} if "ici" in case else {}))
    ref_size = tuple(case["ref_size"]) if case["ref_size"] else None
    return frames, configs, cals, tuple(case["out_size"]), params, ref_size, case, arrays
