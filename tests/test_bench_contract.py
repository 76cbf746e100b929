"""bench.py's contract pieces that need no GPU: both arms print the same
config dict, and the reference arm's row bands reproduce the reference's
full-frame rows (oracle/refarm.py; skipped when the reference is not staged)."""

import math

import numpy as np
import pytest

import bench


def test_both_arms_share_the_config_dict():
    for name, wl in bench.WORKLOADS.items():
        a = bench.config_dict(name, wl, 1)
        b = bench.config_dict(name, wl, 1)
        assert a == b and a["workload"] == name and a["parallelism"] == "frame-parallel x1"
    assert bench.config_dict("cfg3", bench.WORKLOADS["cfg3"], 4)["parallelism"] == \
        "frame-parallel x4"


def test_default_workload_is_the_north_star_config():
    """The driver's plain `python bench.py` measures cfg3: order 2, ICI J=4."""
    import inspect

    assert bench.WORKLOADS["cfg3"]["order"] == 2 and bench.WORKLOADS["cfg3"]["J"] == 4
    assert 'default="cfg3"' in inspect.getsource(bench.main)


def test_reference_band_equals_full_frame_rows():
    from oracle import refarm

    hf = refarm.load()
    if hf is None:
        pytest.skip("reference not staged in oracle/_ref")
    from paper_1308_4908_b200 import simulate as sim

    W, H = 120, 72
    rig = sim.baseline_rig("misaligned", W, H, seed=3)
    frames = sim.simulate_rig(sim.hdr_chart(W, H), rig)
    cals = rig.calibrations()
    rf, rc, rk, _ = refarm.band_inputs(hf, frames, rig.sensors, cals, 0, H, H, 0)
    p = hf.ReconstructionParams(order=2, scale=0.7)
    full = hf.reconstruct_frame(hf.frames_to_samples(rf, rc, rk), (W, H), p).data
    for y0, rows in ((20, 16), (0, 10), (56, 16)):
        _, img = refarm.band_seconds(hf, frames, rig.sensors, cals, W, y0, rows, H, 2, 0.7,
                                     10 * math.sqrt(0.7) + 26)
        assert np.array_equal(img.data, full[y0:y0 + rows], equal_nan=True)
