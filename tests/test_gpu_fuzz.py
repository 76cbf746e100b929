"""Randomised parity sweep of the CUDA path against the oracle at the
north-star bar (every pixel within 1e-4 relative, identical NaN maps, ladder
outcomes and ICI indices): rig kind, sensor count, Bayer pattern, frame size
(odd sizes included), order, ICI, weight mode, scale and output grid drawn
per case from a seeded generator."""

import dataclasses

import numpy as np
import pytest

import paper_1308_4908_b200 as hl
from paper_1308_4908_b200 import simulate as sim
from oracle import compare, oracle

pytestmark = pytest.mark.gpu

PATTERNS = [hl.BayerPattern.RGGB, hl.BayerPattern.BGGR, hl.BayerPattern.GRBG,
            hl.BayerPattern.GBRG]


def _draw(k):
    rng = np.random.default_rng(1000 + k)
    W, H = int(rng.integers(40, 120)), int(rng.integers(30, 90))
    rig_name = ["aligned", "misaligned"][int(rng.integers(0, 2))]
    n_sensors = int(rng.integers(2, 5))
    order = int(rng.integers(0, 3))
    J = int(rng.choice([1, 1, 3, 4]))
    mode = ["variance", "sigma"][int(rng.integers(0, 4) == 0)]
    scale = float(rng.choice([0.5, 0.7, 1.0]))
    up = int(rng.integers(0, 4) == 0)
    pat = PATTERNS[int(rng.integers(0, 4))]
    return dict(W=W, H=H, rig=rig_name, n=n_sensors, order=order, J=J, mode=mode, scale=scale,
                up=up, pat=pat, seed=int(rng.integers(0, 1 << 16)))


@pytest.mark.parametrize("k", range(64))
def test_random_configuration_parity(cuda, k):
    d = _draw(k)
    gt = sim.hdr_chart(d["W"], d["H"])
    rig = sim.baseline_rig(d["rig"], d["W"], d["H"], seed=d["seed"], n_sensors=d["n"])
    rig = dataclasses.replace(rig, sensors=[dataclasses.replace(s, pattern=d["pat"])
                                            for s in rig.sensors])
    frames = sim.simulate_rig(gt, rig)
    cals = rig.calibrations()
    p = hl.ReconstructionParams(order=d["order"], scale=d["scale"], ici_scales=d["J"],
                                weight_mode=d["mode"])
    out_size = (d["W"] * (1 + d["up"]), d["H"] * (1 + d["up"]))
    ref_size = (d["W"], d["H"])
    dev = hl.frames_to_samples(frames, list(rig.sensors), cals).device()
    out = dev.reconstruct(out_size, p, ref_size=ref_size, want_scale_idx=True, want_outcome=True)
    got = {kk: v.cpu().numpy() for kk, v in out.items()}
    ref = oracle.reconstruct(frames, list(rig.sensors), cals, out_size, p, ref_size=ref_size)
    s = compare.summary(got["rgb"], ref["rgb"])
    print(d, s)
    assert s["nan_map_equal"], s
    assert s["frac_over"] == 0 and s["max"] <= 1e-4, s
    assert int((got["outcome"] != ref["outcome"]).sum()) == 0
    assert int((got["scale_idx"] != ref["scale_idx"]).sum()) == 0


@pytest.mark.parametrize("k", range(12))
def test_random_steered_pass_parity(cuda, k):
    """CALPA's steered pass (fast path + exact slow path) on random rigs and
    random steering fields, against the oracle's two-phase evaluation on the
    same field."""
    import torch

    rng = np.random.default_rng(5000 + k)
    W, H = int(rng.integers(40, 100)), int(rng.integers(30, 80))
    rig_name = ["aligned", "misaligned"][k % 2]
    order = int(rng.integers(0, 3))
    gt = sim.hdr_chart(W, H)
    rig = sim.baseline_rig(rig_name, W, H, seed=int(rng.integers(0, 1 << 16)))
    frames = sim.simulate_rig(gt, rig)
    cals = rig.calibrations()
    base = hl.ReconstructionParams(order=order, scale=float(rng.choice([0.5, 0.7])))
    th = rng.uniform(-np.pi, np.pi, (H, W))
    sg = np.exp(rng.uniform(0.0, np.log(float(rng.choice([2.0, 6.0, 20.0]))), (H, W)))
    gm = rng.uniform(0.3, 1.5, (H, W))
    dev = hl.frames_to_samples(frames, list(rig.sensors), cals).device()
    field = tuple(torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (th, sg, gm))
    out = dev.reconstruct_steered((W, H), base, field, want_outcome=True)
    rgb = out["rgb"].cpu().numpy()
    for c in range(3):
        steer = oracle.kernel_inputs(th, sg, gm, oracle.channel_scale(base, c))
        val, _, _, oc = oracle.reconstruct_channel_steered(frames, list(rig.sensors), cals,
                                                           (W, H), base, c, steer)
        s = compare.summary(rgb[:, :, c], np.maximum(val, 0.0).astype(np.float32))
        print(k, c, s)
        assert s["nan_map_equal"], s
        assert s["frac_over"] == 0 and s["max"] <= 1e-4, s
        assert int((out["outcome"][c].cpu().numpy() != oc).sum()) == 0
