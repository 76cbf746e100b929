"""Known-answer tests of the ICI scale-selection rule in the CPU oracle (the
rule has no reference counterpart).  CPU only."""

import dataclasses
import math

import numpy as np
import pytest

import paper_1308_4908_b200 as hl
from paper_1308_4908_b200 import simulate as sim
from oracle import oracle


def rig_frames(W=64, H=48, seed=3, scene=None, noise_free=False, name="misaligned"):
    gt = scene if scene is not None else sim.hdr_chart(W, H)
    rig = sim.baseline_rig(name, W, H, seed=seed)
    rig = dataclasses.replace(rig, noise_free=noise_free)
    return sim.simulate_rig(gt, rig), list(rig.sensors), rig.calibrations()


@pytest.mark.parametrize("order", [0, 1, 2])
def test_gamma_zero_selects_the_base_scale(order):
    frames, cfgs, cals = rig_frames()
    fixed = oracle.reconstruct(frames, cfgs, cals, (64, 48), hl.ReconstructionParams(order=order))
    ici = oracle.reconstruct(frames, cfgs, cals, (64, 48),
                             hl.ReconstructionParams(order=order, ici_scales=4, ici_gamma=0.0))
    assert (ici["scale_idx"] == 0).mean() > 0.999
    sel0 = ici["scale_idx"] == 0
    assert np.array_equal(ici["val"][sel0], fixed["val"][sel0], equal_nan=True)


def test_gamma_infinite_selects_the_largest_valid_scale():
    frames, cfgs, cals = rig_frames()
    J, rho = 3, math.sqrt(2.0)
    ici = oracle.reconstruct(frames, cfgs, cals, (64, 48),
                             hl.ReconstructionParams(order=1, ici_scales=J, ici_gamma=1e300))
    big = oracle.reconstruct(frames, cfgs, cals, (64, 48),
                             hl.ReconstructionParams(order=1, scale=0.7 * rho ** (J - 1)))
    top = ici["scale_idx"] == J - 1
    assert top.mean() > 0.95
    base_ok = big["outcome"] == 16
    m = top & base_ok
    assert np.array_equal(ici["val"][m], big["val"][m])


def test_noise_free_smooth_scene_keeps_the_largest_scale():
    W, H = 64, 48
    x = np.linspace(0, 1, W)[None, :].repeat(H, 0)
    lum = 3e4 + 1e4 * x
    scene = hl.HDRImage(np.ascontiguousarray(np.stack([lum, lum, lum], -1), np.float32))
    frames, cfgs, cals = rig_frames(scene=scene, noise_free=True, name="aligned")
    out = oracle.reconstruct(frames, cfgs, cals, (W, H),
                             hl.ReconstructionParams(order=1, ici_scales=4, ici_gamma=1.5))
    inner = out["scale_idx"][:, 8:-8, 8:-8]
    assert (inner == 3).mean() > 0.9


def test_step_edge_selects_small_scales_at_the_edge():
    W, H = 80, 40
    x = np.arange(W)[None, :].repeat(H, 0)
    lum = np.where(x < 40, 2e4, 1.2e5).astype(np.float64)
    scene = hl.HDRImage(np.ascontiguousarray(np.stack([lum, lum, lum], -1), np.float32))
    frames, cfgs, cals = rig_frames(W, H, seed=9, scene=scene, name="aligned")
    out = oracle.reconstruct(frames, cfgs, cals, (W, H),
                             hl.ReconstructionParams(order=1, ici_scales=4, ici_gamma=1.5))
    s = out["scale_idx"][:, 6:-6, :].astype(float)
    edge = s[:, :, 38:42].mean()
    flat = np.concatenate([s[:, :, 8:28], s[:, :, 52:72]], axis=2).mean()
    assert edge < flat - 1.0, (edge, flat)


def test_invalid_base_scale_falls_back_to_the_ladder():
    W, H = 48, 40
    frames, cfgs, cals = rig_frames(W, H, seed=8, scene=sim.hdr_chart(W, H, top=4e7))
    ici = oracle.reconstruct(frames, cfgs, cals, (W, H),
                             hl.ReconstructionParams(order=2, scale=0.5, ici_scales=3))
    fixed = oracle.reconstruct(frames, cfgs, cals, (W, H),
                               hl.ReconstructionParams(order=2, scale=0.5))
    ladder = fixed["outcome"] != 32
    assert ladder.any()
    assert np.array_equal(ici["val"][ladder], fixed["val"][ladder], equal_nan=True)
    assert (ici["scale_idx"][ladder] == 0).all()
