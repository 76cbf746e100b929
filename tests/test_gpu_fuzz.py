"""Randomised parity sweep of the CUDA path against the oracle at the
north-star bar (every pixel within 1e-4 relative, identical NaN maps, ladder
outcomes and ICI indices): rig kind, sensor count, Bayer pattern, frame size
(odd sizes included), order, ICI, weight mode, scale and output grid drawn
per case from a seeded generator."""

import dataclasses
import os

import numpy as np
import pytest

import paper_1308_4908_b200 as hl
from paper_1308_4908_b200 import simulate as sim
from oracle import compare, oracle

pytestmark = pytest.mark.gpu

# HDR_FUZZ_SCALE multiplies the case counts (stress campaigns on the GPU box;
# the default suite keeps 64 / 12 / 24 cases)
_SCALE = int(os.environ.get("HDR_FUZZ_SCALE", "1"))

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
    d = dict(W=W, H=H, rig=rig_name, n=n_sensors, order=order, J=J, mode=mode, scale=scale,
             up=up, pat=pat, seed=int(rng.integers(0, 1 << 16)), ratio=2 ** 0.5, gamma=1.5)
    if k >= 64:  # stress cases: other ICI ratios / widths, larger windows
        d["ratio"] = float(rng.choice([1.2, 2 ** 0.5, 2.0]))
        d["gamma"] = float(rng.choice([0.5, 1.0, 1.5, 3.0]))
        d["scale"] = float(rng.choice([0.5, 0.7, 1.0, 1.5, 2.0]))
    return d


@pytest.mark.parametrize("k", range(64 * _SCALE))
def test_random_configuration_parity(cuda, k):
    d = _draw(k)
    gt = sim.hdr_chart(d["W"], d["H"])
    rig = sim.baseline_rig(d["rig"], d["W"], d["H"], seed=d["seed"], n_sensors=d["n"])
    rig = dataclasses.replace(rig, sensors=[dataclasses.replace(s, pattern=d["pat"])
                                            for s in rig.sensors])
    frames = sim.simulate_rig(gt, rig)
    cals = rig.calibrations()
    p = hl.ReconstructionParams(order=d["order"], scale=d["scale"], ici_scales=d["J"],
                                weight_mode=d["mode"], ici_ratio=d["ratio"], ici_gamma=d["gamma"])
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


@pytest.mark.parametrize("k", range(12 * _SCALE))
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


@pytest.mark.parametrize("k", range(24 * _SCALE))
def test_random_affine_rig_parity(cuda, k):
    """General affine rigs (translations of several pixels, rotations up to
    5 deg, scales, shears), per-pixel calibration planes, defective pixels,
    mixed exposure scalings and sensor sizes, 16-bit sensors."""
    frames, sensors, cals, p, W, H, n, bit16 = affine_case(k)
    dev = hl.frames_to_samples(frames, sensors, cals).device()
    out = dev.reconstruct((W, H), p, want_scale_idx=True, want_outcome=True)
    got = {kk: v.cpu().numpy() for kk, v in out.items()}
    ref = oracle.reconstruct(frames, sensors, cals, (W, H), p)
    s = compare.summary(got["rgb"], ref["rgb"])
    print(k, n, bit16, p, s)
    assert s["nan_map_equal"], s
    assert s["frac_over"] == 0 and s["max"] <= 1e-4, s
    assert int((got["outcome"] != ref["outcome"]).sum()) == 0
    assert int((got["scale_idx"] != ref["scale_idx"]).sum()) == 0


def affine_case(k):
    """The random affine rig of case k (frames, sensors, calibrations, params,
    W, H, sensor count, 16-bit flag)."""
    rng = np.random.default_rng(9000 + k)
    W, H = int(rng.integers(48, 110)), int(rng.integers(40, 90))
    n = int(rng.integers(2, 5))
    bit16 = bool(rng.integers(0, 4) == 0)
    sensors, noise, sizes = [], [], []
    for i in range(n):
        kind = int(rng.integers(0, 4))
        if i == 0 or kind == 0:
            T = sim.translate_T(*rng.uniform(-3, 3, 2)) if i else sim.identity_T()
        elif kind == 1:
            T = sim.rotate_T(float(rng.uniform(-5, 5)), W / 2, H / 2, *rng.uniform(-1, 1, 2))
        elif kind == 2:
            s = float(rng.uniform(0.95, 1.05))
            T = np.array([[s, 0.0, float(rng.uniform(-1, 1))], [0.0, s, float(rng.uniform(-1, 1))]])
        else:
            sh = float(rng.uniform(-0.05, 0.05))
            T = np.array([[1.0, sh, float(rng.uniform(-1, 1))], [0.0, 1.0, float(rng.uniform(-1, 1))]])
        cfg = sim.kodak_sensor(i, float(2.0 ** -int(rng.integers(0, 10))), T)
        if bit16:
            cfg = dataclasses.replace(cfg, bit_depth=16, saturation_level=int(rng.integers(30000, 65536)))
        if rng.integers(0, 3) == 0:
            cfg = dataclasses.replace(cfg, defective=rng.choice(W * H, size=20, replace=False))
        sensors.append(cfg)
        noise.append(sim.kodak_noise())
        sizes.append((W, H))
    rig = sim.RigSpec(sensors=sensors, noise=noise, sensor_sizes=sizes, seed=int(rng.integers(0, 999)))
    gt = sim.hdr_chart(W, H, top=float(rng.choice([4e5, 4e6])))
    frames = sim.simulate_rig(gt, rig)
    cals = rig.calibrations()
    if rng.integers(0, 2) == 0:  # per-pixel calibration planes on one sensor
        c0 = cals[0]
        cals[0] = hl.NoiseCalibration(
            bias=hl.FloatFrame(c0.bias.data + rng.uniform(-0.5, 0.5, c0.shape)),
            readout_variance=hl.FloatFrame(c0.readout_variance.data * rng.uniform(0.9, 1.1, c0.shape)),
            nonuniformity=hl.FloatFrame(rng.uniform(0.97, 1.03, c0.shape)))
    p = hl.ReconstructionParams(order=int(rng.integers(0, 3)), scale=float(rng.choice([0.5, 0.7, 1.2])),
                                ici_scales=int(rng.choice([1, 3])))
    return frames, sensors, cals, p, W, H, n, bit16


@pytest.mark.parametrize("order", [1, 2])
def test_cosited_steered_pass_merge_ab(cuda, order):
    """CALPA's steered sweep over co-sited merged planes against the per-sensor
    sweep (HDR_FLAG_NO_MERGE) and the oracle, on one random steering field."""
    import torch
    from paper_1308_4908_b200 import _native as N

    rng = np.random.default_rng(77 + order)
    W, H = 83, 61
    rig = sim.baseline_rig("aligned", W, H, seed=11)
    frames = sim.simulate_rig(sim.hdr_chart(W, H), rig)
    cals = rig.calibrations()
    base = hl.ReconstructionParams(order=order, scale=0.7)
    th = rng.uniform(-np.pi, np.pi, (H, W))
    sg = np.exp(rng.uniform(0.0, np.log(6.0), (H, W)))
    gm = rng.uniform(0.3, 1.5, (H, W))
    dev = hl.frames_to_samples(frames, list(rig.sensors), cals).device()
    field = tuple(torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (th, sg, gm))
    a = dev.reconstruct_steered((W, H), base, field, want_outcome=True)
    b = dev.reconstruct_steered((W, H), base, field, want_outcome=True, flags=N.HDR_FLAG_NO_MERGE)
    assert torch.equal(a["outcome"], b["outcome"])
    s = compare.summary(a["rgb"].cpu().numpy(), b["rgb"].cpu().numpy())
    assert s["nan_map_equal"] and s["max"] <= 2e-5, s
    rgb = a["rgb"].cpu().numpy()
    for c in range(3):
        steer = oracle.kernel_inputs(th, sg, gm, oracle.channel_scale(base, c))
        val, _, _, oc = oracle.reconstruct_channel_steered(frames, list(rig.sensors), cals,
                                                           (W, H), base, c, steer)
        s = compare.summary(rgb[:, :, c], np.maximum(val, 0.0).astype(np.float32))
        assert s["nan_map_equal"] and s["frac_over"] == 0 and s["max"] <= 1e-4, s
        assert int((a["outcome"][c].cpu().numpy() != oc).sum()) == 0


@pytest.mark.parametrize("kind,k", [("steered", 80), ("affine", 219), ("affine", 379),
                                    ("steered", 227)])
def test_razor_edge_order1_decisions(cuda, kind, k):
    """Stress-campaign cases: order-1 condition tests where the
    reference's closed-form eigenvalue range decides on rounding noise
    (80, 219, 379: settled in the reference's own summation order,
    exact_ref.cuh), and a strongly anisotropic steered window whose fp32
    quadratic form escaped the precision bound (227: float64 q)."""
    if kind == "steered":
        test_random_steered_pass_parity(cuda, k)
    else:
        test_random_affine_rig_parity(cuda, k)
