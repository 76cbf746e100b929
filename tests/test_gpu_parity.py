"""Parity of the sm_100a path (through the C ABI) against the CPU oracle.

Gates (north star): identical NaN maps, identical
per-pixel ladder outcome (order, radius step), bit-exact ICI scale indices,
and radiance within 1e-4 relative error (floor 10 e/s) on EVERY pixel.
"""

import numpy as np
import pytest

import paper_1308_4908_b200 as hl
from paper_1308_4908_b200 import simulate as sim
from oracle import compare, oracle

pytestmark = pytest.mark.gpu


def _case(rig_name, W, H, seed, n_sensors=3, out=None, pattern=None):
    gt = sim.hdr_chart(W, H)
    rig = sim.baseline_rig(rig_name, W, H, seed=seed, n_sensors=n_sensors)
    frames = sim.simulate_rig(gt, rig)
    return frames, list(rig.sensors), rig.calibrations()


def _run(frames, configs, cals, out_size, params, ref_size=None):
    raw = hl.frames_to_samples(frames, configs, cals)
    dev = raw.device()
    out = dev.reconstruct(out_size, params, ref_size=ref_size, want_grad=True,
                          want_scale_idx=True, want_outcome=True, raw_value=True)
    got = {k: v.cpu().numpy() for k, v in out.items()}
    ref = oracle.reconstruct(frames, configs, cals, out_size, params, ref_size=ref_size)
    return got, ref, dev.slow_items(out_size)


def _check_grad(grad, ref):
    """Gradients (float64 at the API) within 1e-4 of the oracle's on every
    pixel, relative to max(|gradient|, |radiance|, 10) (compare.grad_summary)."""
    for c in range(3):
        for j, key in enumerate(("gx", "gy")):
            s = compare.grad_summary(grad[c, j], ref[key][c], ref["val"][c])
            print("grad", c, key, s)
            assert s["nan_map_equal"], s
            assert s["frac_over"] == 0 and s["max"] <= 1e-4, s


def _check(got, ref, max_tol=1e-4, frac_tol=0.0, max_outcome_mismatch=0, max_sidx_mismatch=0):
    s = compare.summary(got["rgb"], ref["rgb"])
    print("rgb", s)
    assert s["nan_map_equal"], s
    assert s["frac_over"] <= frac_tol, s
    assert s["max"] <= max_tol, s
    mism = int((got["outcome"] != ref["outcome"]).sum())
    print("outcome mismatches", mism, "of", ref["outcome"].size)
    assert mism <= max_outcome_mismatch
    smis = int((got["scale_idx"] != ref["scale_idx"]).sum())
    print("scale-index mismatches", smis)
    assert smis <= max_sidx_mismatch
    if "grad" in got and max_tol <= 1e-4:
        _check_grad(got["grad"], ref)
    return s


@pytest.mark.parametrize("order", [0, 1, 2])
def test_aligned_fixed_scale(cuda, order):
    frames, cfgs, cals = _case("aligned", 160, 112, seed=1)
    p = hl.ReconstructionParams(order=order, scale=0.7)
    got, ref, slow = _run(frames, cfgs, cals, (160, 112), p)
    print("slow items", slow)
    _check(got, ref)


@pytest.mark.parametrize("order", [1, 2])
def test_misaligned_fixed_scale(cuda, order):
    frames, cfgs, cals = _case("misaligned", 160, 112, seed=2)
    p = hl.ReconstructionParams(order=order, scale=0.7)
    got, ref, slow = _run(frames, cfgs, cals, (160, 112), p)
    _check(got, ref)
    # performance guard: only genuine ladder/near-threshold items take the slow path
    ladder = int((ref["outcome"] % 16 != 0).sum() + (ref["outcome"] // 16 != order).sum())
    print("slow items", slow, "reference ladder items", ladder)
    assert slow <= 2 * ladder + 0.01 * ref["outcome"].size


@pytest.mark.parametrize("order", [0, 1, 2])
def test_ici(cuda, order):
    frames, cfgs, cals = _case("misaligned", 128, 96, seed=3)
    p = hl.ReconstructionParams(order=order, scale=0.7, ici_scales=4)
    got, ref, slow = _run(frames, cfgs, cals, (128, 96), p)
    n = ref["scale_idx"].size
    _check(got, ref)
    print("slow items", slow)
    assert slow <= 0.02 * n
    assert np.bincount(ref["scale_idx"].ravel()).size > 1


def test_upsampled_output(cuda):
    frames, cfgs, cals = _case("misaligned", 96, 64, seed=4)
    p = hl.ReconstructionParams(order=2, scale=0.7, ici_scales=4)
    got, ref, _ = _run(frames, cfgs, cals, (192, 128), p, ref_size=(96, 64))
    _check(got, ref)


def test_sigma_weights_and_planes_and_defects(cuda):
    frames, cfgs, cals = _case("misaligned", 96, 80, seed=5)
    rng = np.random.default_rng(0)
    cals = [hl.NoiseCalibration(
        bias=hl.FloatFrame(c.bias.data + rng.uniform(-1, 1, c.shape)),
        readout_variance=hl.FloatFrame(c.readout_variance.data * rng.uniform(0.8, 1.2, c.shape)),
        nonuniformity=hl.FloatFrame(rng.uniform(0.95, 1.05, c.shape))) for c in cals]
    import dataclasses
    cfgs = [dataclasses.replace(cfgs[0], defective=np.array([5, 77, 1000, 2345]))] + cfgs[1:]
    for mode in ("variance", "sigma"):
        p = hl.ReconstructionParams(order=1, scale=0.7, weight_mode=mode)
        got, ref, _ = _run(frames, cfgs, cals, (96, 80), p)
        _check(got, ref)


def test_four_sensors_bggr(cuda):
    W, H = 96, 72
    gt = sim.hdr_chart(W, H)
    rig = sim.baseline_rig("misaligned", W, H, seed=6, n_sensors=4)
    import dataclasses
    sensors = [dataclasses.replace(s, pattern=hl.BayerPattern.BGGR) for s in rig.sensors]
    rig = dataclasses.replace(rig, sensors=sensors)
    frames = sim.simulate_rig(gt, rig)
    p = hl.ReconstructionParams(order=2, scale=0.7)
    got, ref, _ = _run(frames, list(rig.sensors), rig.calibrations(), (W, H), p)
    _check(got, ref)


def test_sparse_ladder_and_nan(cuda):
    """Mostly saturated frames: radius ladder, order fallback and NaN pixels."""
    W, H = 64, 48
    gt = sim.hdr_chart(W, H, top=4e7)
    rig = sim.baseline_rig("misaligned", W, H, seed=8)
    frames = sim.simulate_rig(gt, rig)
    p = hl.ReconstructionParams(order=2, scale=0.5)
    got, ref, slow = _run(frames, list(rig.sensors), rig.calibrations(), (W, H), p)
    print("slow items", slow, "ref outcomes", np.unique(ref["outcome"], return_counts=True))
    _check(got, ref)
    assert slow > 0


def test_unaligned_pitch_staging(cuda):
    """Row pitch not a multiple of 16 bytes (device-resident frames with an odd
    row length): the pre-pass reads any pitch; results must be unchanged."""
    import torch
    from paper_1308_4908_b200.engine import DeviceRig

    frames, cfgs, cals = _case("misaligned", 90, 54, seed=14)
    raws = [torch.from_numpy(f.data.view(np.int16)).to(cuda) for f in frames]  # pitch 90
    dev = DeviceRig.from_device(raws, cfgs, cals)
    p = hl.ReconstructionParams(order=2, scale=0.7, ici_scales=2)
    out = dev.reconstruct((90, 54), p, want_scale_idx=True, want_outcome=True)
    got = {k: v.cpu().numpy() for k, v in out.items()}
    ref = oracle.reconstruct(frames, cfgs, cals, (90, 54), p)
    _check(got, ref)
    aligned = hl.frames_to_samples(frames, cfgs, cals).device().reconstruct((90, 54), p)
    assert np.array_equal(aligned["rgb"].cpu().numpy(), got["rgb"], equal_nan=True)


def test_band_split_bit_identical(cuda):
    frames, cfgs, cals = _case("misaligned", 128, 96, seed=9)
    raw = hl.frames_to_samples(frames, cfgs, cals)
    dev = raw.device()
    p = hl.ReconstructionParams(order=2, scale=0.7, ici_scales=3)
    full = dev.reconstruct((128, 96), p)["rgb"].clone()
    out = dev.allocate_outputs((128, 96))
    for r0, r1 in ((0, 13), (13, 50), (50, 96)):
        dev.reconstruct((128, 96), p, rows=(r0, r1), out=out)
    assert np.array_equal(full.cpu().numpy(), out["rgb"].cpu().numpy(), equal_nan=True)


def test_saturation_masks_bit_exact(cuda):
    frames, cfgs, cals = _case("aligned", 100, 70, seed=10)
    import dataclasses
    cfgs = [dataclasses.replace(cfgs[0], defective=np.array([3, 150, 699]))] + cfgs[1:]
    masks = hl.frames_to_samples(frames, cfgs, cals).saturation_masks()
    for f, c, m in zip(frames, cfgs, masks):
        ref = f.data >= c.saturation_level
        if c.defective is not None:
            ref.ravel()[c.defective] = True
        assert np.array_equal(m, ref)


def test_radiance_planes_match_oracle_samples(cuda):
    frames, cfgs, cals = _case("misaligned", 80, 60, seed=11)
    ms = hl.frames_to_samples(frames, cfgs, cals).materialize()
    pos, ch, val, sig, sid = ms.positions, ms.channels, ms.values, ms.sigmas, ms.sensor_ids
    opos, och, oval, osig, osid = oracle.frames_to_samples(frames, cfgs, cals)
    assert np.array_equal(pos, opos) and np.array_equal(ch, och) and np.array_equal(sid, osid)
    # hdr_sample_planes: float64 radiometry in the reference's operation order
    assert np.array_equal(val, oval) and np.array_equal(sig, osig)


def test_reference_api_shapes(cuda):
    frames, cfgs, cals = _case("aligned", 64, 48, seed=12)
    raw = hl.frames_to_samples(frames, cfgs, cals)
    p = hl.ReconstructionParams(order=1)
    img, grads = hl.reconstruct_frame(raw, (64, 48), p, return_gradients=True)
    assert img.data.shape == (48, 64, 3) and img.data.dtype == np.float32
    assert set(grads) == set(hl.ColorChannel)
    v, gx, gy = hl.reconstruct_channel(raw, (64, 48), p, hl.ColorChannel.G)
    assert v.shape == gx.shape == gy.shape == (48, 64)
    ref = oracle.reconstruct(frames, cfgs, cals, (64, 48), p)
    s = compare.summary(v, ref["val"][1])
    assert s["nan_map_equal"] and s["frac_over"] == 0 and s["max"] <= 1e-4
    for g, key in ((gx, "gx"), (gy, "gy")):
        sg = compare.grad_summary(g, ref[key][1], ref["val"][1])
        print("gradient", key, sg)
        assert sg["nan_map_equal"] and sg["frac_over"] == 0 and sg["max"] <= 1e-4, sg


def test_errors_map_to_reference_exceptions(cuda):
    frames, cfgs, cals = _case("aligned", 32, 32, seed=13)
    with pytest.raises(hl.ShapeMismatchError):
        hl.frames_to_samples(frames[:2], cfgs, cals)
    bad = [hl.NoiseCalibration.uniform(16, 16)] + cals[1:]
    with pytest.raises(hl.ShapeMismatchError):
        hl.frames_to_samples(frames, cfgs, bad)
    with pytest.raises(ValueError):
        hl.ReconstructionParams(order=3)


def test_full_frame_cfg2_parity(cuda):
    """BASELINE cfg2 (the co-sited tap kernel) at its full size, every pixel
    of the 2400x1700 frame against the oracle (outcomes, NaN map, 1e-4
    radiance, gradients)."""
    W, H = 2400, 1700
    frames, cfgs, cals = _case("aligned", W, H, seed=21)
    p = hl.ReconstructionParams(order=1, scale=0.7)
    dev = hl.frames_to_samples(frames, cfgs, cals).device()
    out = dev.reconstruct((W, H), p, want_scale_idx=True, want_outcome=True, want_grad=True)
    got = {k: v.cpu().numpy() for k, v in out.items()}
    ref = oracle.reconstruct(frames, cfgs, cals, (W, H), p)
    _check(got, ref)


# first and last 16 rows (frame borders: clipped windows, ladder pixels) and a
# 64-row interior band of the full-size cfg3 / cfg4 / cfg5 frames
_BANDS = {1: [(0, 16), (832, 896), (1684, 1700)], 2: [(0, 16), (1664, 1728), (3384, 3400)]}


@pytest.mark.parametrize("rig_name,order,J,n_sensors,up", [
    ("misaligned", 2, 4, 3, 1),   # cfg3
    ("misaligned", 2, 4, 3, 2),   # cfg4: 4800x3400 output
    ("misaligned", 2, 4, 4, 1),   # cfg5: 4 sensors
])
def test_full_size_band_parity(cuda, rig_name, order, J, n_sensors, up):
    """BASELINE cfg3-cfg5 at their full size: the whole frame is reconstructed
    on the GPU (tiles, slow-path work list and escalations at production
    scale); border and interior row bands are checked against the oracle."""
    W, H = 2400, 1700
    frames, cfgs, cals = _case(rig_name, W, H, seed=21, n_sensors=n_sensors)
    p = hl.ReconstructionParams(order=order, scale=0.7, ici_scales=J)
    out_size = (W * up, H * up)
    dev = hl.frames_to_samples(frames, cfgs, cals).device()
    out = dev.reconstruct(out_size, p, ref_size=(W, H), want_scale_idx=True, want_outcome=True,
                          want_grad=True)
    for r0, r1 in _BANDS[up]:
        got = {"rgb": out["rgb"][r0:r1].cpu().numpy(),
               "outcome": out["outcome"][:, r0:r1].cpu().numpy(),
               "scale_idx": out["scale_idx"][:, r0:r1].cpu().numpy()}
        ref = oracle.reconstruct(frames, cfgs, cals, out_size, p, ref_size=(W, H), rows=(r0, r1))
        _check(got, ref)
        _check_grad(out["grad"][:, :, r0:r1].cpu().numpy(), ref)


def test_cuda_graph_replay_matches_eager(cuda):
    """DeviceRig.capture: the recorded pre-pass + fast + slow kernels replayed
    on refilled frame buffers give the eager result bit for bit."""
    import torch
    from paper_1308_4908_b200.engine import DeviceRig

    frames_a, cfgs, cals = _case("misaligned", 96, 64, seed=31)
    frames_b, _, _ = _case("misaligned", 96, 64, seed=32)
    dev_a = [torch.from_numpy(f.data.view(np.int16)).to(cuda) for f in frames_a]
    dev_b = [torch.from_numpy(f.data.view(np.int16)).to(cuda) for f in frames_b]
    p = hl.ReconstructionParams(order=2, scale=0.7, ici_scales=4)
    rig = DeviceRig.from_device([t.clone() for t in dev_a], cfgs, cals)
    cap = rig.capture((96, 64), p)
    assert cap.n_kernels >= 3
    for src in (dev_b, dev_a):
        for dst, s in zip(cap.raws, src):
            dst.copy_(s)
        got = cap.replay()["rgb"].clone()
        ref = DeviceRig.from_device(src, cfgs, cals).reconstruct((96, 64), p)["rgb"]
        torch.cuda.synchronize()
        assert torch.equal(torch.nan_to_num(got, nan=-1.0), torch.nan_to_num(ref, nan=-1.0))


def test_aligned_coincident_samples_at_corner(cuda):
    """Identical (aligned) sensors put the B samples of pixel (0, 0) at one
    position: a rank-1 window the reference rejects (radius step 1).  The fast
    path must not accept it from rounding-noise cofactors."""
    gt = sim.hdr_chart(96, 64)
    rig = sim.baseline_rig("aligned", 96, 64, seed=7)
    frames = sim.simulate_rig(gt, rig)
    p = hl.ReconstructionParams(order=1, scale=0.7)
    got, ref, _ = _run(frames, list(rig.sensors), rig.calibrations(), (96, 64), p)
    assert ref["outcome"][2, 0, 0] == 17  # order 1, radius step 1
    _check(got, ref)


@pytest.mark.parametrize("n_sensors,order,J", [(1, 1, 1), (1, 2, 3), (8, 1, 1), (8, 2, 4)])
def test_sensor_count_extremes(cuda, n_sensors, order, J):
    """One sensor (no HDR fusion) and the ABI's maximum of eight sensors
    (translations, rotations and exposures mixed)."""
    import dataclasses

    W, H = 72, 56
    gt = sim.hdr_chart(W, H)
    base = sim.baseline_rig("misaligned", W, H, seed=40, n_sensors=4)
    sensors, noise = [], []
    for i in range(n_sensors):
        src = base.sensors[i % 4]
        T = np.array(src.transform, dtype=float)
        T[:, 2] += (0.13 * (i // 4), -0.07 * (i // 4))
        sensors.append(dataclasses.replace(src, sensor_id=i, transform=T,
                                           exposure_scaling=2.0 ** -(i % 6)))
        noise.append(base.noise[i % 4])
    rig = sim.RigSpec(sensors=sensors, noise=noise, sensor_sizes=[(W, H)] * n_sensors, seed=3)
    frames = sim.simulate_rig(gt, rig)
    p = hl.ReconstructionParams(order=order, scale=0.7, ici_scales=J)
    got, ref, _ = _run(frames, sensors, rig.calibrations(), (W, H), p)
    _check(got, ref)


def test_fp16_streaming_output(cuda):
    """rgb_half (ABI v4) is the float32 output times half_scale rounded to
    IEEE half, NaN kept; the pipeline streams it."""
    import torch

    frames, cfgs, cals = _case("misaligned", 80, 56, seed=50)
    dev = hl.frames_to_samples(frames, cfgs, cals).device()
    p = hl.ReconstructionParams(order=1, scale=0.7)
    out = dev.reconstruct((80, 56), p, out=dev.allocate_outputs((80, 56), rgb_half=True),
                          half_scale=1.0 / 16)
    want = (out["rgb"] * (1.0 / 16)).half()
    got = out["rgb_half"]
    assert torch.equal(torch.isnan(got), torch.isnan(want))
    assert torch.equal(torch.nan_to_num(got, nan=-1.0), torch.nan_to_num(want, nan=-1.0))
    from paper_1308_4908_b200.pipeline import FramePipeline

    pipe = FramePipeline(cfgs, cals, [f.data.shape for f in frames], (80, 56), p,
                         output="float16")
    host = [torch.from_numpy(f.data.view(np.int16)).pin_memory() for f in frames]
    res = torch.empty((56, 80, 3), dtype=torch.float16).pin_memory()
    pipe.submit(host, res)
    pipe.synchronize()
    assert torch.equal(torch.nan_to_num(res, nan=-1.0), torch.nan_to_num(want.cpu(), nan=-1.0))


def test_output_larger_than_one_call(cuda):
    """An output of more than 2^26 pixels (the per-call work-item limit) is
    split into row bands by the engine; every band matches the oracle."""
    W, H = 96, 64
    frames, cfgs, cals = _case("misaligned", W, H, seed=60)
    out_size = (8704, 8192)  # 71.3 M pixels
    p = hl.ReconstructionParams(order=1, scale=0.7)
    dev = hl.frames_to_samples(frames, cfgs, cals).device()
    out = dev.reconstruct(out_size, p, ref_size=(W, H), want_outcome=True)
    for rows in ((0, 2), (7709, 7711), (8190, 8192)):  # the second band starts at row 7710
        got = {"rgb": out["rgb"][rows[0]:rows[1]].cpu().numpy(),
               "outcome": out["outcome"][:, rows[0]:rows[1]].cpu().numpy()}
        ref = oracle.reconstruct(frames, cfgs, cals, out_size, p, ref_size=(W, H), rows=rows)
        s = compare.summary(got["rgb"], ref["rgb"])
        assert s["nan_map_equal"] and s["frac_over"] == 0 and s["max"] <= 1e-4, s
        assert int((got["outcome"] != ref["outcome"]).sum()) == 0


@pytest.mark.parametrize("top,order,J", [(30.0, 1, 1), (30.0, 2, 4), (3e9, 1, 1), (3e9, 2, 3)])
def test_extreme_scenes(cuda, top, order, J):
    """Near-black scenes (radiance around the noise floor: many negative
    samples, where the relative-error floor matters) and blinding scenes
    (every sensor but the shortest exposure saturated; NaN where none is
    left)."""
    W, H = 80, 60
    gt = sim.hdr_chart(W, H, top=top)
    if top < 100:
        gt = hl.HDRImage(gt.data * (top / float(np.nanmax(gt.data))))
    rig = sim.baseline_rig("misaligned", W, H, seed=70)
    frames = sim.simulate_rig(gt, rig)
    p = hl.ReconstructionParams(order=order, scale=0.7, ici_scales=J)
    got, ref, _ = _run(frames, list(rig.sensors), rig.calibrations(), (W, H), p)
    _check(got, ref)


def _cosited_rig(W, H, seed, n_sensors=3, shift=(0.0, 0.0)):
    """Every sensor with the same (translation-only) transform: the co-sited
    tap kernel (one merged sample per position) applies."""
    import dataclasses

    rig = sim.baseline_rig("aligned", W, H, seed=seed, n_sensors=n_sensors)
    T = np.array([[1.0, 0.0, shift[0]], [0.0, 1.0, shift[1]]])
    sensors = [dataclasses.replace(s, transform=T) for s in rig.sensors]
    return dataclasses.replace(rig, sensors=sensors)


@pytest.mark.parametrize("order", [0, 1, 2])
def test_cosited_merge_matches_per_sensor_taps(cuda, order):
    """The merged tap kernel against the per-sensor tap kernel
    (HDR_FLAG_NO_MERGE) and the oracle: identical sample counts, outcomes and
    NaN maps, radiance within the parity bar."""
    from paper_1308_4908_b200 import _native as N

    W, H = 131, 77  # odd sizes: padded phase-plane columns and rows
    rig = _cosited_rig(W, H, seed=21)
    frames = sim.simulate_rig(sim.hdr_chart(W, H), rig)
    cfgs, cals = list(rig.sensors), rig.calibrations()
    p = hl.ReconstructionParams(order=order, scale=0.7)
    dev = hl.frames_to_samples(frames, cfgs, cals).device()
    kw = dict(want_outcome=True, want_count=True)
    a = {k: v.cpu().numpy() for k, v in dev.reconstruct((W, H), p, **kw).items()}
    b = {k: v.cpu().numpy() for k, v in
         dev.reconstruct((W, H), p, flags=N.HDR_FLAG_NO_MERGE, **kw).items()}
    assert np.array_equal(a["count"], b["count"])
    assert np.array_equal(a["outcome"], b["outcome"])
    s = compare.summary(a["rgb"], b["rgb"])
    assert s["nan_map_equal"] and s["max"] <= 2e-5, s
    got, ref, _ = _run(frames, cfgs, cals, (W, H), p)
    _check(got, ref)


@pytest.mark.parametrize("n_sensors,shift", [(2, (0.0, 0.0)), (4, (0.4, -0.45)),
                                             (3, (3.25, 1.5))])
def test_cosited_shifted_and_sensor_counts(cuda, n_sensors, shift):
    W, H = 96, 64
    rig = _cosited_rig(W, H, seed=22, n_sensors=n_sensors, shift=shift)
    frames = sim.simulate_rig(sim.hdr_chart(W, H), rig)
    p = hl.ReconstructionParams(order=1, scale=0.7)
    got, ref, _ = _run(frames, list(rig.sensors), rig.calibrations(), (W, H), p)
    _check(got, ref)


def test_cosited_sigma_weights_planes_and_defects(cuda):
    import dataclasses

    W, H = 96, 80
    rig = _cosited_rig(W, H, seed=23)
    frames = sim.simulate_rig(sim.hdr_chart(W, H), rig)
    cfgs, cals = list(rig.sensors), rig.calibrations()
    rng = np.random.default_rng(1)
    cals = [hl.NoiseCalibration(
        bias=hl.FloatFrame(c.bias.data + rng.uniform(-1, 1, c.shape)),
        readout_variance=hl.FloatFrame(c.readout_variance.data * rng.uniform(0.8, 1.2, c.shape)),
        nonuniformity=hl.FloatFrame(rng.uniform(0.95, 1.05, c.shape))) for c in cals]
    cfgs = [dataclasses.replace(cfgs[1], defective=np.array([3, 97, 1500, 4000]))
            if i == 1 else c for i, c in enumerate(cfgs)]
    for mode in ("variance", "sigma"):
        p = hl.ReconstructionParams(order=1, scale=0.7, weight_mode=mode)
        got, ref, _ = _run(frames, cfgs, cals, (W, H), p)
        _check(got, ref)


@pytest.mark.parametrize("order,J,up", [(1, 3, False), (2, 4, False), (1, 1, True), (2, 3, True)])
def test_cosited_rig_outside_the_merged_mode(cuda, order, J, up):
    """Co-sited sensors where the merged tap kernel does not apply (ICI
    scales, the 2x output grid): the row-tap / sweep kernels take over."""
    W, H = 88, 60
    rig = _cosited_rig(W, H, seed=24, shift=(0.25, -0.5))
    frames = sim.simulate_rig(sim.hdr_chart(W, H), rig)
    p = hl.ReconstructionParams(order=order, scale=0.7, ici_scales=J)
    out = (2 * W, 2 * H) if up else (W, H)
    got, ref, _ = _run(frames, list(rig.sensors), rig.calibrations(), out, p, ref_size=(W, H))
    _check(got, ref)


@pytest.mark.parametrize("n_sensors,scale,J", [(8, 2.0, 4), (4, 30.0, 1), (3, 45.0, 1)])
def test_windows_too_large_to_stage(cuda, n_sensors, scale, J):
    """Rigs whose staged tiles exceed shared memory (many sensors x large
    windows / ICI scales) run every (pixel, channel) through the exact path
    instead of failing (hdr_lpa.cu setup_staging -> all_items)."""
    import dataclasses

    W, H = 48, 40
    gt = sim.hdr_chart(W, H)
    base = sim.baseline_rig("misaligned", W, H, seed=41, n_sensors=4)
    sensors, noise = [], []
    for i in range(n_sensors):
        src = base.sensors[i % 4]
        T = np.array(src.transform, dtype=float)
        T[:, 2] += (0.11 * (i // 4), -0.05 * (i // 4))
        sensors.append(dataclasses.replace(src, sensor_id=i, transform=T,
                                           exposure_scaling=2.0 ** -(i % 6)))
        noise.append(base.noise[i % 4])
    rig = sim.RigSpec(sensors=sensors, noise=noise, sensor_sizes=[(W, H)] * n_sensors, seed=4)
    frames = sim.simulate_rig(gt, rig)
    p = hl.ReconstructionParams(order=1, scale=scale, ici_scales=J)
    got, ref, _ = _run(frames, sensors, rig.calibrations(), (W, H), p)
    _check(got, ref)
