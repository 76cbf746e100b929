"""CALPA (structure-adaptive second pass) on the GPU against the oracle (which
reproduces the reference bit-exactly: tests/test_oracle_golden.py)."""

import numpy as np
import pytest
import torch

import paper_1308_4908_b200 as hl
from golden_cases import calpa_names, load
from paper_1308_4908_b200 import simulate as sim
from oracle import compare, oracle

pytestmark = pytest.mark.gpu


def _case():
    frames, cfgs, cals, out_size, params, ref_size, case, arrays = load(calpa_names()[0])
    ap = hl.AdaptiveParams(base=params, **case["adaptive"])
    return frames, cfgs, cals, out_size, ap, arrays


@pytest.mark.parametrize("window,nan_frac", [(5, 0.0), (9, 0.02), (71, 0.02)])
def test_steering_field_windows_and_nans(cuda, window, nan_frac):
    """The tiled steering-field kernel (windows whose neighbourhood fits shared
    memory) and the per-pixel fallback (window 71) against the oracle, with
    non-finite gradients skipped as the reference skips them
    (_kernels.py:310-392); image edges inside every window."""
    import dataclasses

    rng = np.random.default_rng(window)
    h, w = 61, 83
    gx = (rng.standard_normal((h, w)) * 40).astype(np.float32)
    gy = (rng.standard_normal((h, w)) * 40 + 10).astype(np.float32)
    bad = rng.random((h, w)) < nan_frac
    gx[bad] = np.nan
    gy[rng.random((h, w)) < nan_frac / 2] = np.inf
    frames, cfgs, cals, out_size, ap, arrays = _case()
    ap = dataclasses.replace(ap, gradient_window=window)
    scale = 7.5
    th, sg, gm = oracle.steering_field(gx.astype(np.float64), gy.astype(np.float64), ap, scale)
    f = hl.compute_steering_field((torch.from_numpy(gx).cuda(), torch.from_numpy(gy).cuda()),
                                  ap, scale)
    gth, gsg, ggm = f.numpy()
    np.testing.assert_allclose(gsg, sg, rtol=1e-12)
    np.testing.assert_allclose(ggm, gm, rtol=1e-12)
    np.testing.assert_allclose(gth, th, rtol=1e-9, atol=1e-12)


def test_steering_field_kernel_matches_oracle(cuda):
    frames, cfgs, cals, out_size, ap, arrays = _case()
    o = oracle.reconstruct(frames, cfgs, cals, out_size, ap.base, channels=(1,))
    gx32, gy32 = o["gx"][1].astype(np.float32), o["gy"][1].astype(np.float32)
    scale = oracle.auto_gradient_scale(o["val"][1])
    th, sg, gm = oracle.steering_field(gx32.astype(np.float64), gy32.astype(np.float64), ap, scale)
    f = hl.compute_steering_field((torch.from_numpy(gx32).cuda(), torch.from_numpy(gy32).cuda()),
                                  ap, scale)
    gth, gsg, ggm = f.numpy()
    # same float64 formula, device vs libm exp/atan2/pow: a few ulp
    np.testing.assert_allclose(gsg, sg, rtol=1e-12)
    np.testing.assert_allclose(ggm, gm, rtol=1e-12)
    np.testing.assert_allclose(gth, th, rtol=1e-9, atol=1e-12)


def test_steered_pass_matches_oracle_on_the_same_field(cuda):
    frames, cfgs, cals, out_size, ap, arrays = _case()
    th, sg, gm = (arrays[k] for k in ("theta", "sigma", "gamma"))  # the reference's field
    rig = hl.frames_to_samples(frames, cfgs, cals).device()
    field = tuple(torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (th, sg, gm))
    out = rig.reconstruct_steered(out_size, ap.base, field, want_outcome=True)
    rgb = out["rgb"].cpu().numpy()
    for c in range(3):
        steer = oracle.kernel_inputs(th, sg, gm, oracle.channel_scale(ap.base, c))
        val, _, _, oc = oracle.reconstruct_channel_steered(frames, cfgs, cals, out_size, ap.base,
                                                           c, steer)
        ref = np.maximum(val, 0.0).astype(np.float32)
        s = compare.summary(rgb[:, :, c], ref)
        print(c, s, "outcome mismatches", int((out["outcome"][c].cpu().numpy() != oc).sum()))
        assert s["nan_map_equal"] and s["frac_over"] == 0 and s["max"] <= 1e-4
        assert int((out["outcome"][c].cpu().numpy() != oc).sum()) == 0


def test_calpa_end_to_end_matches_reference(cuda):
    frames, cfgs, cals, out_size, ap, arrays = _case()
    img, fld = hl.calpa_reconstruct(hl.frames_to_samples(frames, cfgs, cals), out_size, ap,
                                    return_field=True)
    s = compare.summary(img.data, arrays["rgb"])  # the reference's own CALPA output
    print("calpa vs reference", s)
    assert s["nan_map_equal"] and s["frac_over"] == 0 and s["max"] <= 1e-4
    th, sg, gm = fld.numpy()
    assert np.abs(sg - arrays["sigma"]).max() / 50.0 < 1e-4


def test_calpa_without_adaptation_equals_lpa(cuda):
    # reference acceptance criterion 8 (test_acceptance.py:324-327): alpha = 0 and
    # sigma_max = 1 make every window the isotropic one
    frames, cfgs, cals, out_size, ap, arrays = _case()
    raw = hl.frames_to_samples(frames, cfgs, cals)
    eq = hl.calpa_reconstruct(raw, out_size, hl.AdaptiveParams(alpha=0.0, sigma_max=1.0,
                                                               base=ap.base))
    iso = hl.reconstruct_frame(raw, out_size, ap.base)
    s = compare.summary(eq.data, iso.data)
    assert s["nan_map_equal"] and s["max"] < 1e-5


@pytest.mark.parametrize("case", ["random", "ties", "nan_inf", "all_nan", "zeros", "single"])
def test_device_gradient_scale_equals_numpy_percentile(cuda, case):
    """hdr_gradient_scale: np.percentile(|finite|, 99.5) (numpy's linear
    interpolation, steering.py:206-211) exactly, 1.0 for none / zero."""
    import torch

    from paper_1308_4908_b200.steering import gradient_scale_device

    rng = np.random.default_rng(7)
    v = {"random": rng.normal(0, 1e4, 1_000_003),
         "ties": rng.integers(-50, 50, 300_001).astype(float),
         "nan_inf": np.where(rng.random(200_000) < 0.1, np.nan, rng.normal(0, 3e5, 200_000)),
         "all_nan": np.full(1000, np.nan), "zeros": np.zeros(5000), "single": np.array([-3.5])}[case]
    v = v.astype(np.float32)
    if case == "nan_inf":
        v[::977] = np.inf
    got = float(gradient_scale_device(torch.from_numpy(v).to(cuda)).item())
    f = np.abs(v[np.isfinite(v)].astype(np.float64))
    want = float(np.percentile(f, 99.5)) if f.size else 1.0
    want = want if want > 0 else 1.0
    assert got == want, (got, want)


def test_calpa_pipeline_equals_host_api(cuda):
    """FramePipeline(calpa=...): the all-device CALPA graph per slot streams the
    same float32 frames as calpa_reconstruct."""
    import torch

    from paper_1308_4908_b200.engine import DeviceRig
    from paper_1308_4908_b200.pipeline import FramePipeline

    W, H = 96, 64
    gt = sim.hdr_chart(W, H)
    rig = sim.baseline_rig("aligned", W, H, seed=9)
    ap = hl.AdaptiveParams(base=hl.ReconstructionParams(order=1))
    sets = [[torch.from_numpy(f.data.view(np.int16)).pin_memory() for f in
             sim.simulate_rig(gt, sim.RigSpec(rig.sensors, rig.noise, rig.sensor_sizes, seed=s))]
            for s in (1, 2, 3)]
    pipe = FramePipeline(rig.sensors, rig.calibrations(), [(H, W)] * 3, (W, H), ap.base,
                         device=cuda, calpa=ap)
    outs = [torch.empty((H, W, 3), dtype=torch.float32).pin_memory() for _ in sets]
    for hs, o in zip(sets, outs):
        pipe.submit(hs, o)
    pipe.synchronize()
    for hs, o in zip(sets, outs):
        dev = DeviceRig.from_device([t.to(cuda) for t in hs], rig.sensors, rig.calibrations())
        want = hl.calpa_reconstruct(dev, (W, H), ap).data
        assert np.array_equal(o.numpy(), want, equal_nan=True)
