"""The device camera simulator (hdr_simulate_sensor, simulate.simulate_rig_device)
against the reference's model (pkg/src/hdrfuse/simulate.py:92-212) and its
statistics tests (pkg/tests/test_simulate.py:49-172): noise-free frames
bit-identical to the numpy simulator, Poisson / normal / readout moments
within the reference's tolerances, reproducible (seed, sensor) streams."""

import dataclasses

import numpy as np
import pytest

import paper_1308_4908_b200 as hl
from paper_1308_4908_b200 import simulate as sim

pytestmark = pytest.mark.gpu


def _frames(rig, gt, cuda, seed=None):
    return [t.cpu().numpy().view(np.uint16) for t in sim.simulate_rig_device(gt, rig, cuda, seed)]


@pytest.mark.parametrize("rig_name", ["aligned", "misaligned"])
def test_noise_free_bit_identical_to_numpy_simulator(cuda, rig_name):
    W, H = 120, 84
    gt = sim.hdr_chart(W, H)
    rig = dataclasses.replace(sim.baseline_rig(rig_name, W, H, seed=3), noise_free=True)
    want = [f.data for f in sim.simulate_rig(gt, rig)]
    got = _frames(rig, gt, cuda)
    for a, b in zip(got, want):
        assert np.array_equal(a, b)


def _flat_rig(f, gain=1.0, bias=0.0, readvar=0.0, seed=0, size=(512, 400)):
    cfg = sim.kodak_sensor(0, 1.0)
    cfg = dataclasses.replace(cfg, gain=gain, exposure_time=1.0, black_level=bias,
                              saturation_level=65535, bit_depth=16)
    gt = hl.HDRImage(np.full((size[1], size[0], 3), f, np.float32))
    rig = sim.RigSpec(sensors=[cfg], noise=[sim.SensorNoise(bias, readvar, 1.0)],
                      sensor_sizes=[size], seed=seed)
    return rig, gt


@pytest.mark.parametrize("lam", [3.0, 9.5, 50.0, 800.0, 5000.0])
def test_electron_counts_follow_the_reference_distribution(cuda, lam):
    """gain 1, no readout noise: y = electrons.  Poisson below the 1000 e
    crossover (multiplication method < 10, PTRS above), rounded normal above
    (simulate.py:117-127): mean within 3 SE, variance within 3 % of lambda,
    integer counts."""
    rig, gt = _flat_rig(lam)
    y = _frames(rig, gt, cuda)[0].astype(np.float64).ravel()
    n = y.size
    assert abs(y.mean() - lam) < 3 * np.sqrt(lam / n)
    assert abs(y.var(ddof=1) / lam - 1) < 0.03
    if lam < 20:  # the Poisson pmf itself at small lambda
        from math import exp, factorial

        for k in range(0, int(3 * lam) + 1):
            p = exp(-lam) * lam ** k / factorial(k)
            assert abs((y == k).mean() - p) < 4 * np.sqrt(p * (1 - p) / n) + 1e-4


def test_expose_matches_reference_model(cuda):
    """The reference's test_expectation/variance_matches_model
    (test_simulate.py:56-74): gain 0.25, t 0.01, bias 32, Var[r] 6.5, f 8e5."""
    cfg = dataclasses.replace(sim.kodak_sensor(0, 1.0), gain=0.25, exposure_time=0.01,
                              saturation_level=65535, bit_depth=16)
    f = 8e5
    gt = hl.HDRImage(np.full((250, 400, 3), f, np.float32))
    rig = sim.RigSpec(sensors=[cfg], noise=[sim.SensorNoise(32.0, 6.5, 1.0)],
                      sensor_sizes=[(400, 250)], seed=1)
    y = _frames(rig, gt, cuda)[0].astype(np.float64).ravel()
    expected = 0.25 * 0.01 * f + 32.0
    var_model = 0.25 ** 2 * 0.01 * f + 6.5
    assert abs(y.mean() - expected) < 3 * np.sqrt(var_model / y.size)
    assert abs(y.var(ddof=1) / var_model - 1) < 0.10


def test_moments_agree_with_numpy_simulator_on_the_chart(cuda):
    """Per sensor of the cfg3 rig, the residual (noisy - noise-free) of the
    device frames has the numpy (reference-algorithm) simulator's mean and
    variance; saturated pixels are clipped alike."""
    W, H = 400, 300
    gt = sim.hdr_chart(W, H)
    rig = sim.baseline_rig("misaligned", W, H, seed=11)
    clean = [f.data.astype(np.float64) for f in
             sim.simulate_rig(gt, dataclasses.replace(rig, noise_free=True))]
    ref = [f.data.astype(np.float64) for f in sim.simulate_rig(gt, rig)]
    got = [f.astype(np.float64) for f in _frames(rig, gt, cuda)]
    for c, r, g in zip(clean, ref, got):
        unsat = c < 4000
        dr, dg = (r - c)[unsat], (g - c)[unsat]
        assert abs(dg.mean() - dr.mean()) < 4 * np.sqrt(dr.var() / dr.size) * np.sqrt(2)
        assert abs(dg.var() / dr.var() - 1) < 0.03
        assert ((g >= 4095) == (r >= 4095)).mean() > 0.99


def test_streams_reproducible_and_independent(cuda):
    W, H = 64, 48
    gt = sim.hdr_chart(W, H)
    rig = sim.baseline_rig("aligned", W, H, seed=5)
    a = _frames(rig, gt, cuda)
    b = _frames(rig, gt, cuda)
    c = _frames(rig, gt, cuda, seed=6)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    assert not np.array_equal(a[0], c[0])
    # (seed, sensor) keyed: the same scene through two sensors differs
    rig2 = dataclasses.replace(rig, sensors=[dataclasses.replace(s, exposure_scaling=1.0)
                                             for s in rig.sensors])
    d = _frames(rig2, gt, cuda)
    assert not np.array_equal(d[0], d[1])


def test_saturation_clipping(cuda):
    rig, gt = _flat_rig(1e10, size=(64, 16))
    rig = dataclasses.replace(rig, sensors=[dataclasses.replace(rig.sensors[0],
                                                                saturation_level=4095)])
    y = _frames(rig, gt, cuda)[0]
    assert (y == 4095).all()
