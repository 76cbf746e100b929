"""Scattered-sample mode (RadianceSamples / LocalPolynomialRegressor) on the GPU:
the reference's known-answer tests (pkg/tests/test_lpa.py) restated, and the
CSR kernel against the oracle on the reference's golden cases."""

import math

import numpy as np
import pytest

import paper_1308_4908_b200 as hl
from golden_cases import load, names
from oracle import oracle

pytestmark = pytest.mark.gpu


def samples(pos, vals, sig=None, channel=0):
    n = len(vals)
    return hl.RadianceSamples(np.asarray(pos, float), np.full(n, channel), np.asarray(vals, float),
                              np.ones(n) if sig is None else np.asarray(sig, float), np.zeros(n))


def window(d, H):
    det = H[0, 0] * H[1, 1] - H[0, 1] * H[1, 0]
    q = (H[1, 1] * d[0] ** 2 - 2 * H[0, 1] * d[0] * d[1] + H[0, 0] * d[1] ** 2) / det
    return math.exp(-q) / (2 * math.pi * det)


def neighbourhood(pos, vals, sig, c, r):
    d = np.asarray(pos) - np.asarray(c)
    keep = (d ** 2).sum(1) <= r * r
    return np.asarray(pos)[keep], np.asarray(vals)[keep], np.asarray(sig)[keep]


def wls(pos, vals, sig, c, order, H):
    """numpy weighted least squares (the reference's lpa.py:168-210 restated)."""
    d = pos - np.asarray(c)
    w = np.array([window(di, H) for di in d]) / sig ** 2
    Phi = np.stack([hl.basis_row(di, order) for di in d])
    A = (Phi * w[:, None]).T @ Phi
    return np.linalg.solve(A, (Phi * w[:, None]).T @ vals)


def test_order0_equals_weighted_average(cuda):
    rng = np.random.default_rng(7)
    n = 300
    pos, vals, sig = rng.uniform(0, 12, (n, 2)), rng.uniform(10, 1000, n), rng.uniform(0.5, 5, n)
    s = samples(pos, vals, sig)
    p = hl.ReconstructionParams(order=0, scale=0.7, per_channel_scale=False)
    plane, _, _ = hl.reconstruct_channel(s, (12, 12), p, hl.ColorChannel.R)
    H, r0 = np.eye(2) * 0.7, 3 * math.sqrt(0.7)
    for y in range(12):
        for x in range(12):
            P, V, S = neighbourhood(pos, vals, sig, (x, y), r0)
            if not len(V):
                assert np.isnan(plane[y, x])
                continue
            w = np.array([window(pp - (x, y), H) for pp in P]) / S ** 2
            assert plane[y, x] == pytest.approx(float((w * V).sum() / w.sum()), rel=1e-12)


def test_regressor_planes_and_gradients(cuda):
    rng = np.random.default_rng(11)
    X = rng.uniform(0, 6, (200, 2))
    reg = hl.LocalPolynomialRegressor(order=1, scale=0.8).fit(X, 2.0 + 0.5 * X[:, 0] - 0.25 * X[:, 1])
    q = np.array([[3.0, 3.0], [2.0, 4.0]])
    np.testing.assert_allclose(reg.predict(q), 2.0 + 0.5 * q[:, 0] - 0.25 * q[:, 1], rtol=1e-9)
    reg = hl.LocalPolynomialRegressor(order=1, scale=0.8).fit(X, 1.0 + 3.0 * X[:, 0] + 2.0 * X[:, 1])
    _, grad = reg.predict(np.array([[3.0, 3.0]]), return_gradients=True)
    np.testing.assert_allclose(grad, [[3.0, 2.0]], rtol=1e-9)


def test_regressor_sigma_weighting(cuda):
    reg = hl.LocalPolynomialRegressor(order=0, scale=10.0).fit(
        np.array([[0.0, 0.0], [0.1, 0.0]]), np.array([10.0, 20.0]), sigma=[1.0, 3.0])
    v = reg.predict(np.array([[0.05, 0.0]]))[0]
    assert abs(v - 10.0) < abs(v - 20.0)


def test_anisotropic_smoothing_matches_wls(cuda):
    rng = np.random.default_rng(14)
    X, y, sig = rng.uniform(0, 8, (300, 2)), rng.uniform(1, 50, 300), rng.uniform(0.5, 2, 300)
    H = np.array([[1.2, 0.3], [0.3, 0.5]])
    reg = hl.LocalPolynomialRegressor(order=1, scale=0.7, max_radius=6.0).fit(X, y, sigma=sig)
    got = reg.predict(np.array([[4.0, 4.0]]), smoothing=H)[0]
    P, V, S = neighbourhood(X, y, sig, (4.0, 4.0), 3.0 * math.sqrt(np.linalg.eigvalsh(H)[-1]))
    assert got == pytest.approx(wls(P, V, S, (4.0, 4.0), 1, H)[0], rel=1e-12)


def test_reconstruct_channel_known_answers(cuda):
    xs, ys = np.meshgrid(np.arange(14, dtype=float), np.arange(14, dtype=float))
    pos = np.column_stack([xs.ravel(), ys.ravel()])
    plane, _, _ = hl.reconstruct_channel(samples(pos, np.full(196, 42.5)), (14, 14),
                                         hl.ReconstructionParams(order=0), hl.ColorChannel.R)
    np.testing.assert_allclose(plane, 42.5, rtol=1e-12)
    vals = 5.0 + 3.0 * pos[:, 0] - 2.0 * pos[:, 1]
    plane, gx, gy = hl.reconstruct_channel(samples(pos, vals), (14, 14),
                                           hl.ReconstructionParams(order=1), hl.ColorChannel.R)
    inner = (slice(2, -2), slice(2, -2))
    np.testing.assert_allclose(plane[inner], (5.0 + 3.0 * xs - 2.0 * ys)[inner], rtol=1e-6, atol=1e-9)
    np.testing.assert_allclose(gx[inner], 3.0, rtol=1e-6)
    np.testing.assert_allclose(gy[inner], -2.0, rtol=1e-6)
    one = samples(np.array([[0.0, 0.0]]), [1.0])
    plane, _, _ = hl.reconstruct_channel(one, (30, 30), hl.ReconstructionParams(
        order=0, scale=0.7, max_support_radius=3.0), hl.ColorChannel.R)
    assert np.isnan(plane[29, 29]) and plane[0, 0] == pytest.approx(1.0)
    plane, _, _ = hl.reconstruct_channel(samples(np.array([[5.0, 5.0]]), [7.0]), (11, 11),
                                         hl.ReconstructionParams(order=1, scale=0.5,
                                                                 max_support_radius=9.0),
                                         hl.ColorChannel.R)
    assert plane[0, 0] == pytest.approx(7.0)  # radius ladder, then order fallback


def test_reflection_symmetry(cuda):
    rng = np.random.default_rng(5)
    pos, vals, sig = rng.uniform(0, 10, (200, 2)), rng.uniform(1, 100, 200), rng.uniform(0.5, 2, 200)
    p = hl.ReconstructionParams(order=1, scale=0.8, per_channel_scale=False)
    a, _, _ = hl.reconstruct_channel(samples(pos, vals, sig), (11, 11), p, hl.ColorChannel.R)
    mir = np.column_stack([10.0 - pos[:, 0], pos[:, 1]])
    b, _, _ = hl.reconstruct_channel(samples(mir, vals, sig), (11, 11), p, hl.ColorChannel.R)
    np.testing.assert_allclose(a, b[:, ::-1], rtol=1e-11, equal_nan=True)


@pytest.mark.parametrize("name", names())
def test_scattered_path_matches_oracle(cuda, name):
    frames, cfgs, cals, out_size, params, ref_size, case, arrays = load(name)
    s = hl.RadianceSamples(*oracle.frames_to_samples(frames, cfgs, cals))
    img = hl.reconstruct_frame(s, out_size, params, ref_size=ref_size)
    ref = oracle.reconstruct(frames, cfgs, cals, out_size, params, ref_size=ref_size)
    assert np.array_equal(np.isnan(img.data), np.isnan(ref["rgb"]))
    fin = np.isfinite(ref["rgb"])
    rel = np.abs(img.data[fin].astype(float) - ref["rgb"][fin]) / np.maximum(np.abs(ref["rgb"][fin]), 10)
    print(name, "max rel", rel.max(), "bit-identical fraction", (img.data[fin] == ref["rgb"][fin]).mean())
    assert rel.max() < 1e-6


def test_gpu_scattered_path_reproduces_reference_pin9_sha(cuda):
    """The CSR kernel evaluated on the reference's own samples reproduces the
    reference's pinned golden SHA-256 (pkg/tests/test_acceptance.py:60)."""
    import hashlib

    from golden_cases import manifest

    frames, cfgs, cals, out_size, params, ref_size, case, arrays = load("pin9_rotation_256x192_o1")
    s = hl.RadianceSamples(*oracle.frames_to_samples(frames, cfgs, cals))
    img = hl.reconstruct_frame(s, out_size, params)
    assert hashlib.sha256(img.data.tobytes()).hexdigest() == manifest()["pin9_sha256_reference_test"]


def test_device_materialized_samples_reproduce_reference_pin9_sha(cuda):
    """End to end on the GPU: raw frames -> hdr_sample_planes (float64
    radiometry) -> device compaction -> GPU SampleIndex -> CSR kernel gives
    the reference's pinned golden SHA-256 bit for bit."""
    import hashlib

    from golden_cases import manifest

    frames, cfgs, cals, out_size, params, ref_size, case, arrays = load("pin9_rotation_256x192_o1")
    s = hl.frames_to_samples(frames, cfgs, cals).materialize()
    assert s.on_device
    img = hl.reconstruct_frame(s, out_size, params)
    assert hashlib.sha256(img.data.tobytes()).hexdigest() == manifest()["pin9_sha256_reference_test"]


def _reference_index(pos, ch, vals, sig, channel):
    """The reference's SampleIndex (radiometry.py:208-242) restated in numpy:
    bbox cells, np.argsort(kind="stable"), CSR, packed [x, y, v, s^2]."""
    sel = np.nonzero(ch == channel)[0]
    x, y = pos[sel, 0], pos[sel, 1]
    x0, y0 = int(np.floor(x.min())), int(np.floor(y.min()))
    nx = int(np.floor(x.max())) - x0 + 1
    ny = int(np.floor(y.max())) - y0 + 1
    cell = (np.floor(y).astype(np.int64) - y0) * nx + (np.floor(x).astype(np.int64) - x0)
    order = np.argsort(cell, kind="stable")
    cs = np.zeros(nx * ny + 1, np.int64)
    np.cumsum(np.bincount(cell, minlength=nx * ny), out=cs[1:])
    packed = np.column_stack([x[order], y[order], vals[sel][order], (sig[sel] ** 2)[order]])
    return (x0, y0, nx, ny), cs, packed


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_native_index_equals_stable_argsort(cuda, seed):
    """hdr_sample_index_build (counting sort + per-cell order restore) equals
    np.argsort(kind='stable') on samples with many ties per cell, negative
    coordinates and channels interleaved at random."""
    rng = np.random.default_rng(seed)
    n = 20000
    pos = np.column_stack([rng.uniform(-7.3, 25.9, n), rng.uniform(-3.1, 11.2, n)])
    pos[::7] = np.floor(pos[::7]) + 0.25            # exact cell-interior duplicates
    pos[::11] = np.floor(pos[::11])                 # exactly on cell corners
    ch = rng.integers(0, 3, n).astype(np.uint8)
    vals, sig = rng.normal(100, 30, n), rng.uniform(0.5, 3.0, n)
    s = hl.RadianceSamples(pos, ch, vals, sig, np.zeros(n))
    for c in range(3):
        ix = s.index(c)
        (x0, y0, nx, ny), cs, packed = _reference_index(pos, ch, vals, sig, c)
        assert (ix.x0, ix.y0, ix.nx, ix.ny) == (x0, y0, nx, ny)
        assert np.array_equal(ix.cell_start.cpu().numpy(), cs)
        assert np.array_equal(ix.packed.cpu().numpy(), packed)


def test_native_materialize_keeps_sensor_ids_and_order(cuda):
    """materialize() through hdr_sample_count / hdr_compact_samples: the
    oracle's sample columns (raster order, sensor-major) and the configs'
    own (non-contiguous) sensor ids (radiometry.py:335)."""
    import dataclasses

    from paper_1308_4908_b200 import simulate as sim

    W, H = 70, 46
    rig = sim.baseline_rig("misaligned", W, H, seed=9)
    sensors = [dataclasses.replace(c, sensor_id=i) for c, i in zip(rig.sensors, (7, 2, 40))]
    frames = sim.simulate_rig(sim.hdr_chart(W, H), rig)
    cals = rig.calibrations()
    s = hl.frames_to_samples(frames, sensors, cals).materialize()
    pos, chan, val, sig, sid = oracle.frames_to_samples(frames, sensors, cals)
    assert np.array_equal(s.positions, pos) and np.array_equal(s.channels, chan)
    assert np.array_equal(s.values, val) and np.array_equal(s.sigmas, sig)
    assert np.array_equal(s.sensor_ids, sid)
    assert set(np.unique(s.sensor_ids)) == {7, 2, 40}
