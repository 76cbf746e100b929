"""Host layer mirroring the reference API (CPU only): known answers and
validation behaviour of the reference's radiometry / params / containers /
rig schema / raster I/O, restated against this package."""

import json
import math
from pathlib import Path

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import paper_1308_4908_b200 as hl
from paper_1308_4908_b200 import pnm, rig as rigmod, simulate as sim


def cfg(**kw):
    base = dict(sensor_id=0, exposure_time=0.01, gain=0.25, exposure_scaling=1.0,
                transform=sim.identity_T(), saturation_level=4095, bit_depth=12,
                pattern=hl.BayerPattern.RGGB)
    base.update(kw)
    return hl.SensorConfig(**base)


def ucal(w=4, h=4, bias=32.0, var=6.5, a=1.0):
    return hl.NoiseCalibration.uniform(w, h, bias=bias, readout_variance=var, nonuniformity=a)


class TestRadiometryKnownAnswers:
    # reference pkg/tests/test_radiometry.py:36-97
    def test_radiance(self):
        assert hl.estimate_radiance(100, 0, cfg(), ucal()) == pytest.approx(27200.0, rel=1e-12)
        assert hl.estimate_radiance(32, 0, cfg(), ucal()) == 0.0
        assert hl.estimate_radiance(20, 0, cfg(), ucal()) < 0  # negative kept

    def test_variance(self):
        assert hl.estimate_variance(27200.0, 0, cfg(), ucal()) == pytest.approx(3.76e6, rel=1e-12)
        assert hl.estimate_variance(0.0, 0, cfg(), ucal()) == pytest.approx(6.5 / (0.25 * 0.01) ** 2)
        assert hl.estimate_variance(-500.0, 0, cfg(), ucal()) == hl.estimate_variance(0.0, 0, cfg(), ucal())

    def test_saturation_threshold(self):
        img = hl.CFAImage(np.array([[4095, 4094], [0, 4095]], np.uint16), 12, hl.BayerPattern.RGGB)
        assert hl.saturation_mask(img, cfg()).tolist() == [[True, False], [False, True]]

    def test_invalid_configs(self):
        with pytest.raises(ValueError):
            cfg(exposure_time=0.0)
        with pytest.raises(hl.ConfigurationError):
            cfg(exposure_scaling=1.5)
        with pytest.raises(hl.ConfigurationError):
            cfg(transform=np.array([[1.0, 0, 0], [2.0, 0, 0]]))
        with pytest.raises(hl.ConfigurationError):
            cfg(saturation_level=5000)
        with pytest.raises(ValueError):
            hl.NoiseCalibration.uniform(2, 2, readout_variance=-1.0)
        with pytest.raises(ValueError):
            hl.NoiseCalibration.uniform(2, 2, nonuniformity=0.0)


class TestFramesToSamplesHandle:
    def test_count_and_shape_mismatch(self):
        f = hl.CFAImage(np.zeros((4, 6), np.uint16), 12, hl.BayerPattern.RGGB)
        with pytest.raises(hl.ShapeMismatchError):
            hl.frames_to_samples([f, f], [cfg()], [ucal(6, 4)])
        with pytest.raises(hl.ShapeMismatchError):
            hl.frames_to_samples([f], [cfg()], [ucal(4, 4)])
        raw = hl.frames_to_samples([f], [cfg()], [ucal(6, 4)])
        assert len(raw) == 1 and raw.reference_size == (6, 4)

    def test_unknown_sample_containers_are_rejected(self):
        with pytest.raises(TypeError):
            hl.reconstruct_frame(object(), (4, 4), hl.ReconstructionParams())

    def test_radiance_samples_validation(self):
        with pytest.raises(ValueError):
            hl.RadianceSamples([[0, 0]], [0], [1.0], [0.0], [0])
        with pytest.raises(ValueError):
            hl.RadianceSamples([[np.nan, 0]], [0], [1.0], [1.0], [0])
        s = hl.RadianceSamples.concatenate([hl.RadianceSamples.empty(),
                                            hl.RadianceSamples([[1, 2]], [1], [3.0], [0.5], [4])])
        assert len(s) == 1 and s[0].position == (1.0, 2.0) and s[0].channel == hl.ColorChannel.G

    def test_regressor_validation(self):
        reg = hl.LocalPolynomialRegressor()
        with pytest.raises(RuntimeError):
            reg.predict(np.zeros((1, 2)))
        with pytest.raises(ValueError):
            reg.fit(np.zeros((3, 2)), np.zeros(4))
        from sklearn.base import clone
        r2 = clone(hl.LocalPolynomialRegressor(order=2, scale=0.3, cond_threshold=1e6))
        assert r2.get_params()["order"] == 2 and r2.get_params()["scale"] == 0.3


class TestParams:
    def test_validation(self):
        for kw in (dict(order=3), dict(scale=0.0), dict(scale=4.0, max_support_radius=1.0),
                   dict(weight_mode="quartic"), dict(ici_scales=0), dict(ici_scales=9),
                   dict(ici_scales=2, ici_ratio=1.0), dict(ici_gamma=-1.0)):
            with pytest.raises(ValueError):
                hl.ReconstructionParams(**kw)

    def test_channel_scale_and_max_radius(self):
        p = hl.ReconstructionParams(order=1, scale=0.7)
        assert p.channel_scale(hl.ColorChannel.G) == pytest.approx(0.7 / math.sqrt(2))
        assert p.channel_scale(hl.ColorChannel.R) == 0.7
        assert hl.ReconstructionParams(per_channel_scale=False).channel_scale(1) == 0.7
        assert p.resolved_max_radius() == 10 * math.sqrt(0.7)  # from scale, not channel scale
        p4 = hl.ReconstructionParams(scale=0.7, ici_scales=4)
        assert p4.channel_scales(0) == [0.7 * math.sqrt(2) ** k for k in range(4)]

    def test_basis_row(self):
        assert hl.basis_row((2, 3), 2).tolist() == [1, 2, 3, 4, 6, 9]
        assert hl.basis_row((1, -2), 1).tolist() == [1, 1, -2]
        assert hl.basis_row((5, 5), 0).tolist() == [1]
        with pytest.raises(ValueError):
            hl.basis_row((0, 0), 3)

    def test_grid_coordinates(self):
        xs, ys = hl.grid_coordinates((4, 2), (4, 2))
        assert xs.tolist() == [0, 1, 2, 3] and ys.tolist() == [0, 1]
        xs, _ = hl.grid_coordinates((4, 2), (2, 1))
        assert xs.tolist() == [-0.25, 0.25, 0.75, 1.25]


class TestContainers:
    def test_cfa_validation(self):
        with pytest.raises(ValueError):
            hl.CFAImage(np.zeros((2, 2, 2), np.uint16), 12, hl.BayerPattern.RGGB)
        with pytest.raises(ValueError):
            hl.CFAImage(np.full((2, 2), 5000, np.uint16), 12, hl.BayerPattern.RGGB)
        with pytest.raises(ValueError):
            hl.CFAImage(np.zeros((2, 2), np.float32), 12, hl.BayerPattern.RGGB)

    def test_hdr_validation(self):
        hl.HDRImage(np.full((2, 2, 3), np.nan, np.float32))
        with pytest.raises(ValueError):
            hl.HDRImage(np.full((2, 2, 3), -1.0, np.float32))
        with pytest.raises(ValueError):
            hl.HDRImage(np.zeros((2, 2), np.float32))


@settings(max_examples=40, deadline=None)
@given(st.sampled_from(list(hl.BayerPattern)), st.integers(1, 17), st.integers(1, 17))
def test_channel_map_periodicity(pattern, w, h):
    cmap = hl.channel_map(pattern, w, h)
    for y in range(h):
        for x in range(w):
            assert cmap[y, x] == int(pattern.channel_at(x, y))
    masks = hl.channel_masks(pattern, w, h)
    assert (sum(m.astype(int) for m in masks.values()) == 1).all()


@settings(max_examples=25, deadline=None)
@given(w=st.integers(1, 9), h=st.integers(1, 9), depth=st.integers(9, 16), rnd=st.randoms())
def test_pgm16_round_trip(tmp_path_factory, w, h, depth, rnd):
    d = tmp_path_factory.mktemp("pgm")
    data = np.array([[rnd.randrange(1 << depth) for _ in range(w)] for _ in range(h)], np.uint16)
    img = hl.CFAImage(data, depth, hl.BayerPattern.RGGB)
    pnm.write_pgm16(img, d / "a.pgm")
    back = pnm.read_pgm16(d / "a.pgm")
    assert np.array_equal(back.data, data)


def test_pfm_round_trip(tmp_path):
    rgb = np.random.default_rng(0).uniform(0, 1e6, (5, 7, 3)).astype(np.float32)
    rgb[1, 2, 0] = np.nan
    pnm.write_pfm(hl.HDRImage(rgb), tmp_path / "a.pfm")
    back = pnm.read_pfm(tmp_path / "a.pfm")
    assert np.array_equal(back.data, rgb, equal_nan=True)
    plane = np.random.default_rng(1).uniform(0, 2, (4, 3))
    pnm.write_pfm(hl.FloatFrame(plane), tmp_path / "b.pfm")
    assert np.allclose(pnm.read_pfm(tmp_path / "b.pfm").data, plane.astype(np.float32))
    (tmp_path / "bad.pfm").write_bytes(b"PX\n1 1\n-1\n0000")
    with pytest.raises(pnm.PnmParseError):
        pnm.read_pfm(tmp_path / "bad.pfm")


class TestRigSchema:
    def _doc(self):
        return json.loads((Path(__file__).parent.parent / "configs" / "cfg3_misaligned_ici_4mpx.json").read_text())

    def test_shipped_configs_load(self):
        for p in (Path(__file__).parent.parent / "configs").glob("*.json"):
            r = rigmod.load_rig(p)
            assert len(r.sensors) >= 3
            r.params()

    def test_unknown_keys_rejected(self, tmp_path):
        d = self._doc()
        d["sensors"][0]["exposure"] = 1
        (tmp_path / "r.json").write_text(json.dumps(d))
        with pytest.raises(rigmod.ConfigError):
            rigmod.load_rig(tmp_path / "r.json")
        d = self._doc()
        d["reconstruction"]["ordr"] = 1
        (tmp_path / "r.json").write_text(json.dumps(d))
        with pytest.raises(rigmod.ConfigError):
            rigmod.load_rig(tmp_path / "r.json")

    def test_schema_errors(self, tmp_path):
        for mutate in (lambda d: d.update(schema_version=2),
                       lambda d: d["sensors"][0].pop("gain_dv_per_e"),
                       lambda d: d["sensors"][0].update(transform=[1, 0, 0]),
                       lambda d: d["sensors"][0].update(bayer_phase="RGBG"),
                       lambda d: d["sensors"][0].update(exposure_scaling=2.0),
                       lambda d: d["sensors"][0].pop("height")):
            d = self._doc()
            mutate(d)
            (tmp_path / "r.json").write_text(json.dumps(d))
            with pytest.raises(rigmod.ConfigError):
                rigmod.load_rig(tmp_path / "r.json")

    def test_pfm_noise_entries(self, tmp_path):
        d = self._doc()
        plane = np.full((4, 6), 3.5)
        pnm.write_pfm(hl.FloatFrame(plane), tmp_path / "bias.pfm")
        d["sensors"][0]["bias"] = "bias.pfm"
        (tmp_path / "r.json").write_text(json.dumps(d))
        r = rigmod.load_rig(tmp_path / "r.json")
        assert r.sensors[0].calibration(6, 4).bias.data.tolist() == plane.tolist()
        with pytest.raises(hl.ShapeMismatchError):
            r.sensors[0].calibration(5, 4)

    @pytest.mark.skipif(not Path("/root/reference/pkg/configs").exists(),
                        reason="reference checkout only in the dev container")
    def test_reference_configs_load_unchanged(self):
        for p in sorted(Path("/root/reference/pkg/configs").glob("*.json")):
            r = rigmod.load_rig(p)
            assert r.params().order in (0, 1, 2)


def test_band_split_limits_pixels_per_call():
    from paper_1308_4908_b200.engine import MAX_BAND_PIXELS, band_split

    for out_w, r0, r1 in ((2400, 0, 1700), (16384, 0, 8192), (9000, 37, 9001), (70000000, 0, 3)):
        bands = band_split(r0, r1, out_w)
        assert bands[0][0] == r0 and bands[-1][1] == r1
        assert all(a[1] == b[0] for a, b in zip(bands, bands[1:]))
        assert all((b1 - b0) * out_w <= MAX_BAND_PIXELS or b1 - b0 == 1 for b0, b1 in bands)
    assert band_split(0, 1700, 2400) == [(0, 1700)]
