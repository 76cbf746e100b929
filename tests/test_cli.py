"""CLI (reconstruct / simulate / video) exit codes and outputs."""

import json
from pathlib import Path

import numpy as np
import pytest
from click.testing import CliRunner

from paper_1308_4908_b200 import cli, pnm

CFG = Path(__file__).resolve().parent.parent / "configs" / "cfg3_misaligned_ici_4mpx.json"


def _small_rig(tmp_path, w=48, h=40):
    d = json.loads(CFG.read_text())
    for s in d["sensors"]:
        s["width"], s["height"] = w, h
    p = tmp_path / "rig.json"
    p.write_text(json.dumps(d))
    return p


def test_simulate_writes_frames(tmp_path):
    rig = _small_rig(tmp_path)
    r = CliRunner().invoke(cli.main, ["simulate", "--rig", str(rig), "--out-dir",
                                      str(tmp_path / "f"), "--frames", "2"])
    assert r.exit_code == 0, r.output
    f = pnm.read_pgm16(tmp_path / "f" / "frame_000001_s2.pgm")
    assert f.data.shape == (40, 48) and f.data.max() <= 4095


def test_reconstruct_exit_codes(tmp_path):
    rig = _small_rig(tmp_path)
    CliRunner().invoke(cli.main, ["simulate", "--rig", str(rig), "--out-dir", str(tmp_path / "f")])
    frames = [str(tmp_path / "f" / f"frame_000000_s{i}.pgm") for i in range(3)]
    run = lambda *a: CliRunner().invoke(cli.main, ["reconstruct", *a])  # noqa: E731
    assert run("--rig", str(tmp_path / "missing.json"), "--out", str(tmp_path / "o.pfm"),
               *frames).exit_code == cli.EXIT_USAGE
    assert run("--rig", str(rig), "--out", str(tmp_path / "o.pfm"), *frames[:2]).exit_code == \
        cli.EXIT_SHAPE
    assert run("--rig", str(rig), "--out", str(tmp_path / "o.pfm"), *frames[:2],
               str(tmp_path / "nope.pgm")).exit_code == cli.EXIT_USAGE
    assert run("--rig", str(rig), "--out", str(tmp_path / "o.pfm"), "--scale", "-1",
               *frames).exit_code == cli.EXIT_USAGE


@pytest.mark.gpu
def test_reconstruct_end_to_end(cuda, tmp_path):
    import paper_1308_4908_b200 as hl
    from oracle import compare, oracle
    from paper_1308_4908_b200.rig import load_rig

    rig_path = _small_rig(tmp_path)
    CliRunner().invoke(cli.main, ["simulate", "--rig", str(rig_path), "--out-dir",
                                  str(tmp_path / "f")])
    frames = [str(tmp_path / "f" / f"frame_000000_s{i}.pgm") for i in range(3)]
    r = CliRunner().invoke(cli.main, ["reconstruct", "--rig", str(rig_path), "--out",
                                      str(tmp_path / "o.pfm"), *frames])
    assert r.exit_code == 0, r.output
    img = pnm.read_pfm(tmp_path / "o.pfm")
    man = json.loads((tmp_path / "o.pfm.manifest.json").read_text())
    assert man["parameters"]["ici_scales"] == 4 and len(man["frames"]) == 3
    rig = load_rig(rig_path)
    raws = [pnm.read_pgm16(f) for f in frames]
    cals = [s.calibration(48, 40) for s in rig.sensors]
    ref = oracle.reconstruct(raws, rig.configs, cals, (48, 40), rig.params())
    s = compare.summary(img.data, ref["rgb"])
    assert s["nan_map_equal"] and s["frac_over"] < 1e-3


@pytest.mark.gpu
def test_video_resumable(cuda, tmp_path):
    rig = _small_rig(tmp_path)
    CliRunner().invoke(cli.main, ["simulate", "--rig", str(rig), "--out-dir", str(tmp_path / "f"),
                                  "--frames", "3"])
    r = CliRunner().invoke(cli.main, ["video", "--rig", str(rig), "--out-dir",
                                      str(tmp_path / "o"), str(tmp_path / "f")])
    assert r.exit_code == 0, r.output
    outs = sorted(p.name for p in (tmp_path / "o").glob("frame_*.pfm"))
    assert outs == [f"frame_{k:06d}.pfm" for k in range(3)]
    first = pnm.read_pfm(tmp_path / "o" / "frame_000000.pfm").data
    single = CliRunner().invoke(cli.main, [
        "reconstruct", "--rig", str(rig), "--out", str(tmp_path / "s.pfm"),
        *[str(tmp_path / "f" / f"frame_000000_s{i}.pgm") for i in range(3)]])
    assert single.exit_code == 0
    assert np.array_equal(first, pnm.read_pfm(tmp_path / "s.pfm").data, equal_nan=True)
    (tmp_path / "o" / "frame_000001.pfm").unlink()
    r = CliRunner().invoke(cli.main, ["video", "--rig", str(rig), "--out-dir",
                                      str(tmp_path / "o"), str(tmp_path / "f")])
    assert r.exit_code == 0 and "1 frames" in r.output


def test_reconstruct_reference_argument_form(tmp_path):
    """The reference's invocation `reconstruct RIG FRAMES... -o OUT`
    (pkg/src/hdrfuse/cli.py:156-171): same exit codes as the --rig form."""
    rig = _small_rig(tmp_path)
    CliRunner().invoke(cli.main, ["simulate", "--rig", str(rig), "--out-dir", str(tmp_path / "f")])
    frames = [str(tmp_path / "f" / f"frame_000000_s{i}.pgm") for i in range(3)]
    run = lambda *a: CliRunner().invoke(cli.main, ["reconstruct", *a])  # noqa: E731
    assert run(str(tmp_path / "missing.json"), *frames, "-o",
               str(tmp_path / "o.pfm")).exit_code == cli.EXIT_USAGE
    assert run(str(rig), *frames[:2], "-o", str(tmp_path / "o.pfm")).exit_code == cli.EXIT_SHAPE
    assert run(str(rig), "-o", str(tmp_path / "o.pfm")).exit_code != 0  # no frames
    assert run(str(rig), *frames, "-o", str(tmp_path / "o.pfm"), "--threads", "2", "--scale",
               "-1").exit_code == cli.EXIT_USAGE


@pytest.mark.gpu
def test_reconstruct_reference_form_calpa_preview(cuda, tmp_path):
    """`reconstruct RIG FRAMES -o OUT --calpa --alpha --grad-window --preview`:
    the CALPA output equals calpa_reconstruct's, and the preview PNG exists."""
    import paper_1308_4908_b200 as hl
    from paper_1308_4908_b200.rig import load_rig

    rig_path = _small_rig(tmp_path)
    CliRunner().invoke(cli.main, ["simulate", "--rig", str(rig_path), "--out-dir",
                                  str(tmp_path / "f")])
    frames = [str(tmp_path / "f" / f"frame_000000_s{i}.pgm") for i in range(3)]
    r = CliRunner().invoke(cli.main, ["reconstruct", str(rig_path), *frames, "-o",
                                      str(tmp_path / "c.pfm"), "--calpa", "--alpha", "0.01",
                                      "--grad-window", "7", "--threads", "4", "--order", "1",
                                      "--ici-scales", "1", "--preview", str(tmp_path / "c.png")])
    assert r.exit_code == 0, r.output
    man = json.loads((tmp_path / "c.pfm.manifest.json").read_text())
    assert man["parameters"]["calpa"] is True and man["parameters"]["grad_window"] == 7
    assert (tmp_path / "c.png").stat().st_size > 0
    rig = load_rig(rig_path)
    raws = [pnm.read_pgm16(f) for f in frames]
    cals = [s.calibration(48, 40) for s in rig.sensors]
    ap = hl.AdaptiveParams(alpha=0.01, gradient_window=7, base=rig.params(order=1, ici_scales=1))
    want = hl.calpa_reconstruct(hl.frames_to_samples(raws, rig.configs, cals), (48, 40), ap)
    assert np.array_equal(pnm.read_pfm(tmp_path / "c.pfm").data, want.data, equal_nan=True)
