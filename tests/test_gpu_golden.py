"""The CUDA path on the reference-generated golden cases (tests/golden):
against the reference's own stored output where present and against the
bit-exact oracle everywhere (NaN map, ladder outcome, 1e-4 radiance)."""

import numpy as np
import pytest

from golden_cases import load, names
from oracle import compare, oracle

import paper_1308_4908_b200 as hl

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", names())
def test_gpu_matches_reference_golden(cuda, name):
    frames, cfgs, cals, out_size, params, ref_size, case, arrays = load(name)
    raw = hl.frames_to_samples(frames, cfgs, cals)
    out = raw.device().reconstruct(out_size, params, ref_size=ref_size, want_outcome=True,
                                   want_grad=True)
    rgb = out["rgb"].cpu().numpy()
    ref = oracle.reconstruct(frames, cfgs, cals, out_size, params, ref_size=ref_size)
    s = compare.summary(rgb, ref["rgb"])
    print(name, s)
    assert s["nan_map_equal"]
    assert s["frac_over"] == 0 and s["max"] <= 1e-4
    assert int((out["outcome"].cpu().numpy() != ref["outcome"]).sum()) == 0
    if "rgb" in arrays:  # the reference's own float32 output
        s2 = compare.summary(rgb, arrays["rgb"])
        assert s2["nan_map_equal"] and s2["frac_over"] == 0 and s2["max"] <= 1e-4
    g = out["grad"].cpu().numpy()
    for j, key in enumerate(("gx", "gy")):  # every pixel, 1e-4 (compare.grad_summary)
        sg = compare.grad_summary(g[:, j], ref[key], ref["val"])
        assert sg["nan_map_equal"] and sg["frac_over"] == 0 and sg["max"] <= 1e-4, sg
    if "grad" in arrays:  # the reference's own float64 gradients
        for j in range(2):
            sg = compare.grad_summary(g[:, j], arrays["grad"][:, j], ref["val"])
            assert sg["nan_map_equal"] and sg["frac_over"] == 0 and sg["max"] <= 1e-4, sg


@pytest.mark.parametrize("name", __import__("golden_cases").ici_names())
def test_gpu_ici_matches_reference_fits(cuda, name):
    """ICI on the GPU against the goldens built from the reference's own
    per-scale gather + wls_fit (oracle/gen_ici_golden.py): scale indices
    bit-exact, radiance within 1e-4 on every pixel."""
    frames, cfgs, cals, out_size, params, ref_size, case, arrays = load(name)
    raw = hl.frames_to_samples(frames, cfgs, cals)
    out = raw.device().reconstruct(out_size, params, want_scale_idx=True)
    sidx = out["scale_idx"].cpu().numpy()
    mism = int((sidx != arrays["scale_idx"]).sum())
    assert mism == 0, f"{mism} scale-index mismatches"
    s = compare.summary(out["rgb"].cpu().numpy(), arrays["rgb"])
    print(name, s)
    assert s["nan_map_equal"] and s["frac_over"] == 0 and s["max"] <= 1e-4, s
