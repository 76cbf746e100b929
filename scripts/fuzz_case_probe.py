"""Diagnose one stress-fuzz affine case (tests/test_gpu_fuzz.py::affine_case):
the mismatching pixel-channels' values, scale indices and outcomes, GPU vs
oracle, with and without the exact path.  usage: fuzz_case_probe.py K"""
import sys
from pathlib import Path

sys.path[:0] = [str(Path(__file__).resolve().parents[1]), str(Path(__file__).resolve().parents[1] / "tests")]
import numpy as np  # noqa: E402

import paper_1308_4908_b200 as hl  # noqa: E402
from paper_1308_4908_b200 import _native as N  # noqa: E402
from oracle import oracle  # noqa: E402
from test_gpu_fuzz import affine_case  # noqa: E402

k = int(sys.argv[1])
frames, sensors, cals, p, W, H, n, bit16 = affine_case(k)
print(p, "sensors", n)
dev = hl.frames_to_samples(frames, sensors, cals).device()
ref = oracle.reconstruct(frames, sensors, cals, (W, H), p)
for flags in (0, N.HDR_FLAG_FAST_ONLY):
    out = dev.reconstruct((W, H), p, want_scale_idx=True, want_outcome=True, raw_value=True,
                          flags=flags)
    got = {kk: v.cpu().numpy() for kk, v in out.items()}
    rel = np.abs(got["rgb"] - ref["rgb"]) / np.maximum(np.abs(ref["rgb"]), 10.0)
    bad = np.argwhere(np.nan_to_num(rel, nan=0.0) > 1e-4)
    print("flags", flags, "bad", len(bad), "slow items", dev.slow_items((W, H)))
    for y, x, c in bad[:5]:
        print(f"  ({y},{x}) c{c}: gpu {got['rgb'][y, x, c]:.6g} ref {ref['rgb'][y, x, c]:.6g} "
              f"sidx gpu {got['scale_idx'][c, y, x]} ref {ref['scale_idx'][c, y, x]} "
              f"outcome gpu {got['outcome'][c, y, x]} ref {ref['outcome'][c, y, x]}")
