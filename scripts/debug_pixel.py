"""Locate and dump the worst pixel of a GPU-vs-oracle comparison."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1308_4908_b200 as hl  # noqa: E402
from paper_1308_4908_b200 import simulate as sim  # noqa: E402
from paper_1308_4908_b200 import _native as N  # noqa: E402
from oracle import oracle  # noqa: E402

W, H = 96, 64
rig_name, order, J, seed = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
gt = sim.hdr_chart(W, H)
rig = sim.baseline_rig(rig_name, W, H, seed=seed)
frames = sim.simulate_rig(gt, rig)
cals = rig.calibrations()
p = hl.ReconstructionParams(order=order, scale=0.7, ici_scales=J)
dev = hl.frames_to_samples(frames, rig.sensors, cals).device()
for flags in (0, N.HDR_FLAG_FAST_ONLY):
    out = dev.reconstruct((W, H), p, want_scale_idx=True, want_outcome=True, raw_value=True,
                          want_count=True, want_work=True, flags=flags)
    got = {k: v.cpu().numpy() for k, v in out.items()}
    print("flags", flags, "slow items", dev.slow_items((W, H)))
ref = oracle.reconstruct(frames, rig.sensors, cals, (W, H), p)
rel = np.abs(got["rgb"].astype(float) - ref["rgb"]) / np.maximum(np.abs(ref["rgb"]), 10)
rel[np.isnan(rel)] = 0
out = dev.reconstruct((W, H), p, want_scale_idx=True, want_outcome=True, raw_value=True,
                      want_count=True, want_work=True)
got = {k: v.cpu().numpy() for k, v in out.items()}
rel = np.abs(got["rgb"].astype(float) - ref["rgb"]) / np.maximum(np.abs(ref["rgb"]), 10)
rel[np.isnan(rel)] = 0
for idx in np.argsort(rel.ravel())[::-1][:5]:
    y, x, c = np.unravel_index(idx, rel.shape)
    print(f"pixel ({x},{y}) ch {c}: rel {rel[y, x, c]:.3g} got {got['rgb'][y, x, c]} ref {ref['rgb'][y, x, c]}"
          f" val got {got['value'][c, y, x]} ref {ref['val'][c, y, x]} outcome got {got['outcome'][c, y, x]}"
          f" ref {ref['outcome'][c, y, x]} count got {got['count'][c, y, x]} ref {ref['count'][c, y, x]}"
          f" work {got['work'][c, y, x]}")
