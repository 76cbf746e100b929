"""Diagnose one stress-fuzz steered case (tests/test_gpu_fuzz.py): the pixels
beyond 1e-4, GPU (with / without the exact path) against the oracle.
usage: steer_case_probe.py K"""
import sys
from pathlib import Path

sys.path[:0] = [str(Path(__file__).resolve().parents[1])]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1308_4908_b200 as hl  # noqa: E402
from paper_1308_4908_b200 import _native as N  # noqa: E402
from paper_1308_4908_b200 import simulate as sim  # noqa: E402
from oracle import oracle  # noqa: E402

k = int(sys.argv[1])
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
print(rig_name, "order", order, "scale", base.scale, W, H)
dev = hl.frames_to_samples(frames, list(rig.sensors), cals).device()
field = tuple(torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (th, sg, gm))
outs = {f: dev.reconstruct_steered((W, H), base, field, want_outcome=True, raw_value=True, flags=f)
        for f in (0, N.HDR_FLAG_FAST_ONLY)}
for c in range(3):
    steer = oracle.kernel_inputs(th, sg, gm, oracle.channel_scale(base, c))
    val, _, _, oc = oracle.reconstruct_channel_steered(frames, list(rig.sensors), cals, (W, H),
                                                       base, c, steer)
    ref = np.maximum(val, 0.0)
    got = outs[0]["rgb"][:, :, c].cpu().numpy()
    rel = np.abs(got - ref) / np.maximum(np.abs(ref), 10.0)
    for y, x in np.argwhere(np.nan_to_num(rel) > 1e-4):
        fo = outs[N.HDR_FLAG_FAST_ONLY]
        print(f"c{c} ({y},{x}) gpu {got[y, x]:.8g} ref {ref[y, x]:.8g} rel {rel[y, x]:.2e} "
              f"outcome gpu {int(outs[0]['outcome'][c, y, x])} ref {int(oc[y, x])} "
              f"fast-only value {float(fo['value'][c, y, x]):.8g} outcome {int(fo['outcome'][c, y, x])}")
