"""Phase timing of the reference-signature call reconstruct_frame(frames_to_samples(...))
on host numpy frames (cfg3 by default)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1308_4908_b200 as hl  # noqa: E402
from paper_1308_4908_b200.engine import to_host  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
rig, frames = bench._host_frames(wl, seed=1)
cals = rig.calibrations()
params = bench._params(wl)
W, H = wl["size"]
for it in range(6):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    raw = hl.frames_to_samples(frames, rig.sensors, cals)
    t.append(time.perf_counter())
    dev = raw.device()
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    out = dev.reconstruct(wl["out"], params, ref_size=(W, H))
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    img = hl.HDRImage._from_device_output(to_host(out["rgb"]))
    t.append(time.perf_counter())
    dev.status(wl["out"])
    t.append(time.perf_counter())
    d = [f"{(b - a) * 1e3:.2f}" for a, b in zip(t, t[1:])]
    print("frames_to_samples / device() / reconstruct / to_host / status ms:", d,
          f"total {(t[-1] - t[0]) * 1e3:.1f}")

for it in range(4):  # the whole public call
    t0 = time.perf_counter()
    img = hl.reconstruct_frame(hl.frames_to_samples(frames, rig.sensors, cals), wl["out"], params,
                               ref_size=(W, H))
    print(f"reconstruct_frame(frames_to_samples(...)) {(time.perf_counter() - t0) * 1e3:.1f} ms")
