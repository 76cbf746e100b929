"""Small driver for ncu: N reconstructions of one workload (no timing output)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1308_4908_b200 import simulate as sim  # noqa: E402
from paper_1308_4908_b200.engine import DeviceRig  # noqa: E402

wl_name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
wl = bench.WORKLOADS[wl_name]
dev = torch.device("cuda", 0)
W, H = wl["size"]
gt = sim.hdr_chart(W, H)
rs = sim.baseline_rig(wl["rig"], W, H, seed=0, n_sensors=wl.get("sensors", 3))
frames = sim.simulate_rig_device(gt, rs, dev, seed=1)
rig = DeviceRig.from_device(frames, rs.sensors, rs.calibrations())
out = rig.allocate_outputs(wl["out"])
p = bench._params(wl)
for i in range(steps):
    rig.reconstruct(wl["out"], p, ref_size=(W, H), out=out)
torch.cuda.synchronize()
print("done", rig.slow_items(wl["out"]))
