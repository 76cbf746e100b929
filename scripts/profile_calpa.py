"""Small driver for ncu: N device CALPA frames (cfg2 frames; no timing output).
The steered pass is every second lpa_fast_kernel launch."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1308_4908_b200 import simulate as sim  # noqa: E402
from paper_1308_4908_b200.engine import DeviceRig  # noqa: E402
from paper_1308_4908_b200.steering import CalpaScratch, calpa_device  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
wl = bench.WORKLOADS["calpa"]
dev = torch.device("cuda", 0)
W, H = wl["size"]
rs = sim.baseline_rig(wl["rig"], W, H, seed=0)
frames = sim.simulate_rig_device(sim.hdr_chart(W, H), rs, dev, seed=1)
rig = DeviceRig.from_device(frames, rs.sensors, rs.calibrations())
sc = CalpaScratch(rig, wl["out"])
ap = bench._calpa_params()
for i in range(steps):
    calpa_device(rig, wl["out"], ap, scratch=sc)
torch.cuda.synchronize()
print("done")
