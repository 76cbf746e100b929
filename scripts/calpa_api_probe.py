import sys, time
sys.path.insert(0, "/root/repo")
import torch, numpy as np
import bench
import paper_1308_4908_b200 as hl
from paper_1308_4908_b200 import simulate as sim
from paper_1308_4908_b200.engine import DeviceRig, to_host
from paper_1308_4908_b200.steering import CalpaScratch, calpa_device
wl = bench.WORKLOADS["calpa"]; W, H = wl["size"]
rs = sim.baseline_rig("aligned", W, H, seed=0)
fr = sim.simulate_rig_device(sim.hdr_chart(W, H), rs, "cuda:0", seed=1)
rig = DeviceRig.from_device(fr, rs.sensors, rs.calibrations())
ap = hl.AdaptiveParams(base=hl.ReconstructionParams(order=1))
for i in range(8):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    sc = CalpaScratch(rig, (W, H)); torch.cuda.synchronize(); t1 = time.perf_counter()
    out = calpa_device(rig, (W, H), ap, scratch=sc); torch.cuda.synchronize(); t2 = time.perf_counter()
    img = to_host(out["rgb"]); t3 = time.perf_counter()
    print(f"scratch {1e3*(t1-t0):.2f} calpa {1e3*(t2-t1):.2f} to_host {1e3*(t3-t2):.2f}")
