import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1308_4908_b200 as hl
from paper_1308_4908_b200 import simulate as sim
from paper_1308_4908_b200 import _native as N
torch.cuda.set_device(0)
case = sys.argv[1]
W, H = 64, 48
gt = sim.hdr_chart(W, H)
rig = sim.baseline_rig("aligned" if case != "mis" else "misaligned", W, H, seed=1)
frames = sim.simulate_rig(gt, rig)
raw = hl.frames_to_samples(frames, rig.sensors, rig.calibrations())
dev = raw.device()
order = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p = hl.ReconstructionParams(order=order)
flags = int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = dev.reconstruct((W, H), p, flags=flags)
torch.cuda.synchronize()
print(case, order, flags, "OK", float(np.nanmean(out["rgb"].cpu().numpy())))
