"""Breakdown of the exact-path work items of one reconstruction (diagnostic):
kk = 0 full exact evaluation, kk = k + 1 float64 recomputation at scale k;
per channel.  usage: slow_items_probe.py [workload]"""
import collections
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1308_4908_b200 import simulate as sim  # noqa: E402
from paper_1308_4908_b200.engine import DeviceRig  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
dev = torch.device("cuda", 0)
W, H = wl["size"]
rs = sim.baseline_rig(wl["rig"], W, H, seed=0, n_sensors=wl.get("sensors", 3))
frames = sim.simulate_rig_device(sim.hdr_chart(W, H), rs, dev, seed=1)
rig = DeviceRig.from_device(frames, rs.sensors, rs.calibrations())
p = bench._params(wl)
ow, oh = wl["out"]
out = rig.reconstruct(wl["out"], p, ref_size=(W, H), want_scale_idx=True, want_outcome=True)
n = rig.slow_items(wl["out"])
ws = rig.workspace(ow, oh)
hdr = ws[:24].view(torch.int32).cpu().numpy().astype("uint32")  # header words 0..5
all_items = ws[ws.numel() - ow * oh * 3 * 4:].view(torch.int32).cpu().numpy().astype("uint32")
cap = ow * oh * 3
back = all_items[cap - hdr[4]:][::-1]  # recomputation slots (after lpa_precise_kernel)
print("full evaluations", hdr[0], "recomputations", hdr[4],
      "of which failed -> full", int(((back != 0xFFFFFFFF) & (((back >> 2) & 15) == 0)).sum()))
items = all_items[:hdr[0]]
kk = (items >> 2) & 15
ch = items & 3
pix = items >> 6
print("items", n, "of", ow * oh * 3)
print("kk", sorted(collections.Counter(kk.tolist()).items()))
print("channel", sorted(collections.Counter(ch.tolist()).items()))
sidx = out["scale_idx"].cpu().numpy()
oc = out["outcome"].cpu().numpy()
sel = sidx[ch, pix // ow, pix % ow]
print("selected scale of the items", sorted(collections.Counter(sel.tolist()).items()))
print("outcomes of the items", sorted(collections.Counter(oc[ch, pix // ow, pix % ow].tolist()).items())[:12])
print("all selected scales", [int((sidx == k).sum()) for k in range(4)])
