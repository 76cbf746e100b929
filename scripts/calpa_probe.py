"""CALPA stage timings at the cfg2 size (host wall clock with syncs)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1308_4908_b200 as hl  # noqa: E402
from paper_1308_4908_b200 import simulate as sim  # noqa: E402
from paper_1308_4908_b200.engine import DeviceRig  # noqa: E402
from paper_1308_4908_b200.steering import (auto_gradient_scale, compute_steering_field,  # noqa: E402
                                           gradient_field)

W, H = 2400, 1700
dev = torch.device("cuda", 0)
rs = sim.baseline_rig("aligned", W, H, seed=0)
frames = sim.simulate_rig_device(sim.hdr_chart(W, H), rs, dev, seed=1)
rig = DeviceRig.from_device(frames, rs.sensors, rs.calibrations())
ap = hl.AdaptiveParams(base=hl.ReconstructionParams(order=1, scale=0.7))


def t(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, 1e3 * (time.perf_counter() - t0)


for it in range(3):
    (val, gx, gy), a = t(lambda: gradient_field(rig, (W, H), ap.base, hl.ColorChannel.G))
    sc, b = t(lambda: auto_gradient_scale(val))
    fld, c = t(lambda: compute_steering_field((gx, gy), ap, sc))
    out, d = t(lambda: rig.reconstruct_steered((W, H), ap.base, (fld.theta, fld.sigma, fld.gamma)))
    print(f"pass1 {a:.2f} ms, scale {b:.2f} ms, field {c:.2f} ms, steered {d:.2f} ms", flush=True)

# the public API end to end (device frames in, host image out)
for it in range(3):
    img, e = t(lambda: hl.calpa_reconstruct(rig, (W, H), ap))
    o, f = t(lambda: rig.reconstruct_steered((W, H), ap.base, (fld.theta, fld.sigma, fld.gamma)))
    _, g = t(lambda: o["rgb"].cpu().numpy())
    print(f"calpa_reconstruct {e:.2f} ms; of which D2H of the RGB image (pageable) ~{g:.2f} ms",
          flush=True)
