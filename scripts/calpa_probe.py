"""CALPA (two-pass steered reconstruction) throughput at the cfg2/cfg3 size."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1308_4908_b200 as hl  # noqa: E402
from paper_1308_4908_b200 import simulate as sim  # noqa: E402
from paper_1308_4908_b200.engine import DeviceRig  # noqa: E402
from paper_1308_4908_b200.steering import gradient_field, compute_steering_field  # noqa: E402

W, H = 2400, 1700
dev = torch.device("cuda", 0)
rig_name = sys.argv[1] if len(sys.argv) > 1 else "aligned"
rs = sim.baseline_rig(rig_name, W, H, seed=0)
frames = sim.simulate_rig_torch(sim.hdr_chart(W, H), rs, dev, seed=1)
rig = DeviceRig.from_device(frames, rs.sensors, rs.calibrations())
ap = hl.AdaptiveParams(base=hl.ReconstructionParams(order=1, scale=0.7))
base = ap.base
for it in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    val, gx, gy = gradient_field(rig, (W, H), base, hl.ColorChannel.G, None)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    from paper_1308_4908_b200.steering import auto_gradient_scale
    fld = compute_steering_field((gx, gy), ap, ap.gradient_scale or auto_gradient_scale(val))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    out = rig.reconstruct_steered((W, H), base, (fld.theta, fld.sigma, fld.gamma))
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"{rig_name}: pass1 {1e3*(t1-t0):.1f} ms, steering {1e3*(t2-t1):.1f} ms, "
          f"steered pass {1e3*(t3-t2):.1f} ms, total {1e3*(t3-t0):.1f} ms", flush=True)
