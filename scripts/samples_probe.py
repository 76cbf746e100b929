"""Scattered-sample path (RadianceSamples -> GPU SampleIndex -> CSR kernel)
throughput at the cfg2 size."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1308_4908_b200 as hl  # noqa: E402
from paper_1308_4908_b200 import simulate as sim  # noqa: E402
from paper_1308_4908_b200.engine import DeviceRig  # noqa: E402
from paper_1308_4908_b200.samples import RadianceSamples, SampleIndex, evaluate_index  # noqa: E402

W, H = 2400, 1700
dev = torch.device("cuda", 0)
rs = sim.baseline_rig("misaligned", W, H, seed=0)
frames = sim.simulate_rig_device(sim.hdr_chart(W, H), rs, dev, seed=1)
rig = DeviceRig.from_device(frames, rs.sensors, rs.calibrations())
samples = RadianceSamples(*rig.materialize_samples())
print("samples", len(samples), flush=True)
for order in (1, 2):
    p = hl.ReconstructionParams(order=order, scale=0.7)
    for it in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        samples._indexes.clear()
        idx = [samples.index(c) for c in hl.ColorChannel]
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        img = hl.reconstruct_frame(samples, (W, H), p)
        t2 = time.perf_counter()
        print(f"order {order}: index {1e3*(t1-t0):.1f} ms, evaluate+host {1e3*(t2-t1):.1f} ms",
              flush=True)
