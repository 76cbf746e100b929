"""FramePipeline throughput vs slots for a workload (cfg3 / cfg4)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1308_4908_b200 import simulate as sim  # noqa: E402
from paper_1308_4908_b200.pipeline import FramePipeline  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
W, H = wl["size"]
out_w, out_h = wl["out"]
dev = torch.device("cuda", 0)
rs = sim.baseline_rig(wl["rig"], W, H, seed=0)
sets = [sim.simulate_rig_device(sim.hdr_chart(W, H), rs, dev, seed=i) for i in range(3)]
host = [[t.cpu().pin_memory() for t in fs] for fs in sets]
p = bench._params(wl)
for slots in (1, 2, 3):
    outs = [torch.empty((out_h, out_w, 3), dtype=torch.float32).pin_memory() for _ in range(slots)]
    pipe = FramePipeline(rs.sensors, rs.calibrations(), [tuple(t.shape) for t in sets[0]],
                         (out_w, out_h), p, ref_size=(W, H), device=dev, slots=slots)
    for i in range(slots + 1):
        pipe.submit(host[i % 3], outs[i % slots])
    pipe.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(pipe.s_in)
    n = 8
    for i in range(n):
        pipe.submit(host[i % 3], outs[i % slots])
    pipe.s_in.wait_stream(pipe.s_out)
    e1.record(pipe.s_in)
    pipe.synchronize()
    print(f"slots {slots}: {e0.elapsed_time(e1) / n:.2f} ms/frame", flush=True)
