"""End-to-end pipeline throughput vs the number of D2H streams (cfg2)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1308_4908_b200 as hl  # noqa: E402
from paper_1308_4908_b200 import simulate as sim  # noqa: E402
from paper_1308_4908_b200.pipeline import FramePipeline  # noqa: E402

W, H = 2400, 1700
dev = torch.device("cuda", 0)
rig = sim.baseline_rig("aligned", W, H, seed=0)
gt = sim.hdr_chart(W, H)
sets = [sim.simulate_rig_device(gt, rig, dev, seed=i) for i in range(4)]
host = [[t.cpu().pin_memory() for t in fs] for fs in sets]
outs = [torch.empty((H, W, 3), dtype=torch.float32).pin_memory() for _ in range(2)]
p = hl.ReconstructionParams(order=1, scale=0.7)
for nd in (1, 2, 3, 4):
    for slots in (2, 3):
        pipe = FramePipeline(rig.sensors, rig.calibrations(), [tuple(t.shape) for t in sets[0]],
                             (W, H), p, device=dev, slots=slots, d2h_streams=nd)
        for i in range(5):
            pipe.submit(host[i % 4], outs[i % 2])
        pipe.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(pipe.s_in)
        n = 60
        for i in range(n):
            pipe.submit(host[i % 4], outs[i % 2])
        pipe.s_in.wait_stream(pipe.s_out)
        e1.record(pipe.s_in)
        pipe.synchronize()
        ms = e0.elapsed_time(e1) / n
        print(f"d2h_streams={nd} slots={slots}: {ms:.3f} ms/frame  {1000 / ms:.1f} fps  "
              f"D2H {pipe.d2h_bytes / ms / 1e6:.1f} GB/s", flush=True)
# raw copy rates
src = torch.empty((H, W, 3), dtype=torch.float32, device=dev)
for nd in (1, 2, 4):
    ss = [torch.cuda.Stream(dev) for _ in range(nd)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for it in range(20):
        cuts = [H * i // nd for i in range(nd + 1)]
        for j, s in enumerate(ss):
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                outs[0][cuts[j]:cuts[j + 1]].copy_(src[cuts[j]:cuts[j + 1]], non_blocking=True)
        for s in ss:
            torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"pure D2H {nd} streams: {src.numel() * 4 / ms / 1e6:.1f} GB/s")
