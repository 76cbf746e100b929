"""Per-frame device time of a workload: fast kernel alone, full graph on one
stream, full graphs on 2/3 streams (frames alternating)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1308_4908_b200 import _native as N  # noqa: E402
from paper_1308_4908_b200 import simulate as sim  # noqa: E402
from paper_1308_4908_b200.engine import DeviceRig  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
W, H = wl["size"]
out_size = wl["out"]
dev = torch.device("cuda", 0)
rs = sim.baseline_rig(wl["rig"], W, H, seed=0)
cals = rs.calibrations()
sets = [sim.simulate_rig_device(sim.hdr_chart(W, H), rs, dev, seed=i) for i in range(6)]
p = bench._params(wl)
rigs = [DeviceRig.from_device(fs, rs.sensors, cals) for fs in sets]
n = 6


def timeit(fn, streams):
    torch.cuda.synchronize()
    main = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    for s in streams:
        s.wait_stream(main)
    for i in range(n):
        fn(i)
    for s in streams:
        main.wait_stream(s)
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


out = rigs[0].allocate_outputs(out_size)
for i in range(2):
    rigs[i].reconstruct(out_size, p, ref_size=(W, H), out=out, flags=N.HDR_FLAG_FAST_ONLY)
print("fast only, eager: %.2f ms" % timeit(lambda i: rigs[i].reconstruct(out_size, p, ref_size=(W, H), out=out, flags=N.HDR_FLAG_FAST_ONLY), []))
print("full, eager: %.2f ms" % timeit(lambda i: rigs[i].reconstruct(out_size, p, ref_size=(W, H), out=out), []))
print("slow items", rigs[0].slow_items(out_size))
for lanes in (1, 2, 3):
    streams = [torch.cuda.Stream(dev) for _ in range(lanes)]
    ws = [rigs[0].workspace(*out_size)] + [torch.empty_like(rigs[0].workspace(*out_size)) for _ in range(lanes - 1)]
    outs = [out] + [rigs[0].allocate_outputs(out_size) for _ in range(lanes - 1)]
    caps = []
    for i in range(n):
        r = DeviceRig.from_device(sets[i], rs.sensors, cals)
        r._workspaces[tuple(out_size)] = ws[i % lanes]
        caps.append(r.capture(out_size, p, ref_size=(W, H), out=outs[i % lanes]))

    def run(i):
        with torch.cuda.stream(streams[i % lanes]):
            caps[i].replay()
    run(0)
    print("graphs, %d lanes: %.2f ms/frame" % (lanes, timeit(run, streams)))
