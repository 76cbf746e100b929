"""Small reconstructions of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): cfg2-style co-sited taps, cfg3-style
row taps + rotated sweep + ICI, 2x grid, CALPA, scattered samples, the exact
path fallback.  Exits non-zero if a result is not finite where expected."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1308_4908_b200 as hl  # noqa: E402
from paper_1308_4908_b200 import simulate as sim  # noqa: E402

W, H = 96, 64
gt = sim.hdr_chart(W, H)
which = sys.argv[1] if len(sys.argv) > 1 else "all"


def case(rig, order, J, out=(W, H), scale=0.7):
    r = sim.baseline_rig(rig, W, H, seed=5)
    frames = sim.simulate_rig(gt, r)
    raw = hl.frames_to_samples(frames, r.sensors, r.calibrations())
    p = hl.ReconstructionParams(order=order, scale=scale, ici_scales=J)
    dev = raw.device()
    o = dev.reconstruct(out, p, ref_size=(W, H), want_outcome=True, want_scale_idx=True,
                        want_grad=True)
    torch.cuda.synchronize()
    print(rig, order, J, out, "slow items", dev.status(out), "nan frac",
          float(torch.isnan(o["rgb"]).float().mean()))
    return raw


if which in ("all", "cfg2"):
    case("aligned", 1, 1)                    # co-sited merged taps
if which in ("all", "cfg3"):
    case("misaligned", 2, 4)                 # row taps + rotated sweep + ICI
if which in ("all", "cfg4"):
    case("misaligned", 2, 4, out=(2 * W, 2 * H))
if which in ("all", "big"):
    case("misaligned", 1, 1, scale=45.0)     # too large to stage: exact path for all
if which in ("all", "calpa"):
    r = sim.baseline_rig("aligned", W, H, seed=5)
    raw = hl.frames_to_samples(sim.simulate_rig(gt, r), r.sensors, r.calibrations())
    img = hl.calpa_reconstruct(raw, (W, H), hl.AdaptiveParams(base=hl.ReconstructionParams(order=1)))
    print("calpa nan frac", float(np.isnan(img.data).mean()))
if which in ("all", "samples"):
    r = sim.baseline_rig("misaligned", W, H, seed=5)
    raw = hl.frames_to_samples(sim.simulate_rig(gt, r), r.sensors, r.calibrations())
    img = hl.reconstruct_frame(raw.materialize(), (W, H), hl.ReconstructionParams(order=1))
    print("samples nan frac", float(np.isnan(img.data).mean()))
print("OK")
