"""Distributed logic of the frame-parallel / row-band runner on CPU with two
gloo ranks (the CUDA compute is replaced by the oracle, which computes the
same per-pixel function)."""

import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1308_4908_b200 import runner


def test_row_bands_cover_and_align():
    for h in (1, 7, 8, 96, 1700, 3400):
        for w in (1, 2, 3, 4, 8):
            b = runner.row_bands(h, w)
            assert b[0][0] == 0 and b[-1][1] == h
            assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
            assert all(r0 % 8 == 0 for r0, _ in b)
            assert max(r1 - r0 for r0, r1 in b) - min(r1 - r0 for r0, r1 in b) <= 8 or h < 8 * w


def test_frame_assignment_partitions():
    for n in (0, 1, 5, 300):
        for w in (1, 2, 4, 8):
            got = sorted(k for r in range(w) for k in runner.frame_assignment(n, w, r))
            assert got == list(range(n))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, tmpdir, q):
    import paper_1308_4908_b200 as hl
    from paper_1308_4908_b200 import simulate as sim
    from oracle import oracle

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        W, H = 40, 37
        gt = sim.hdr_chart(W, H)
        rig = sim.baseline_rig("misaligned", W, H, seed=5)
        frames = sim.simulate_rig(gt, rig)
        params = hl.ReconstructionParams(order=2, ici_scales=2)

        def band(r0, r1):
            out = oracle.reconstruct(frames, rig.sensors, rig.calibrations(), (W, H), params,
                                     rows=(r0, r1), threads=1)
            return torch.from_numpy(out["rgb"])

        full = runner.reconstruct_banded(band, H, W)
        # frame-parallel: 5 frames, results written per frame by their owner
        sink, exists = runner.pfm_sink(tmpdir)
        fr = runner.FrameParallelRunner(5)
        done = fr.run(lambda k: torch.full((4, 4, 3), float(k)), sink, exists)
        all_done = fr.all_done(done)
        if rank == 0:
            ref = oracle.reconstruct(frames, rig.sensors, rig.calibrations(), (W, H), params)
            q.put(("band", bool(np.array_equal(full.numpy(), ref["rgb"], equal_nan=True))))
            q.put(("frames", all_done))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_band_split_and_frame_parallel(tmp_path):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, str(tmp_path), q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res["band"] is True
    assert res["frames"] == [0, 1, 2, 3, 4]
    assert sorted(p.name for p in tmp_path.glob("frame_*.pfm")) == [
        f"frame_{k:06d}.pfm" for k in range(5)]


def test_bench_gpus_n_relaunches_n_ranks():
    """`bench.py --gpus 2` without torchrun re-launches itself with one rank per
    GPU (here: gloo, dry run -- the plumbing a SCALE run takes)."""
    import json
    import os
    import subprocess
    import sys

    root = __import__("pathlib").Path(__file__).resolve().parent.parent
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env["HDR_DIST_BACKEND"] = "gloo"
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--dry-run",
                          "--steps", "9"], env=env, capture_output=True, text=True, timeout=240)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line == {"dry_run": True, "n_gpus": 2, "ranks_seen": 2, "frames_total": 9,
                    "max_rank": 1}


def test_bench_rejects_world_size_mismatch():
    import os
    import subprocess
    import sys

    root = __import__("pathlib").Path(__file__).resolve().parent.parent
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--dry-run"],
                         env=env, capture_output=True, text=True, timeout=120)
    assert out.returncode != 0 and "WORLD_SIZE=1" in out.stderr
