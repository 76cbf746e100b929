"""The multi-rank code paths on the GPU box with its one GPU: two processes
(gloo for the host collectives) each reconstruct their own row band or frames
on cuda:0 with the CUDA engine -- no kernel waits on another rank -- and the
gathered results are bit-identical to a single-rank reconstruction
(output invariant under the band / GPU split, the analogue
of the reference's thread invariance, pkg/tests/test_acceptance.py:334-357)."""

import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

W, H = 160, 104


def _case():
    from paper_1308_4908_b200 import simulate as sim

    rig = sim.baseline_rig("misaligned", W, H, seed=17)
    return rig, sim.simulate_rig(sim.hdr_chart(W, H), rig)


def _worker(rank, world, port, q):
    import paper_1308_4908_b200 as hl
    from paper_1308_4908_b200 import runner

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        torch.cuda.set_device(0)
        rig, frames = _case()
        p = hl.ReconstructionParams(order=2, scale=0.7, ici_scales=4)
        dev = hl.frames_to_samples(frames, rig.sensors, rig.calibrations()).device()
        fn = runner.engine_band_fn(dev, (W, H), p)
        full = runner.reconstruct_banded(lambda r0, r1: fn(r0, r1).cpu(), H, W)
        # frame-parallel: frames k -> rank k mod N, each computed on this rank
        fr = runner.FrameParallelRunner(4)
        got = {}
        for k in fr.my_frames():
            fs = frames if k % 2 == 0 else frames[::-1]
            cfg = rig.sensors if k % 2 == 0 else rig.sensors[::-1]
            cal = rig.calibrations() if k % 2 == 0 else rig.calibrations()[::-1]
            img = hl.reconstruct_frame(hl.frames_to_samples(fs, cfg, cal), (W, H), p)
            got[k] = img.data
        if rank == 0:
            q.put(("band", full.numpy()))
        q.put(("frames", got))
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu_band_split_bit_identical(cuda):
    import paper_1308_4908_b200 as hl

    rig, frames = _case()
    p = hl.ReconstructionParams(order=2, scale=0.7, ici_scales=4)
    single = hl.reconstruct_frame(hl.frames_to_samples(frames, rig.sensors,
                                                       rig.calibrations()), (W, H), p).data
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(3)]
    for pr in procs:
        pr.join(300)
        assert pr.exitcode == 0
    band = [v for k, v in res if k == "band"][0]
    assert np.array_equal(band, single, equal_nan=True)
    frames_done = {}
    for k, v in res:
        if k == "frames":
            frames_done.update(v)
    assert sorted(frames_done) == [0, 1, 2, 3]
    for k in (0, 2):
        assert np.array_equal(frames_done[k], single, equal_nan=True)
