"""Multi-GPU execution: one process per GPU, torch.distributed for plumbing.

The operator is embarrassingly parallel: every frame is
independent, and inside a frame every output pixel is independent given the
read-only raw frames.  Two partitionings are provided:

* frame-parallel (the throughput mode): frame k is processed by rank
  k mod world; no collective on the data path.  Results are written per frame
  by their owner (resumable: frames whose output exists are skipped).
* row-band split of one frame (the latency mode): rank r reconstructs output
  rows [r0, r1) -- each band stages its own halo from the raw frames, so no
  halo exchange is needed -- and the bands are gathered to rank 0 with one
  collective.  The result is bit-identical to a single-GPU reconstruction
  because a pixel's arithmetic never depends on the band or tile it is in.

The compute callbacks default to the CUDA engine; tests inject the CPU oracle
to exercise the distributed logic with the gloo backend.
"""

from __future__ import annotations

import os
from pathlib import Path
from typing import Callable, Iterable, Optional

import torch
import torch.distributed as dist

TILE_ROWS = 8  # lpa_fast_kernel tile height: bands are aligned to it


def world_info(group=None):
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def frame_assignment(n_frames: int, world: int, rank: int) -> list:
    """Round-robin frame ownership: frame k -> rank k mod world."""
    return list(range(rank, n_frames, world))


def row_bands(out_h: int, world: int, align: int = TILE_ROWS) -> list:
    """Contiguous output-row bands, balanced to whole tile rows."""
    tiles = (out_h + align - 1) // align
    bounds = [min(out_h, (tiles * r // world) * align) for r in range(world + 1)]
    bounds[-1] = out_h
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def gather_bands(band: torch.Tensor, bands: list, out_shape, group=None, dst: int = 0):
    """Gather per-rank row bands (rows x ...) into the full frame on ``dst``.

    Bands are padded to the largest band so a single fixed-size collective
    (all_gather_into_tensor on NCCL, all_gather on gloo) carries them.
    Returns the assembled tensor on ``dst``, None elsewhere.
    """
    world, rank = world_info(group)
    if world == 1:
        return band
    rows = max(r1 - r0 for r0, r1 in bands)
    pad = torch.zeros((rows,) + tuple(band.shape[1:]), dtype=band.dtype, device=band.device)
    pad[: band.shape[0]] = band
    backend = dist.get_backend(group)
    if backend == "nccl":
        allb = torch.empty((world * rows,) + tuple(band.shape[1:]), dtype=band.dtype,
                           device=band.device)
        dist.all_gather_into_tensor(allb, pad, group=group)
        parts = allb.view((world, rows) + tuple(band.shape[1:]))
    else:
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
    if rank != dst:
        return None
    out = torch.empty(tuple(out_shape), dtype=band.dtype, device=band.device)
    for r, (r0, r1) in enumerate(bands):
        out[r0:r1] = parts[r][: r1 - r0]
    return out


def reconstruct_banded(compute_band: Callable[[int, int], torch.Tensor], out_h: int, out_w: int,
                       channels: int = 3, group=None):
    """Split one frame's output rows over the ranks and gather to rank 0.

    ``compute_band(r0, r1)`` returns the (r1 - r0, out_w, channels) band.
    """
    world, rank = world_info(group)
    bands = row_bands(out_h, world)
    r0, r1 = bands[rank]
    band = compute_band(r0, r1)
    return gather_bands(band, bands, (out_h, out_w, channels), group=group)


def engine_band_fn(rig, out_size, params, ref_size=None):
    """compute_band for the CUDA engine: reconstruct rows [r0, r1) of one frame."""
    out = rig.allocate_outputs(out_size)

    def fn(r0, r1):
        rig.reconstruct(out_size, params, ref_size=ref_size, rows=(r0, r1), out=out)
        return out["rgb"][r0:r1]

    return fn


class FrameParallelRunner:
    """Process a frame sequence frame-parallel across the ranks.

    ``process(k)`` computes frame k on this rank's GPU and returns the result;
    ``sink(k, result)`` stores it (e.g. writes a PFM).  With ``out_dir`` and
    ``exists(k)``, frames already written are skipped (resume).
    """

    def __init__(self, n_frames: int, group=None):
        self.n_frames = n_frames
        self.group = group
        self.world, self.rank = world_info(group)

    def my_frames(self) -> list:
        return frame_assignment(self.n_frames, self.world, self.rank)

    def run(self, process: Callable[[int], object], sink: Callable[[int, object], None],
            exists: Optional[Callable[[int], bool]] = None) -> list:
        done = []
        for k in self.my_frames():
            if exists is not None and exists(k):
                continue
            sink(k, process(k))
            done.append(k)
        return done

    def all_done(self, done: Iterable[int]) -> list:
        """Frames processed by every rank (all-gather of the lists)."""
        if self.world == 1:
            return sorted(done)
        lists = [None] * self.world
        dist.all_gather_object(lists, list(done), group=self.group)
        return sorted(k for l in lists for k in l)


def init_from_env(backend: Optional[str] = None):
    """init_process_group from torchrun's environment (RANK, WORLD_SIZE,
    MASTER_ADDR/PORT); NCCL when CUDA is available, else gloo."""
    if int(os.environ.get("WORLD_SIZE", "1")) <= 1 or dist.is_initialized():
        return
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    if backend == "nccl":
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group(backend, device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)


def pfm_sink(out_dir: Path):
    from .images import HDRImage
    from .pnm import write_pfm

    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)

    def sink(k, rgb):
        arr = rgb.cpu().numpy() if isinstance(rgb, torch.Tensor) else rgb
        tmp = out_dir / f".frame_{k:06d}.pfm.tmp"
        write_pfm(HDRImage(arr), tmp)
        os.replace(tmp, out_dir / f"frame_{k:06d}.pfm")

    def exists(k):
        return (out_dir / f"frame_{k:06d}.pfm").exists()

    return sink, exists
