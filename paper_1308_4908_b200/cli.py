"""Command line: reconstruct / video / simulate.

Mirrors the reference CLI's reconstruct command (pkg/src/hdrfuse/cli.py:156-238):
per-sensor 16-bit PGM frames + a rig JSON in, an HDR PFM out, plus a run
manifest (parameters, input SHA-256s, timing) next to it.  Exit codes follow
the reference (cli.py:43-68): 0 ok, 2 usage/config error, 3 shape mismatch,
4 numeric failure.  ``video`` streams a frame sequence through the pinned
double-buffered pipeline, frame-parallel across torchrun ranks, resumable.
"""

from __future__ import annotations

import functools
import hashlib
import json
import sys
import time
from pathlib import Path

import click
import numpy as np

from . import __version__
from .lpa import reconstruct_frame
from .pnm import PnmParseError, read_pgm16, write_pfm, write_pgm16
from .radiometry import ConfigurationError, frames_to_samples
from .rig import ConfigError, load_rig
from .validation import ShapeMismatchError

EXIT_USAGE, EXIT_SHAPE, EXIT_NUMERIC = 2, 3, 4


def _exit_codes(f):
    @functools.wraps(f)
    def wrapper(*args, **kwargs):
        try:
            return f(*args, **kwargs)
        except (ConfigError, ConfigurationError, PnmParseError, FileNotFoundError) as e:
            click.echo(f"error: {e}", err=True)
            sys.exit(EXIT_USAGE)
        except ShapeMismatchError as e:
            click.echo(f"error: {e}", err=True)
            sys.exit(EXIT_SHAPE)
        except (FloatingPointError, ZeroDivisionError) as e:
            click.echo(f"numeric failure: {e}", err=True)
            sys.exit(EXIT_NUMERIC)
        except ValueError as e:
            click.echo(f"error: {e}", err=True)
            sys.exit(EXIT_USAGE)

    return wrapper


def _sha256(path) -> str:
    return hashlib.sha256(Path(path).read_bytes()).hexdigest()


def _params(rig, order, scale, max_radius, cond_threshold, ici_scales, ici_gamma):
    kw = {}
    if order is not None:
        kw["order"] = order
    if scale is not None:
        kw["scale"] = scale
    if max_radius is not None:
        kw["max_support_radius"] = max_radius
    if cond_threshold is not None:
        kw["cond_threshold"] = cond_threshold
    if ici_scales is not None:
        kw["ici_scales"] = ici_scales
    if ici_gamma is not None:
        kw["ici_gamma"] = ici_gamma
    return rig.params(**kw)


def _load_frames(rig, paths):
    if len(paths) != len(rig.sensors):
        raise ShapeMismatchError(
            f"frame count mismatch: {len(paths)} frames for {len(rig.sensors)} sensors")
    raws = []
    for path, sensor in zip(paths, rig.sensors):
        if not Path(path).exists():
            raise ConfigError(f"frame does not exist: {path}")
        raws.append(read_pgm16(path, pattern=sensor.config.pattern))
    cals = [s.calibration(r.width, r.height) for s, r in zip(rig.sensors, raws)]
    return raws, cals


recon_options = [
    click.option("--order", "-M", type=click.IntRange(0, 2), default=None),
    click.option("--scale", "-h", type=float, default=None, help="window scale h (px^2)"),
    click.option("--max-radius", type=float, default=None),
    click.option("--cond-threshold", type=float, default=None),
    click.option("--ici-scales", type=click.IntRange(1, 8), default=None,
                 help="ICI scale count J (1 = fixed scale)"),
    click.option("--ici-gamma", type=float, default=None),
    click.option("--width", type=int, default=None),
    click.option("--height", type=int, default=None),
]


def _with(opts):
    def deco(f):
        for o in reversed(opts):
            f = o(f)
        return f

    return deco


@click.group()
@click.version_option(__version__)
def main():
    """B200-native unified HDR LPA reconstruction."""


@main.command("reconstruct")
@click.argument("args", nargs=-1, type=click.Path(path_type=Path))
@click.option("--rig", "rig_opt", type=click.Path(path_type=Path), default=None,
              help="rig JSON (alternative to the positional RIG_CONFIG)")
@click.option("--out", "-o", type=click.Path(path_type=Path), required=True, help="Output PFM.")
@_with(recon_options)
@click.option("--calpa", is_flag=True, help="Structure-adaptive second pass (steering.py).")
@click.option("--alpha", type=float, default=None, help="Structure sensitivity (CALPA).")
@click.option("--grad-window", type=int, default=None, help="Gradient analysis window (odd).")
@click.option("--threads", type=int, default=None,
              help="accepted for compatibility (host threads do not drive the GPU path)")
@click.option("--preview", type=click.Path(path_type=Path), default=None,
              help="Also write an 8-bit gamma preview PNG.")
@_exit_codes
def cmd_reconstruct(args, rig_opt, out, order, scale, max_radius, cond_threshold, ici_scales,
                    ici_gamma, width, height, calpa, alpha, grad_window, threads, preview):
    """reconstruct RIG_CONFIG FRAMES... -o OUT.pfm (reference cli.py:156-238):
    an HDR PFM from per-sensor raw PGM frames."""
    from .steering import AdaptiveParams, calpa_reconstruct

    args = list(args)
    if rig_opt is None:
        if not args:
            raise click.UsageError("missing RIG_CONFIG")
        rig_config, frames = args[0], args[1:]
    else:
        rig_config, frames = rig_opt, args
    if not frames:
        raise click.UsageError("missing FRAMES")
    rig = load_rig(rig_config)
    raws, cals = _load_frames(rig, list(frames))
    params = _params(rig, order, scale, max_radius, cond_threshold, ici_scales, ici_gamma)
    defaults = dict(getattr(rig, "reconstruction", {}) or {})
    alpha = alpha if alpha is not None else float(defaults.get("alpha", 0.005))
    grad_window = grad_window if grad_window is not None else int(defaults.get("grad_window", 9))
    ref_size = (raws[0].width, raws[0].height)            # reference cli.py:199
    out_size = (width or ref_size[0], height or ref_size[1])
    t0 = time.perf_counter()
    samples = frames_to_samples(raws, rig.configs, cals)
    if calpa:
        adaptive = AdaptiveParams(alpha=alpha, gradient_window=grad_window, base=params)
        hdr = calpa_reconstruct(samples, out_size, adaptive, ref_size=ref_size)
    else:
        hdr = reconstruct_frame(samples, out_size, params, ref_size=ref_size)
    elapsed = time.perf_counter() - t0
    out.parent.mkdir(parents=True, exist_ok=True)
    write_pfm(hdr, out)
    manifest = {
        "command": "reconstruct", "version": __version__, "rig_config": str(rig_config),
        "frames": [{"path": str(p), "sha256": _sha256(p)} for p in frames],
        "parameters": {"order": params.order, "scale": params.scale,
                       "max_radius": params.max_support_radius,
                       "cond_threshold": params.cond_threshold, "calpa": bool(calpa),
                       "alpha": alpha, "grad_window": grad_window,
                       "ici_scales": params.ici_scales, "ici_ratio": params.ici_ratio,
                       "ici_gamma": params.ici_gamma, "width": out_size[0],
                       "height": out_size[1]},
        "threads": threads, "device": _device_name(), "seconds": elapsed,
        "nan_fraction": float(np.isnan(hdr.data).mean()),
    }
    Path(str(out) + ".manifest.json").write_text(json.dumps(manifest, indent=2) + "\n")
    click.echo(f"wrote {out} ({elapsed:.3f} s)")
    if preview is not None:
        _write_preview(hdr, rig, preview)
        click.echo(f"wrote {preview}")


def _write_preview(hdr, rig, path: Path) -> None:
    """Gamma-2.2 8-bit preview (reference cli.py:241-255): NaNs take the least
    sensitive sensor's saturation radiance, scaled by the 99th percentile."""
    from PIL import Image

    data = hdr.data.astype(np.float64).copy()
    sat = [(c.saturation_level - c.black_level) / (c.gain * c.exposure_time * c.exposure_scaling)
           for c in rig.configs]
    data[~np.isfinite(data)] = max(sat)
    finite = data[np.isfinite(data)]
    top = np.percentile(finite, 99.0) if finite.size else 1.0
    norm = np.clip(data / max(top, 1e-30), 0.0, 1.0) ** (1.0 / 2.2)
    Path(path).parent.mkdir(parents=True, exist_ok=True)
    Image.fromarray((norm * 255.0 + 0.5).astype(np.uint8)).save(path)


@main.command("video")
@click.option("--rig", "rig_config", type=click.Path(path_type=Path), required=True)
@click.option("--out-dir", type=click.Path(path_type=Path), required=True)
@click.argument("frames_dir", type=click.Path(path_type=Path))
@_with(recon_options)
@_exit_codes
def cmd_video(rig_config, out_dir, frames_dir, order, scale, max_radius, cond_threshold,
              ici_scales, ici_gamma, width, height):
    """Reconstruct a sequence: FRAMES_DIR/frame_<k>_s<i>.pgm -> OUT_DIR/frame_<k>.pfm.

    Frame-parallel across torchrun ranks (frame k on rank k mod N), streamed
    through the pinned double-buffered H2D / compute / D2H pipeline; frames
    whose output exists are skipped (resume)."""
    import torch

    from .pipeline import FramePipeline
    from .runner import FrameParallelRunner, init_from_env, pfm_sink

    init_from_env()
    rig = load_rig(rig_config)
    n_s = len(rig.sensors)
    ks = sorted({int(p.name.split("_")[1]) for p in Path(frames_dir).glob("frame_*_s0.pgm")})
    if not ks:
        raise ConfigError(f"no frame_<k>_s0.pgm files in {frames_dir}")
    first, cals = _load_frames(rig, [Path(frames_dir) / f"frame_{ks[0]:06d}_s{i}.pgm"
                                     for i in range(n_s)])
    params = _params(rig, order, scale, max_radius, cond_threshold, ici_scales, ici_gamma)
    ref_size = (first[0].width, first[0].height)
    out_size = (width or ref_size[0], height or ref_size[1])
    pipe = FramePipeline(rig.configs, cals, [f.data.shape for f in first], out_size, params,
                         ref_size=ref_size)
    sink, exists = pfm_sink(out_dir)
    runner = FrameParallelRunner(len(ks))
    host_out = [torch.empty((out_size[1], out_size[0], 3), dtype=torch.float32).pin_memory()
                for _ in range(2)]
    mine = [i for i in runner.my_frames() if not exists(ks[i])]
    inflight, done = [], []

    def drain_one():
        j, ev, slot = inflight.pop(0)
        ev.synchronize()
        sink(ks[j], slot.numpy())
        done.append(j)

    t0 = time.perf_counter()
    for n, i in enumerate(mine):
        raws, _ = _load_frames(rig, [Path(frames_dir) / f"frame_{ks[i]:06d}_s{j}.pgm"
                                     for j in range(n_s)])
        host = [torch.from_numpy(r.data.view(np.int16)).pin_memory() for r in raws]
        if len(inflight) == 2:  # output slot n % 2 is about to be reused
            drain_one()
        inflight.append((i, pipe.submit(host, host_out[n % 2]), host_out[n % 2]))
    while inflight:
        drain_one()
    pipe.synchronize()
    total = runner.all_done(done)
    click.echo(f"rank {runner.rank}: {len(done)} frames in {time.perf_counter() - t0:.2f} s; "
               f"{len(total)} frames done across ranks")


@main.command("simulate")
@click.option("--rig", "rig_config", type=click.Path(path_type=Path), required=True)
@click.option("--out-dir", type=click.Path(path_type=Path), required=True)
@click.option("--frames", "n_frames", type=int, default=1)
@click.option("--seed", type=int, default=0)
@click.option("--width", type=int, default=None)
@click.option("--height", type=int, default=None)
@_exit_codes
def cmd_simulate(rig_config, out_dir, n_frames, seed, width, height):
    """Synthetic raw frames of the HDR test chart for a rig (input generator)."""
    from . import simulate as sim

    rig = load_rig(rig_config)
    sizes = [s.size or (width, height) for s in rig.sensors]
    W, H = width or sizes[0][0], height or sizes[0][1]
    gt = sim.hdr_chart(W, H)
    noise = [sim.SensorNoise(float(np.mean(s.bias.value)), float(np.mean(s.readout_variance.value)),
                             float(np.mean(s.nonuniformity.value))) for s in rig.sensors]
    out_dir.mkdir(parents=True, exist_ok=True)
    for k in range(n_frames):
        spec = sim.RigSpec(sensors=rig.configs, noise=noise, sensor_sizes=[(W, H)] * len(noise),
                           seed=seed + k)
        for i, f in enumerate(sim.simulate_rig(gt, spec)):
            write_pgm16(f, out_dir / f"frame_{k:06d}_s{i}.pgm")
    click.echo(f"wrote {n_frames} x {len(rig.sensors)} frames to {out_dir}")


def _device_name():
    try:
        import torch

        return torch.cuda.get_device_name(torch.cuda.current_device())
    except Exception:
        return None


if __name__ == "__main__":
    main()
