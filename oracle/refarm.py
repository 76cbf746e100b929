"""The reference's own CPU path, staged for timing -- TEST/BENCH INFRASTRUCTURE.

``stage()`` installs the unmodified reference package (``hdrfuse``, pure
Python + numba) from ``/root/reference/pkg`` into ``oracle/_ref/`` with the
reference's own build recipe (``pip install --no-index --no-deps --target``).
``oracle/_ref/`` is git-ignored (no reference source enters the history) but
travels to the GPU box with the repo snapshot, so ``bench.py --impl
reference`` can time the REAL reference (``frames_to_samples`` +
``reconstruct_frame``, numba ``lpa_evaluate`` on all host cores) on the box's
host, beside the C restatement (``lpa_oracle.c``, kind "port").

Only ``bench.py``'s reference/cpu-baseline legs and ``tests/`` use this
module; the product package never imports it.

Band samples: the reference has no row-band entry, so a band of output rows
[y0, y0 + rows) is timed by the public API on the sensor frames cropped to
the rows that band can reach, with every sensor transform shifted so that the
cropped frame's row 0 is sensor row s0 and the output grid's row 0 is
reference row y0 (``T02 += T01*s0``, ``T12 += T11*s0 - y0``; s0 even so the
Bayer phase is unchanged).  The work per output row equals the full frame's;
the timing covers frames_to_samples + SampleIndex + the per-pixel fits of the
band, scaled to a frame by ``out_h / rows``.
"""

from __future__ import annotations

import math
import os
import shutil
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_DIR = HERE / "_ref"
REF_SRC = Path("/root/reference/pkg")


def stage(force: bool = False) -> bool:
    """pip-install the reference into oracle/_ref (dev container only: the GPU
    box has no /root/reference and uses the staged copy).  True when staged."""
    if (REF_DIR / "hdrfuse" / "__init__.py").exists() and not force:
        return True
    if not REF_SRC.exists():
        return False
    tmp = HERE / f"_ref.{os.getpid()}.tmp"
    shutil.rmtree(tmp, ignore_errors=True)
    r = subprocess.run([sys.executable, "-m", "pip", "install", "--quiet", "--no-index",
                        "--no-build-isolation", "--no-deps", "--find-links", "/opt/wheelhouse",
                        "--target", str(tmp), str(REF_SRC)],
                       capture_output=True, text=True)
    if r.returncode != 0 or not (tmp / "hdrfuse" / "__init__.py").exists():
        shutil.rmtree(tmp, ignore_errors=True)
        print(f"refarm.stage: reference install failed: {r.stderr.strip()[-300:]}",
              file=sys.stderr)
        return False
    shutil.rmtree(REF_DIR, ignore_errors=True)
    os.replace(tmp, REF_DIR)
    return True


_hf = None


def load():
    """Import the staged reference (``hdrfuse``), or None when it is absent."""
    global _hf
    if _hf is not None:
        return _hf
    if not (REF_DIR / "hdrfuse" / "__init__.py").exists():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/hdr_numba_cache")
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    try:
        import hdrfuse  # noqa: F401
        from hdrfuse import _kernels
    except Exception as e:  # numba missing on the box, broken install, ...
        print(f"refarm.load: {type(e).__name__}: {e}", file=sys.stderr)
        return None
    import numba

    # all host cores (launchers such as torchrun set OMP_NUM_THREADS=1)
    try:
        ncpu = len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        ncpu = os.cpu_count() or 1
    numba.set_num_threads(max(1, min(ncpu, numba.config.NUMBA_NUM_THREADS)))
    _kernels.warmup()  # JIT outside any timed region (_kernels.py:395)
    _hf = hdrfuse
    return _hf


def threads() -> int:
    import numba

    return int(numba.get_num_threads())


def _shifted_config(hf, cfg, s0: int, y0: int):
    T = np.array(cfg.transform, dtype=np.float64)
    T[0, 2] = T[0, 2] + T[0, 1] * s0
    T[1, 2] = T[1, 2] + T[1, 1] * s0 - y0
    return hf.SensorConfig(sensor_id=int(cfg.sensor_id), exposure_time=float(cfg.exposure_time),
                           gain=float(cfg.gain), exposure_scaling=float(cfg.exposure_scaling),
                           transform=T, saturation_level=int(cfg.saturation_level),
                           bit_depth=int(cfg.bit_depth),
                           pattern=hf.BayerPattern(str(getattr(cfg.pattern, "value", cfg.pattern))),
                           black_level=float(cfg.black_level), defective=None)


def band_inputs(hf, frames, configs, cals, y0: int, rows: int, out_h: int, reach: float):
    """Reference objects for output rows [y0, y0+rows): cropped frames, shifted
    transforms, cropped calibration planes.  ``reach`` = how far (sensor rows)
    a band's windows extend beyond it (max radius + misalignment)."""
    H = frames[0].data.shape[0]
    s0 = max(0, int(math.floor(y0 - reach)) & ~1)
    s1 = min(H, int(math.ceil(y0 + rows + reach)))
    rf, rc, rk = [], [], []
    for f, c, cal in zip(frames, configs, cals):
        rf.append(hf.CFAImage(np.ascontiguousarray(f.data[s0:s1]), int(f.bit_depth),
                              hf.BayerPattern(str(getattr(f.pattern, "value", f.pattern)))))
        rc.append(_shifted_config(hf, c, s0, y0))
        planes = [np.ascontiguousarray(np.asarray(getattr(cal, a).data)[s0:s1])
                  for a in ("bias", "readout_variance", "nonuniformity")]
        rk.append(hf.NoiseCalibration(bias=hf.FloatFrame(planes[0]),
                                      readout_variance=hf.FloatFrame(planes[1]),
                                      nonuniformity=hf.FloatFrame(planes[2]),
                                      gain_estimate=float(getattr(cal, "gain_estimate", 0.0)
                                                          or c.gain)))
    return rf, rc, rk, s1 - s0


def band_seconds(hf, frames, configs, cals, out_w: int, y0: int, rows: int, out_h: int,
                 order: int, scale: float, reach: float):
    """Seconds the reference takes for output rows [y0, y0+rows) of an
    out_w x out_h reconstruction on the reference grid (public API:
    frames_to_samples + reconstruct_frame)."""
    rf, rc, rk, _ = band_inputs(hf, frames, configs, cals, y0, rows, out_h, reach)
    params = hf.ReconstructionParams(order=order, scale=scale)
    t0 = time.perf_counter()
    samples = hf.frames_to_samples(rf, rc, rk)
    img = hf.reconstruct_frame(samples, (out_w, rows), params, ref_size=(out_w, rows))
    dt = time.perf_counter() - t0
    return dt, img
