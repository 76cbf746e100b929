"""CPU oracle for the unified HDR LPA operator -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm may import this module, and only as the checker or the timed CPU
baseline.  The product path (``paper_1308_4908_b200``) never imports it.

It wraps ``lpa_oracle.c`` (a float64 C restatement of the reference's
``frames_to_samples`` -> ``SampleIndex`` -> ``reconstruct_frame`` path, see
the header of that file for file:line citations) through ctypes.  Inputs are
duck-typed so the same call accepts the reference's own ``hdrfuse`` objects
(for pinning, in the dev container) and this repo's mirrors of them.

Parity status: pinned.  ``tests/test_oracle_golden.py`` checks the oracle
bit-for-bit against golden vectors produced by the reference itself
(``oracle/gen_golden.py``), including the reference's PIN9 SHA-256
(``pkg/tests/test_acceptance.py:60``).  The ICI extension has no reference
counterpart; its parity is pinned only by this repo's known-answer tests.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_BUILD = _HERE / "_build"
_LIB_PATH = _BUILD / "liblpa_oracle.so"
_SRC = _HERE / "lpa_oracle.c"
_lock = threading.Lock()
_lib = None

SUPPORT_SIGMAS = 3.0  # lpa.py:37

# phase -> 2x2 tile indexed [y%2][x%2] (bayer.py:24-29)
_TILES = {
    "RGGB": (0, 1, 1, 2),
    "BGGR": (2, 1, 1, 0),
    "GRBG": (1, 0, 2, 1),
    "GBRG": (1, 2, 0, 1),
}


class OSensor(ctypes.Structure):
    _fields_ = [
        ("width", ctypes.c_int),
        ("height", ctypes.c_int),
        ("raw", ctypes.c_void_p),
        ("saturation_level", ctypes.c_int),
        ("exposure_time", ctypes.c_double),
        ("gain", ctypes.c_double),
        ("exposure_scaling", ctypes.c_double),
        ("T", ctypes.c_double * 6),
        ("tile", ctypes.c_int * 4),
        ("bias", ctypes.c_void_p),
        ("readvar", ctypes.c_void_p),
        ("nonuni", ctypes.c_void_p),
        ("bias_s", ctypes.c_double),
        ("readvar_s", ctypes.c_double),
        ("nonuni_s", ctypes.c_double),
        ("defective", ctypes.c_void_p),
        ("sensor_id", ctypes.c_int),
    ]


def build(force: bool = False) -> Path:
    """Compile lpa_oracle.c (gcc, -ffp-contract=off so the reference's float64
    operation order is kept) into oracle/_build/liblpa_oracle.so."""
    if _LIB_PATH.exists() and not force and _LIB_PATH.stat().st_mtime >= _SRC.stat().st_mtime:
        return _LIB_PATH
    _BUILD.mkdir(exist_ok=True)
    tmp = _LIB_PATH.with_suffix(f".{os.getpid()}.tmp.so")
    cmd = [
        "gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
        "-shared", "-o", str(tmp), str(_SRC), "-lm",
    ]
    subprocess.run(cmd, check=True)
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        lib = ctypes.CDLL(str(build()))
        lib.oracle_set_dsyevd.argtypes = [ctypes.c_void_p]
        lib.oracle_has_dsyevd.restype = ctypes.c_int
        lib.oracle_max_threads.restype = ctypes.c_int
        lib.oracle_frames_to_samples.restype = ctypes.c_int64
        lib.oracle_frames_to_samples.argtypes = [
            ctypes.POINTER(OSensor), ctypes.c_int,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
        ]
        lib.oracle_reconstruct_channel.restype = ctypes.c_int
        lib.oracle_reconstruct_channel.argtypes = [
            ctypes.POINTER(OSensor), ctypes.c_int, ctypes.c_int,
            ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int,
            ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_double, ctypes.c_int,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_void_p,
        ]
        fn = _scipy_dsyevd()
        if fn:
            lib.oracle_set_dsyevd(fn)
        _lib = lib
        return lib


def _scipy_dsyevd():
    """The LAPACK dsyevd numba binds for np.linalg.eigvalsh (numba/_lapack.c
    imports it from scipy.linalg.cython_lapack); None if SciPy is absent."""
    try:
        from scipy.linalg import cython_lapack
    except Exception:  # pragma: no cover - SciPy is in the image
        return None
    cap = cython_lapack.__pyx_capi__["dsyevd"]
    get_name = ctypes.pythonapi.PyCapsule_GetName
    get_name.restype = ctypes.c_char_p
    get_name.argtypes = [ctypes.py_object]
    get_ptr = ctypes.pythonapi.PyCapsule_GetPointer
    get_ptr.restype = ctypes.c_void_p
    get_ptr.argtypes = [ctypes.py_object, ctypes.c_char_p]
    return get_ptr(cap, get_name(cap))


def has_lapack() -> bool:
    return bool(_load().oracle_has_dsyevd())


def max_threads() -> int:
    """Host cores this process may use (not OMP_NUM_THREADS, which launchers
    such as torchrun set to 1 per process)."""
    try:
        return len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        return int(_load().oracle_max_threads())


def _pattern_name(pattern) -> str:
    return getattr(pattern, "value", pattern)


def _as_plane(entry, shape):
    """Calibration entry -> (plane f64 contiguous or None, scalar)."""
    data = getattr(entry, "data", entry)
    arr = np.asarray(data, dtype=np.float64)
    if arr.ndim == 0:
        return None, float(arr)
    if arr.shape != shape:
        raise ValueError(f"calibration plane shape {arr.shape} != frame shape {shape}")
    if arr.size and np.all(arr == arr.flat[0]):
        return None, float(arr.flat[0])
    return np.ascontiguousarray(arr), 0.0


def make_sensors(frames, configs, cals):
    """ctypes OSensor array + keep-alive list from duck-typed reference objects."""
    if not (len(frames) == len(configs) == len(cals)):
        raise ValueError("frames, configs and cals must align")
    keep = []
    arr = (OSensor * len(frames))()
    for k, (fr, cfg, cal) in enumerate(zip(frames, configs, cals)):
        raw = np.ascontiguousarray(getattr(fr, "data", fr), dtype=np.uint16)
        h, w = raw.shape
        keep.append(raw)
        s = arr[k]
        s.width, s.height = w, h
        s.raw = raw.ctypes.data
        s.saturation_level = int(cfg.saturation_level)
        s.sensor_id = int(getattr(cfg, "sensor_id", k))
        s.exposure_time = float(cfg.exposure_time)
        s.gain = float(cfg.gain)
        s.exposure_scaling = float(cfg.exposure_scaling)
        T = np.asarray(cfg.transform, dtype=np.float64).reshape(6)
        for i in range(6):
            s.T[i] = float(T[i])
        tile = _TILES[_pattern_name(cfg.pattern)]
        for i in range(4):
            s.tile[i] = tile[i]
        for name, field, sfield in (
            ("bias", "bias", "bias_s"),
            ("readout_variance", "readvar", "readvar_s"),
            ("nonuniformity", "nonuni", "nonuni_s"),
        ):
            plane, scal = _as_plane(getattr(cal, name), (h, w))
            if plane is None:
                setattr(s, field, None)
                setattr(s, sfield, scal)
            else:
                keep.append(plane)
                setattr(s, field, plane.ctypes.data)
                setattr(s, sfield, 0.0)
        defective = getattr(cfg, "defective", None)
        if defective is not None and len(defective):
            mask = np.zeros(h * w, np.uint8)
            mask[np.asarray(defective, dtype=np.int64)] = 1
            keep.append(mask)
            s.defective = mask.ctypes.data
        else:
            s.defective = None
    return arr, keep


def frames_to_samples(frames, configs, cals):
    """(positions (n,2), channels u8, values, sigmas, sensor_ids) exactly as
    hdrfuse.frames_to_samples would produce them (radiometry.py:303-349)."""
    lib = _load()
    arr, keep = make_sensors(frames, configs, cals)
    total = sum(int(np.asarray(getattr(f, "data", f)).size) for f in frames)
    pos = np.empty((max(total, 1), 2))
    chan = np.empty(max(total, 1), np.uint8)
    val = np.empty(max(total, 1))
    sig = np.empty(max(total, 1))
    sid = np.empty(max(total, 1), np.int32)
    n = lib.oracle_frames_to_samples(
        arr, len(frames), pos.ctypes.data, chan.ctypes.data, val.ctypes.data,
        sig.ctypes.data, sid.ctypes.data,
    )
    del keep
    return pos[:n], chan[:n], val[:n], sig[:n], sid[:n]


def grid_coordinates(out_size, ref_size):
    """lpa.py:213-224."""
    out_w, out_h = out_size
    ref_w, ref_h = ref_size
    xs = (np.arange(out_w) + 0.5) * (ref_w / out_w) - 0.5
    ys = (np.arange(out_h) + 0.5) * (ref_h / out_h) - 0.5
    return np.ascontiguousarray(xs), np.ascontiguousarray(ys)


def channel_scale(params, channel: int) -> float:
    """ReconstructionParams.channel_scale (lpa.py:66-69)."""
    if params.per_channel_scale and channel == 1:
        return params.scale / math.sqrt(2.0)
    return params.scale


def resolved_max_radius(params) -> float:
    """lpa.py:71-74 (always from params.scale, never the channel scale)."""
    if params.max_support_radius is not None:
        return float(params.max_support_radius)
    return 10.0 * math.sqrt(params.scale)


def scale_ladder(h: float, n_scales: int, ratio: float):
    """ICI scale set h_k = h * ratio**k (ICI spec)."""
    return [h * ratio ** k for k in range(n_scales)]


def reconstruct(frames, configs, cals, out_size, params, ref_size=None, threads=None,
                channels=(0, 1, 2), rows=None):
    """Reference-semantics reconstruction on the CPU.

    Returns a dict: ``rgb`` (H, W, 3) float32 clamped like lpa.py:428 (NaN kept),
    ``val``/``gx``/``gy`` (3, H, W) float64 unclamped, ``outcome`` (3, H, W) u8
    (order*16 + radius step, 0xFF = NaN), ``scale_idx`` (3, H, W) u8, ``count``
    (3, H, W) u16 samples in the accepted window.  ``rows=(r0, r1)`` restricts
    the evaluation to that band of output rows (the outputs cover the band).
    """
    lib = _load()
    arr, keep = make_sensors(frames, configs, cals)
    out_w, out_h = out_size
    if ref_size is None:
        ref_size = out_size
    xs, ys = grid_coordinates(out_size, ref_size)
    if rows is not None:
        ys = np.ascontiguousarray(ys[rows[0]:rows[1]])
        out_h = len(ys)
    n_scales = int(getattr(params, "ici_scales", 1) or 1)
    ratio = float(getattr(params, "ici_ratio", math.sqrt(2.0)))
    gamma = float(getattr(params, "ici_gamma", 1.5))
    use_sigma = 1 if params.weight_mode == "sigma" else 0
    max_r = resolved_max_radius(params)
    m = out_w * out_h
    val = np.full((3, out_h, out_w), np.nan)
    gx = np.full((3, out_h, out_w), np.nan)
    gy = np.full((3, out_h, out_w), np.nan)
    outcome = np.full((3, out_h, out_w), 0xFF, np.uint8)
    sidx = np.zeros((3, out_h, out_w), np.uint8)
    count = np.zeros((3, out_h, out_w), np.uint16)
    nthreads = int(threads) if threads else 0
    for c in channels:
        hs = scale_ladder(channel_scale(params, c), n_scales, ratio)
        hinv = np.array([1.0 / h for h in hs])
        rk = np.array([SUPPORT_SIGMAS * math.sqrt(h) for h in hs])
        bufs = [np.empty(m) for _ in range(3)] + [np.empty(m, np.uint8) for _ in range(2)] + [
            np.empty(m, np.uint16)]
        lib.oracle_reconstruct_channel(
            arr, len(frames), c, xs.ctypes.data, out_w, ys.ctypes.data, out_h,
            int(params.order), n_scales, hinv.ctypes.data, rk.ctypes.data,
            max_r, float(params.cond_threshold), use_sigma, gamma, nthreads,
            bufs[0].ctypes.data, bufs[1].ctypes.data, bufs[2].ctypes.data,
            bufs[3].ctypes.data, bufs[4].ctypes.data, bufs[5].ctypes.data,
        )
        val[c] = bufs[0].reshape(out_h, out_w)
        gx[c] = bufs[1].reshape(out_h, out_w)
        gy[c] = bufs[2].reshape(out_h, out_w)
        outcome[c] = bufs[3].reshape(out_h, out_w)
        sidx[c] = bufs[4].reshape(out_h, out_w)
        count[c] = bufs[5].reshape(out_h, out_w)
    del keep
    rgb = np.empty((out_h, out_w, 3), np.float32)
    for c in range(3):
        rgb[:, :, c] = np.maximum(val[c], 0.0).astype(np.float32)
    return {"rgb": rgb, "val": val, "gx": gx, "gy": gy, "outcome": outcome, "scale_idx": sidx,
            "count": count}


# ---------------------------------------------------------------------------
# CALPA (reference steering.py) -- structure-adaptive second pass
# ---------------------------------------------------------------------------
def _load_calpa(lib):
    if getattr(lib, "_calpa_ready", False):
        return lib
    lib.oracle_steering_field.argtypes = [
        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
        ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
    ]
    lib.oracle_reconstruct_channel_steered.argtypes = [
        ctypes.POINTER(OSensor), ctypes.c_int, ctypes.c_int,
        ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
        ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int,
        ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
    ]
    lib._calpa_ready = True
    return lib


def steering_field(gx, gy, adaptive, gradient_scale=1.0, threads=None):
    """(theta, sigma, gamma) planes: compute_steering_field (steering.py:177-203)
    with _kernels.steering_field_kernel (_kernels.py:310-392)."""
    lib = _load_calpa(_load())
    scale = float(gradient_scale)
    gxs = np.ascontiguousarray(np.asarray(gx, dtype=np.float64) / scale)
    gys = np.ascontiguousarray(np.asarray(gy, dtype=np.float64) / scale)
    h, w = gxs.shape
    theta, sigma, gamma = (np.empty_like(gxs) for _ in range(3))
    lib.oracle_steering_field(gxs.ctypes.data, gys.ctypes.data, w, h,
                              adaptive.gradient_window // 2, adaptive.gradient_window / 4.0,
                              float(adaptive.lambda1), float(adaptive.lambda2),
                              float(adaptive.alpha), float(adaptive.sigma_max),
                              theta.ctypes.data, sigma.ctypes.data, gamma.ctypes.data,
                              int(threads) if threads else 0)
    return theta, sigma, gamma


def kernel_inputs(theta, sigma, gamma, scale):
    """SteeringField.covariance_entries + kernel_inputs (steering.py:80-107), in
    numpy exactly as the reference evaluates them."""
    ct = np.cos(theta)
    st = np.sin(theta)
    s = sigma
    c11 = gamma * (s * ct * ct + st * st / s)
    c12 = gamma * (ct * st) * (1.0 / s - s)
    c22 = gamma * (s * st * st + ct * ct / s)
    r0 = SUPPORT_SIGMAS * np.sqrt(scale * sigma / gamma)
    return ((c11 / scale).ravel(), (c12 / scale).ravel(), (c22 / scale).ravel(), r0.ravel())


def auto_gradient_scale(values):
    """steering.py:206-211."""
    finite = values[np.isfinite(values)]
    if not len(finite):
        return 1.0
    s = float(np.percentile(np.abs(finite), 99.5))
    return s if s > 0 else 1.0


def reconstruct_channel_steered(frames, configs, cals, out_size, base, channel, steering,
                                ref_size=None, threads=None):
    """reconstruct_channel(..., steering=...) (lpa.py:379-408, two-phase)."""
    lib = _load_calpa(_load())
    arr, keep = make_sensors(frames, configs, cals)
    out_w, out_h = out_size
    xs, ys = grid_coordinates(out_size, ref_size or out_size)
    m = out_w * out_h
    h = channel_scale(base, channel)
    an = [np.ascontiguousarray(a, dtype=np.float64) for a in steering]
    bufs = [np.empty(m) for _ in range(3)] + [np.empty(m, np.uint8)]
    lib.oracle_reconstruct_channel_steered(
        arr, len(frames), int(channel), xs.ctypes.data, out_w, ys.ctypes.data, out_h,
        int(base.order), an[0].ctypes.data, an[1].ctypes.data, an[2].ctypes.data,
        an[3].ctypes.data, 1.0 / h, SUPPORT_SIGMAS * math.sqrt(h),
        resolved_max_radius(base), float(base.cond_threshold),
        1 if base.weight_mode == "sigma" else 0, int(threads) if threads else 0,
        *[b.ctypes.data for b in bufs])
    del keep
    return tuple(b.reshape(out_h, out_w) for b in bufs)


def calpa(frames, configs, cals, out_size, adaptive, ref_size=None, threads=None):
    """calpa_reconstruct (steering.py:214-248): isotropic G pass -> gradient scale
    -> steering field -> steered pass per channel.  Returns a dict with rgb
    (float32 HWC), the field and the per-channel outcome codes."""
    base = adaptive.base
    out_w, out_h = out_size

    def field_for(c):
        o = reconstruct(frames, configs, cals, out_size, base, ref_size=ref_size,
                        threads=threads, channels=(c,))
        val, gx, gy = o["val"][c], o["gx"][c], o["gy"][c]
        scale = adaptive.gradient_scale or auto_gradient_scale(val)
        return steering_field(gx, gy, adaptive, scale, threads), scale

    shared = field_for(1) if adaptive.share_steering else None
    rgb = np.empty((out_h, out_w, 3), np.float32)
    outcome = np.empty((3, out_h, out_w), np.uint8)
    for c in range(3):
        (theta, sigma, gamma), scale = shared if shared is not None else field_for(c)
        steering = kernel_inputs(theta, sigma, gamma, channel_scale(base, c))
        val, _, _, oc = reconstruct_channel_steered(frames, configs, cals, out_size, base, c,
                                                    steering, ref_size, threads)
        rgb[:, :, c] = np.maximum(val, 0.0).astype(np.float32)
        outcome[c] = oc
    theta, sigma, gamma = shared[0] if shared is not None else (None, None, None)
    return {"rgb": rgb, "theta": theta, "sigma": sigma, "gamma": gamma, "outcome": outcome,
            "gradient_scale": shared[1] if shared is not None else None}
