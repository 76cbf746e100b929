"""ctypes binding of the C ABI in include/hdr_lpa.h (libhdrlpa.so).

The shared library is built in-tree for sm_100a by :func:`build` (called by
``__graft_entry__.build()``) and loaded from ``paper_1308_4908_b200/``.  There
is no fallback: if the library cannot be built or loaded, every entry point
raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from pathlib import Path

from .radiometry import ConfigurationError
from .validation import ShapeMismatchError

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
LIB_PATH = PKG / "libhdrlpa.so"
SOURCES = sorted((PKG / "csrc").glob("*.cu*")) + [ROOT / "include" / "hdr_lpa.h"]

MAX_SENSORS = 8
MAX_SCALES = 8

(HDR_OK, HDR_ERR_ARG, HDR_ERR_CONFIG, HDR_ERR_SHAPE, HDR_ERR_WORKSPACE, HDR_ERR_CUDA,
 HDR_ERR_FAULT) = range(7)
HDR_FAULT_MBAR_TIMEOUT = 1
HDR_FAULT_BOUNDS = 2
HDR_WEIGHT_VARIANCE, HDR_WEIGHT_SIGMA = 0, 1
HDR_OUTCOME_NAN = 0xFF
HDR_FLAG_FAST_ONLY = 1
HDR_FLAG_NO_MERGE = 2
HDR_FLAG_SKIP_R = 4
HDR_FLAG_SKIP_G = 8
HDR_FLAG_SKIP_B = 16

EXPORTED = (
    "hdr_lpa_workspace_bytes",
    "hdr_lpa_reconstruct",
    "hdr_lpa_reconstruct_steered",
    "hdr_steering_field",
    "hdr_lpa_evaluate_samples",
    "hdr_saturation_mask",
    "hdr_radiance_planes",
    "hdr_sample_planes",
    "hdr_lpa_slow_items",
    "hdr_lpa_workspace_status",
    "hdr_sample_count_workspace_bytes",
    "hdr_sample_count",
    "hdr_compact_samples",
    "hdr_sample_index_workspace_bytes",
    "hdr_sample_index_bbox",
    "hdr_sample_index_build",
    "hdr_simulate_sensor",
    "hdr_gradient_scale_workspace_bytes",
    "hdr_gradient_scale",
    "hdr_steering_field_devscale",
    "hdr_fp64_peak_probe",
    "hdr_lpa_status_string",
    "hdr_lpa_last_error",
    "hdr_lpa_abi_version",
    "hdr_lpa_launch_count",
    "hdr_lpa_kernel_timer",
    "hdr_lpa_kernel_timer_read",
)


class HdrSensor(ctypes.Structure):
    _fields_ = [
        ("raw", ctypes.c_void_p),
        ("width", ctypes.c_int),
        ("height", ctypes.c_int),
        ("pitch", ctypes.c_int),
        ("saturation_level", ctypes.c_int),
        ("tile", ctypes.c_int * 4),
        ("exposure_time", ctypes.c_double),
        ("gain", ctypes.c_double),
        ("exposure_scaling", ctypes.c_double),
        ("transform", ctypes.c_double * 6),
        ("bias", ctypes.c_double),
        ("readout_variance", ctypes.c_double),
        ("nonuniformity", ctypes.c_double),
        ("bias_plane", ctypes.c_void_p),
        ("readvar_plane", ctypes.c_void_p),
        ("nonuni_plane", ctypes.c_void_p),
        ("defective", ctypes.c_void_p),
    ]


class HdrParams(ctypes.Structure):
    _fields_ = [
        ("order", ctypes.c_int),
        ("weight_mode", ctypes.c_int),
        ("n_scales", ctypes.c_int),
        ("flags", ctypes.c_int),
        ("scale", (ctypes.c_double * MAX_SCALES) * 3),
        ("max_radius", ctypes.c_double),
        ("cond_threshold", ctypes.c_double),
        ("ici_gamma", ctypes.c_double),
    ]


class HdrOutputs(ctypes.Structure):
    _fields_ = [
        ("rgb", ctypes.c_void_p),
        ("grad", ctypes.c_void_p),
        ("scale_idx", ctypes.c_void_p),
        ("outcome", ctypes.c_void_p),
        ("value", ctypes.c_void_p),
        ("count", ctypes.c_void_p),
        ("work", ctypes.c_void_p),
        ("rgb_half", ctypes.c_void_p),
        ("half_scale", ctypes.c_float),
    ]


class HdrSampleIndex(ctypes.Structure):
    _fields_ = [("packed", ctypes.c_void_p), ("cell_start", ctypes.c_void_p),
                ("n", ctypes.c_int64), ("x0", ctypes.c_int), ("y0", ctypes.c_int),
                ("nx", ctypes.c_int), ("ny", ctypes.c_int)]


class HdrSteering(ctypes.Structure):
    _fields_ = [("theta", ctypes.c_void_p), ("sigma", ctypes.c_void_p), ("gamma", ctypes.c_void_p)]


_lock = threading.Lock()
_lib = None


UNITS = ("hdr_lpa.cu", "fast_o0.cu", "fast_o1.cu", "fast_o2.cu")
NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC"]


def compile_library(out: Path, extra_flags=(), verbose_ptxas: bool = False) -> Path:
    """nvcc every translation unit of csrc/ for sm_100a in parallel, then link
    the shared library ``out``."""
    import tempfile

    with tempfile.TemporaryDirectory(prefix="hdrlpa_build_") as tmp:
        procs, objs = [], []
        for unit in UNITS:
            obj = Path(tmp) / (unit + ".o")
            cmd = ["nvcc", *NVCC_FLAGS, *extra_flags, "-I", str(ROOT / "include"), "-c", "-o",
                   str(obj), str(PKG / "csrc" / unit)]
            if verbose_ptxas:
                cmd[1:1] = ["-Xptxas", "-v"]
            procs.append((unit, subprocess.Popen(cmd, stderr=subprocess.PIPE, text=True)))
            objs.append(str(obj))
        errs = []
        for unit, p in procs:
            _, err = p.communicate()
            if p.returncode != 0:
                errs.append(f"{unit}:\n{err}")
            elif verbose_ptxas:
                print(err, end="")
        if errs:
            raise RuntimeError("nvcc failed:\n" + "\n".join(errs))
        subprocess.run(["nvcc", "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o",
                        str(out), *objs, "-lcuda"], check=True)
    return out


def build(force: bool = False) -> Path:
    """Compile libhdrlpa.so for sm_100a in-tree (skipped when up to date)."""
    if LIB_PATH.exists() and not force:
        mtime = LIB_PATH.stat().st_mtime
        if all(s.stat().st_mtime <= mtime for s in SOURCES):
            return LIB_PATH
    tmp = LIB_PATH.with_name(f"libhdrlpa.{os.getpid()}.tmp.so")
    compile_library(tmp)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


def lib():
    """The loaded library (built first if missing or stale).  HDR_LPA_LIB may
    point at an alternative build of the same sources (experiments)."""
    global _lib
    with _lock:
        if _lib is None:
            alt = os.environ.get("HDR_LPA_LIB")
            L = ctypes.CDLL(alt if alt else str(build()))
            L.hdr_lpa_workspace_bytes.argtypes = [ctypes.POINTER(HdrSensor), ctypes.c_int,
                                                  ctypes.c_int, ctypes.c_int,
                                                  ctypes.POINTER(ctypes.c_size_t)]
            L.hdr_lpa_reconstruct.argtypes = [
                ctypes.POINTER(HdrSensor), ctypes.c_int, ctypes.POINTER(HdrParams),
                ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                ctypes.c_int, ctypes.c_int, ctypes.POINTER(HdrOutputs),
                ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
            ]
            L.hdr_lpa_reconstruct_steered.argtypes = [
                ctypes.POINTER(HdrSensor), ctypes.c_int, ctypes.POINTER(HdrParams),
                ctypes.POINTER(HdrSteering), ctypes.c_int, ctypes.c_int, ctypes.c_double,
                ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.POINTER(HdrOutputs),
                ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
            ]
            L.hdr_lpa_evaluate_samples.argtypes = [
                ctypes.POINTER(HdrSampleIndex), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
            ]
            L.hdr_steering_field.argtypes = [
                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                ctypes.c_void_p,
            ]
            L.hdr_saturation_mask.argtypes = [ctypes.POINTER(HdrSensor), ctypes.c_void_p,
                                              ctypes.c_int, ctypes.c_void_p]
            L.hdr_radiance_planes.argtypes = [ctypes.POINTER(HdrSensor), ctypes.c_int,
                                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
            L.hdr_sample_planes.argtypes = [ctypes.POINTER(HdrSensor), ctypes.c_void_p,
                                            ctypes.c_void_p, ctypes.c_void_p]
            L.hdr_lpa_slow_items.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint32),
                                             ctypes.c_void_p]
            L.hdr_lpa_workspace_status.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint32),
                                                   ctypes.POINTER(ctypes.c_uint32), ctypes.c_void_p]
            i64, vp, P64 = ctypes.c_longlong, ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong)
            L.hdr_sample_count_workspace_bytes.argtypes = [ctypes.c_int,
                                                           ctypes.POINTER(ctypes.c_size_t)]
            L.hdr_sample_count.argtypes = [ctypes.POINTER(HdrSensor), vp, P64, vp, vp]
            L.hdr_compact_samples.argtypes = [ctypes.POINTER(HdrSensor), ctypes.c_int, vp, vp, i64,
                                              vp, vp, vp, vp, vp, vp, vp]
            L.hdr_sample_index_workspace_bytes.argtypes = [i64, i64,
                                                           ctypes.POINTER(ctypes.c_size_t)]
            PI = ctypes.POINTER(ctypes.c_int)
            L.hdr_sample_index_bbox.argtypes = [vp, vp, i64, ctypes.c_int, P64, PI, PI, PI, PI, vp,
                                                vp]
            L.hdr_sample_index_build.argtypes = [vp, vp, vp, vp, i64, ctypes.c_int, ctypes.c_int,
                                                 ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp,
                                                 vp, ctypes.c_size_t, vp]
            L.hdr_simulate_sensor.argtypes = [vp, ctypes.c_int, ctypes.c_int,
                                              ctypes.POINTER(HdrSensor), ctypes.c_ulonglong,
                                              ctypes.c_int, ctypes.c_int, vp]
            L.hdr_gradient_scale_workspace_bytes.argtypes = [ctypes.POINTER(ctypes.c_size_t)]
            L.hdr_gradient_scale.argtypes = [vp, i64, ctypes.c_double, vp, vp, ctypes.c_size_t, vp]
            L.hdr_steering_field_devscale.argtypes = [
                vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                ctypes.c_double, ctypes.c_double, ctypes.c_double, vp, vp, vp, vp, vp]
            L.hdr_fp64_peak_probe.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_void_p]
            L.hdr_lpa_status_string.restype = ctypes.c_char_p
            L.hdr_lpa_status_string.argtypes = [ctypes.c_int]
            L.hdr_lpa_last_error.restype = ctypes.c_char_p
            for name in EXPORTED:
                if name not in ("hdr_lpa_status_string", "hdr_lpa_last_error",
                                "hdr_lpa_launch_count"):
                    getattr(L, name).restype = ctypes.c_int
            L.hdr_lpa_launch_count.restype = ctypes.c_ulonglong
            L.hdr_lpa_launch_count.argtypes = []
            L.hdr_lpa_kernel_timer.argtypes = [ctypes.c_int]
            L.hdr_lpa_kernel_timer_read.argtypes = [ctypes.POINTER(ctypes.c_float)]
            if L.hdr_lpa_abi_version() != 5:
                raise RuntimeError("libhdrlpa.so ABI version mismatch")
            _lib = L
        return _lib


def check(status: int, what: str) -> None:
    """Map C status codes onto the reference's exception types."""
    if status == HDR_OK:
        return
    msg = f"{what}: {lib().hdr_lpa_status_string(status).decode()}"
    if status == HDR_ERR_CONFIG:
        raise ConfigurationError(msg)
    if status == HDR_ERR_SHAPE:
        raise ShapeMismatchError(msg)
    if status in (HDR_ERR_ARG, HDR_ERR_WORKSPACE):
        raise ValueError(msg)
    raise RuntimeError(f"{msg} ({lib().hdr_lpa_last_error().decode()})")
