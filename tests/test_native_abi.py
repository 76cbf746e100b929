"""The C-ABI shared library: loads without a GPU, exports every entry point
declared in include/hdr_lpa.h, struct layouts agree between C and ctypes,
argument validation returns the documented status codes."""

import ctypes
import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

from paper_1308_4908_b200 import _native as N

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "hdr_lpa.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?(?:unsigned\s+)?(?:long\s+)*\w+\s*\*?\s*(hdr_\w+)\s*\(",
                                  text, re.M)))


def test_library_loads_and_exports_every_declared_symbol():
    L = N.lib()
    decl = declared_functions()
    assert len(decl) >= 8
    for name in decl:
        assert hasattr(L, name), name
    assert set(decl) == set(N.EXPORTED)
    out = subprocess.run(["nm", "-D", "--defined-only", str(N.LIB_PATH)], capture_output=True,
                         text=True).stdout
    for name in decl:
        assert re.search(rf"\bT {name}\b", out), name


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_the_header(tmp_path):
    src = tmp_path / "sizes.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "hdr_lpa.h"\n'
                   'int main(void){printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(HdrSensor),'
                   ' sizeof(HdrParams), sizeof(HdrOutputs), offsetof(HdrSensor, transform),'
                   ' offsetof(HdrParams, max_radius), offsetof(HdrSensor, defective));return 0;}\n')
    exe = tmp_path / "sizes"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), "-o", str(exe), str(src)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(N.HdrSensor), ctypes.sizeof(N.HdrParams), ctypes.sizeof(N.HdrOutputs),
            N.HdrSensor.transform.offset, N.HdrParams.max_radius.offset,
            N.HdrSensor.defective.offset]
    assert got == want


def test_abi_version_and_status_strings():
    L = N.lib()
    assert L.hdr_lpa_abi_version() == 5
    for code, text in ((0, "ok"), (1, "invalid argument"), (2, "invalid sensor configuration"),
                       (3, "dimension mismatch"), (4, "workspace too small"), (5, "CUDA error"),
                       (6, "kernel fault")):
        assert L.hdr_lpa_status_string(code).decode() == text


def test_workspace_size():
    n = ctypes.c_size_t()
    s = (N.HdrSensor * 3)()
    for k in range(3):
        s[k].width, s[k].height = 2400, 1700
    assert N.lib().hdr_lpa_workspace_bytes(s, 3, 2400, 1700, ctypes.byref(n)) == 0
    phase = 4 * 1200 * 850 * 8  # four (f_hat, 1/den) float2 phase planes per sensor
    lut = 65536 * 16  # exact (f_hat, 1/den) float64 per raw value
    assert n.value == 256 + 64 * 1024 + 3 * (phase + lut) + 2400 * 1700 * 3 * 4
    s[0].width = 2399  # odd width: phase planes padded to an even float2 count
    assert N.lib().hdr_lpa_workspace_bytes(s, 1, 2400, 1700, ctypes.byref(n)) == 0
    assert n.value == 256 + 64 * 1024 + 4 * 1200 * 850 * 8 + lut + 2400 * 1700 * 3 * 4
    assert N.lib().hdr_lpa_workspace_bytes(s, 3, 0, 10, ctypes.byref(n)) == N.HDR_ERR_ARG


def _sensor(**kw):
    s = N.HdrSensor()
    s.raw = 4096  # never dereferenced: validation fails or succeeds before any launch
    s.width, s.height, s.pitch = 64, 48, 64
    s.saturation_level = 4095
    for i, c in enumerate((0, 1, 1, 2)):
        s.tile[i] = c
    s.exposure_time, s.gain, s.exposure_scaling = 0.1, 0.27, 1.0
    for i, v in enumerate((1, 0, 0, 0, 1, 0)):
        s.transform[i] = v
    s.nonuniformity = 1.0
    for k, v in kw.items():
        setattr(s, k, v)
    return s


def _params(**kw):
    p = N.HdrParams()
    p.order, p.n_scales, p.max_radius, p.cond_threshold = 1, 1, 8.0, 1e8
    for c in range(3):
        p.scale[c][0] = 0.7
    for k, v in kw.items():
        setattr(p, k, v)
    return p


@pytest.mark.parametrize("sensor_kw, params_kw, code", [
    ({}, {"order": 3}, N.HDR_ERR_ARG),
    ({}, {"n_scales": 0}, N.HDR_ERR_ARG),
    ({}, {"weight_mode": 7}, N.HDR_ERR_ARG),
    ({"exposure_scaling": 1.5}, {}, N.HDR_ERR_CONFIG),
    ({"gain": 0.0}, {}, N.HDR_ERR_ARG),
    ({"nonuniformity": 0.0}, {}, N.HDR_ERR_CONFIG),
    ({"pitch": 10}, {}, N.HDR_ERR_ARG),
])
def test_reconstruct_argument_validation(sensor_kw, params_kw, code):
    arr = (N.HdrSensor * 1)(_sensor(**sensor_kw))
    o = N.HdrOutputs()
    o.rgb = 8192
    rc = N.lib().hdr_lpa_reconstruct(arr, 1, ctypes.byref(_params(**params_kw)), 64, 48, 64.0,
                                     48.0, 0, 0, ctypes.byref(o), 16384, 1 << 20, None)
    assert rc == code


def test_singular_transform_is_a_configuration_error():
    s = _sensor()
    for i, v in enumerate((1, 2, 0, 2, 4, 0)):
        s.transform[i] = v
    arr = (N.HdrSensor * 1)(s)
    o = N.HdrOutputs()
    o.rgb = 8192
    rc = N.lib().hdr_lpa_reconstruct(arr, 1, ctypes.byref(_params()), 64, 48, 64.0, 48.0, 0, 0,
                                     ctypes.byref(o), 16384, 1 << 20, None)
    assert rc == N.HDR_ERR_CONFIG


def test_gradient_scale_argument_validation():
    """hdr_gradient_scale rejects arguments before any device work (its
    histogram counters are 32-bit: n < 2^32; q in [0, 1]; workspace size)."""
    need = ctypes.c_size_t()
    assert N.lib().hdr_gradient_scale_workspace_bytes(ctypes.byref(need)) == N.HDR_OK
    L = N.lib()
    assert L.hdr_gradient_scale(8192, 1 << 32, 0.995, 16384, 1 << 20, need.value, None) == \
        N.HDR_ERR_ARG
    assert L.hdr_gradient_scale(8192, 100, 1.5, 16384, 1 << 20, need.value, None) == N.HDR_ERR_ARG
    assert L.hdr_gradient_scale(8192, -1, 0.5, 16384, 1 << 20, need.value, None) == N.HDR_ERR_ARG
    assert L.hdr_gradient_scale(8192, 100, 0.5, 16384, 1 << 20, need.value - 1, None) == \
        N.HDR_ERR_WORKSPACE


def test_status_codes_map_to_reference_exceptions():
    import paper_1308_4908_b200 as hl

    with pytest.raises(hl.ConfigurationError):
        N.check(N.HDR_ERR_CONFIG, "x")
    with pytest.raises(hl.ShapeMismatchError):
        N.check(N.HDR_ERR_SHAPE, "x")
    with pytest.raises(ValueError):
        N.check(N.HDR_ERR_ARG, "x")
    with pytest.raises(RuntimeError):
        N.check(N.HDR_ERR_CUDA, "x")
    N.check(N.HDR_OK, "x")


def test_missing_native_library_fails_loudly():
    """No CPU fallback: without the CUDA library the product path raises."""
    code = ("import paper_1308_4908_b200 as hl\n"
            "from paper_1308_4908_b200 import _native as N\n"
            "N.lib()\n")
    env = dict(os.environ, HDR_LPA_LIB=str(ROOT / "no_such_lib.so"))
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                       text=True)
    assert r.returncode != 0
    assert "no_such_lib.so" in r.stderr
