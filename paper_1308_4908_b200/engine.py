"""Device-resident rig: raw frames + sensor descriptors on one GPU.

PyTorch is used only as the device-memory and stream provider: raw frames,
calibration planes, outputs and the workspace are torch tensors whose device
pointers go through the C ABI (``hdr_lpa_reconstruct``,
``hdr_saturation_mask``, ``hdr_radiance_planes``) on the current torch stream.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _native as N
from .lpa import ReconstructionParams
from .validation import ShapeMismatchError


def _uniform_value(plane: np.ndarray):
    """Scalar if the calibration plane is uniform (exactly), else None."""
    flat = plane.ravel()
    if flat.size and (flat == flat[0]).all():
        return float(flat[0])
    return None


def hdr_params(params: ReconstructionParams, flags: int = 0) -> N.HdrParams:
    """Resolve ReconstructionParams into the C struct (per-channel scales)."""
    P = N.HdrParams()
    P.flags = int(flags)
    P.order = int(params.order)
    P.weight_mode = N.HDR_WEIGHT_SIGMA if params.weight_mode == "sigma" else N.HDR_WEIGHT_VARIANCE
    P.n_scales = int(params.ici_scales)
    for c in range(3):
        for k, h in enumerate(params.channel_scales(c)):
            P.scale[c][k] = float(h)
    P.max_radius = float(params.resolved_max_radius())
    P.cond_threshold = float(params.cond_threshold)
    P.ici_gamma = float(params.ici_gamma)
    return P


# one hdr_lpa_reconstruct call covers < 2^26 output pixels (work-item packing,
# include/hdr_lpa.h); larger outputs are split into row bands here
MAX_BAND_PIXELS = (1 << 26) - 1


def to_host(t: torch.Tensor) -> np.ndarray:
    """A device result as a numpy array, through a pinned block of torch's
    caching host allocator: the copy runs at PCIe DMA speed and recycled
    blocks are already paged in (a pageable ``.cpu()`` of a 49 MB RGB frame
    took ~22 ms, ~2 GB/s).  The array keeps the pinned tensor alive."""
    if t.device.type != "cuda":
        return t.numpy()
    h = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return h.numpy()


def band_split(r0: int, r1: int, out_w: int):
    """Row bands [b0, b1) of at most MAX_BAND_PIXELS output pixels covering [r0, r1)."""
    step = max(1, MAX_BAND_PIXELS // max(1, out_w))
    return [(b, min(b + step, r1)) for b in range(r0, r1, step)]


class DeviceRig:
    """Sensors of one rig resident on a CUDA device.

    ``raws`` are (h, w) int16 tensors holding the uint16 bits of each frame
    (torch has no general uint16 arithmetic; the kernels read the bits as
    uint16).  Configs/calibrations are the host objects of
    :mod:`.radiometry` (or any object with the same attributes).
    """

    def __init__(self, raws, configs, cal_entries, defective, device):
        if len(raws) > N.MAX_SENSORS:
            raise ValueError(f"at most {N.MAX_SENSORS} sensors are supported")
        self.device = torch.device(device)
        self.configs = list(configs)
        self._cal = cal_entries      # per sensor: dict name -> (scalar or device f64 tensor)
        self._defective = defective  # per sensor: device u8 tensor or None
        self._workspaces = {}
        self.raws = []
        self.set_frames(raws)

    # -- construction ------------------------------------------------------
    @classmethod
    def from_host(cls, frames, configs, cals, device=None):
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        device = torch.device(device)
        raws, cal_entries, defective = [], [], []
        for f, cfg, cal in zip(frames, configs, cals):
            data = np.ascontiguousarray(getattr(f, "data", f), dtype=np.uint16)
            h, w = data.shape
            # rows padded to a multiple of 8 elements (16 bytes) so the kernels
            # can stage tiles with TMA bulk tensor copies
            pw = (w + 7) // 8 * 8
            buf = torch.empty((h, pw), dtype=torch.int16, device=device)
            buf[:, :w].copy_(torch.from_numpy(data.view(np.int16)))
            raws.append(buf[:, :w])
            entry = {}
            for name in ("bias", "readout_variance", "nonuniformity"):
                plane = np.asarray(getattr(getattr(cal, name), "data", getattr(cal, name)),
                                   dtype=np.float64)
                if plane.ndim == 0:
                    entry[name] = float(plane)
                    continue
                if plane.shape != (h, w):
                    raise ShapeMismatchError(
                        f"dimension mismatch: {name} {plane.shape} vs frame {(h, w)}")
                u = cal.scalar(name) if hasattr(cal, "scalar") else _uniform_value(plane)
                entry[name] = u if u is not None else torch.from_numpy(
                    np.ascontiguousarray(plane)).to(device)
            cal_entries.append(entry)
            d = getattr(cfg, "defective", None)
            if d is not None and len(d):
                m = np.zeros(h * w, np.uint8)
                m[np.asarray(d, dtype=np.int64)] = 1
                defective.append(torch.from_numpy(m).to(device))
            else:
                defective.append(None)
        return cls(raws, configs, cal_entries, defective, device)

    @classmethod
    def from_device(cls, raws, configs, cals):
        """Rig over raw frames already on a device (int16/uint16 tensors);
        calibrations must be uniform (scalars) or host planes."""
        device = raws[0].device
        entries = []
        for cal, r in zip(cals, raws):
            entry = {}
            for name in ("bias", "readout_variance", "nonuniformity"):
                plane = np.asarray(getattr(getattr(cal, name), "data", getattr(cal, name)),
                                   dtype=np.float64)
                u = float(plane) if plane.ndim == 0 else (
                    cal.scalar(name) if hasattr(cal, "scalar") else _uniform_value(plane))
                entry[name] = u if u is not None else torch.from_numpy(
                    np.ascontiguousarray(plane)).to(device)
            entries.append(entry)
        defective = []
        for cfg, r in zip(configs, raws):
            d = getattr(cfg, "defective", None)
            if d is not None and len(d):
                m = torch.zeros(r.numel(), dtype=torch.uint8, device=device)
                m[torch.as_tensor(np.asarray(d, dtype=np.int64), device=device)] = 1
                defective.append(m)
            else:
                defective.append(None)
        return cls(list(raws), configs, entries, defective, device)

    def set_frames(self, raws):
        """Point the rig at new raw frames (same shapes), e.g. the next video frame."""
        raws = list(raws)
        if len(raws) != len(self.configs):
            raise ShapeMismatchError(f"{len(raws)} frames for {len(self.configs)} sensors")
        for k, r in enumerate(raws):
            if r.dtype not in (torch.int16, torch.uint16) or r.dim() != 2 or r.device != self.device:
                raise ValueError("raw frames must be 2-D int16/uint16 tensors on the rig's device")
            if r.stride(1) != 1:
                raise ValueError("raw frames must be row-contiguous")
            if self.raws and tuple(r.shape) != tuple(self.raws[k].shape):
                raise ShapeMismatchError("frame shape changed")
        self.raws = raws
        self._sensors = self._build_sensors()

    def _build_sensors(self):
        arr = (N.HdrSensor * len(self.raws))()
        for k, (raw, cfg) in enumerate(zip(self.raws, self.configs)):
            s = arr[k]
            s.raw = raw.data_ptr()
            s.height, s.width = int(raw.shape[0]), int(raw.shape[1])
            s.pitch = int(raw.stride(0))
            s.saturation_level = int(cfg.saturation_level)
            pat = cfg.pattern
            tile = pat.flat_tile() if hasattr(pat, "flat_tile") else tuple(
                int(pat.tile[i][j]) for i in (0, 1) for j in (0, 1))
            for i in range(4):
                s.tile[i] = int(tile[i])
            s.exposure_time = float(cfg.exposure_time)
            s.gain = float(cfg.gain)
            s.exposure_scaling = float(cfg.exposure_scaling)
            T = np.asarray(cfg.transform, dtype=np.float64).reshape(6)
            for i in range(6):
                s.transform[i] = float(T[i])
            cal = self._cal[k]
            for name, sfield, pfield in (("bias", "bias", "bias_plane"),
                                         ("readout_variance", "readout_variance", "readvar_plane"),
                                         ("nonuniformity", "nonuniformity", "nonuni_plane")):
                v = cal[name]
                if isinstance(v, torch.Tensor):
                    setattr(s, sfield, 0.0)
                    setattr(s, pfield, v.data_ptr())
                else:
                    setattr(s, sfield, float(v))
                    setattr(s, pfield, None)
            d = self._defective[k]
            s.defective = d.data_ptr() if d is not None else None
        return arr

    # -- hot path ----------------------------------------------------------
    def workspace(self, out_w: int, out_h: int) -> torch.Tensor:
        key = (out_w, out_h)
        if key not in self._workspaces:
            nbytes = ctypes.c_size_t()
            N.check(N.lib().hdr_lpa_workspace_bytes(self._sensors, len(self.raws), out_w, out_h,
                                                     ctypes.byref(nbytes)),
                    "hdr_lpa_workspace_bytes")
            self._workspaces[key] = torch.empty(int(nbytes.value), dtype=torch.uint8,
                                                device=self.device)
        return self._workspaces[key]

    def allocate_outputs(self, out_size, want_grad=False, want_scale_idx=False,
                         want_outcome=False, raw_value=False, want_count=False,
                         want_work=False, rgb_half=False, want_rgb=True):
        out_w, out_h = out_size
        dev = self.device
        out = {}
        if want_rgb or not rgb_half:
            out["rgb"] = torch.empty((out_h, out_w, 3), dtype=torch.float32, device=dev)
        if rgb_half:  # fp16 copy of the clamped radiance times half_scale (ABI v4)
            out["rgb_half"] = torch.empty((out_h, out_w, 3), dtype=torch.float16, device=dev)
        if want_grad:
            out["grad"] = torch.empty((3, 2, out_h, out_w), dtype=torch.float32, device=dev)
        if want_scale_idx:
            out["scale_idx"] = torch.empty((3, out_h, out_w), dtype=torch.uint8, device=dev)
        if want_outcome:
            out["outcome"] = torch.empty((3, out_h, out_w), dtype=torch.uint8, device=dev)
        if raw_value:
            out["value"] = torch.empty((3, out_h, out_w), dtype=torch.float32, device=dev)
        if want_count:
            out["count"] = torch.empty((3, out_h, out_w), dtype=torch.int16, device=dev)
        if want_work:
            out["work"] = torch.zeros((3, out_h, out_w), dtype=torch.int32, device=dev)
        return out

    def reconstruct(self, out_size, params: ReconstructionParams, ref_size=None, rows=None,
                    want_grad=False, want_scale_idx=False, want_outcome=False, raw_value=False,
                    want_count=False, want_work=False, out=None, stream=None, flags=0,
                    half_scale=1.0 / 16):
        """Launch the reconstruction on the current (or given) stream.

        Returns the dict of output tensors (``rgb`` (H, W, 3) float32 and the
        optional ``grad``/``scale_idx``/``outcome``/``value``/``count``/``work``
        planes; ``work`` = inside-window samples over every moment sweep).  With
        ``rows=(r0, r1)`` only that output row band is computed.
        """
        out_w, out_h = int(out_size[0]), int(out_size[1])
        if ref_size is None:
            ref_size = (out_w, out_h)  # lpa.py:393 (ref_size or out_size)
        if out is None:
            out = self.allocate_outputs((out_w, out_h), want_grad, want_scale_idx,
                                        want_outcome, raw_value, want_count, want_work)
        o = N.HdrOutputs()
        o.rgb = out["rgb"].data_ptr() if "rgb" in out else None
        if "rgb_half" in out:
            o.rgb_half = out["rgb_half"].data_ptr()
            o.half_scale = float(half_scale)
        o.grad = out["grad"].data_ptr() if "grad" in out else None
        o.scale_idx = out["scale_idx"].data_ptr() if "scale_idx" in out else None
        o.outcome = out["outcome"].data_ptr() if "outcome" in out else None
        o.value = out["value"].data_ptr() if "value" in out else None
        o.count = out["count"].data_ptr() if "count" in out else None
        o.work = out["work"].data_ptr() if "work" in out else None
        ws = self.workspace(out_w, out_h)
        r0, r1 = (0, out_h) if rows is None else (int(rows[0]), int(rows[1]))
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        hp = hdr_params(params, flags)
        with torch.cuda.device(self.device):
            for b0, b1 in band_split(r0, r1, out_w):  # stream-ordered, one workspace
                rc = N.lib().hdr_lpa_reconstruct(
                    self._sensors, len(self.raws), ctypes.byref(hp), out_w, out_h,
                    float(ref_size[0]), float(ref_size[1]), b0, b1, ctypes.byref(o),
                    ws.data_ptr(), ws.numel(), st.cuda_stream)
                N.check(rc, "hdr_lpa_reconstruct")
        return out

    def reconstruct_steered(self, out_size, params: ReconstructionParams, field, ref_size=None,
                            rows=None, out=None, want_outcome=False, raw_value=False,
                            want_work=False, stream=None, flags=0):
        """CALPA second pass with a steering field (theta, sigma, gamma float64
        device tensors over the output grid): hdr_lpa_reconstruct_steered."""
        out_w, out_h = int(out_size[0]), int(out_size[1])
        if ref_size is None:
            ref_size = (out_w, out_h)
        if out is None:
            out = self.allocate_outputs((out_w, out_h), want_outcome=want_outcome,
                                        raw_value=raw_value, want_work=want_work)
        th, sg, gm = (t.contiguous() for t in field)
        for t in (th, sg, gm):
            if t.dtype != torch.float64 or tuple(t.shape) != (out_h, out_w) or t.device != self.device:
                raise ValueError("steering planes must be float64 (out_h, out_w) device tensors")
        steer = N.HdrSteering(th.data_ptr(), sg.data_ptr(), gm.data_ptr())
        o = N.HdrOutputs()
        o.rgb = out["rgb"].data_ptr()
        o.outcome = out["outcome"].data_ptr() if "outcome" in out else None
        o.value = out["value"].data_ptr() if "value" in out else None
        o.work = out["work"].data_ptr() if "work" in out else None
        ws = self.workspace(out_w, out_h)
        r0, r1 = (0, out_h) if rows is None else (int(rows[0]), int(rows[1]))
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        hp = hdr_params(params, flags)
        with torch.cuda.device(self.device):
            for b0, b1 in band_split(r0, r1, out_w):
                rc = N.lib().hdr_lpa_reconstruct_steered(
                    self._sensors, len(self.raws), ctypes.byref(hp), ctypes.byref(steer), out_w,
                    out_h, float(ref_size[0]), float(ref_size[1]), b0, b1, ctypes.byref(o),
                    ws.data_ptr(), ws.numel(), st.cuda_stream)
                N.check(rc, "hdr_lpa_reconstruct_steered")
        return out

    def capture(self, out_size, params: ReconstructionParams, ref_size=None, out=None,
                half_scale=1.0 / 16, **want) -> "CapturedReconstruction":
        """Record one reconstruction (pre-pass, fast and slow kernels) as a CUDA
        graph over this rig's current frame buffers: ``replay()`` re-runs it
        with one launch.  Refill the frames in place (``copy_`` into
        ``rig.raws``) between replays; ``set_frames`` invalidates the graph.
        The outputs ``out`` (allocated if None) are the graph's."""
        if out is None:
            out = self.allocate_outputs(tuple(out_size), **want)
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        # one eager run first: workspace allocation, kernel attributes
        self.reconstruct(out_size, params, ref_size=ref_size, out=out, stream=side,
                         half_scale=half_scale)
        side.synchronize()
        graph = torch.cuda.CUDAGraph()
        n0 = N.lib().hdr_lpa_launch_count()
        with torch.cuda.graph(graph, stream=side):
            self.reconstruct(out_size, params, ref_size=ref_size, out=out,
                             stream=torch.cuda.current_stream(self.device), half_scale=half_scale)
        n_kernels = int(N.lib().hdr_lpa_launch_count() - n0)
        return CapturedReconstruction(graph, out, n_kernels, list(self.raws))

    def slow_items(self, out_size) -> int:
        """Work items the last reconstruct on this output size sent to the slow
        path (raises RuntimeError if that call's kernels raised a fault)."""
        return self.status(out_size)

    def status(self, out_size, stream=None) -> int:
        """Synchronous check of the last reconstruct on this output size: the
        slow-path item count; RuntimeError if a kernel raised a fault bit
        (e.g. a staging-barrier timeout -- the outputs are incomplete)."""
        ws = self.workspace(int(out_size[0]), int(out_size[1]))
        n, f = ctypes.c_uint32(), ctypes.c_uint32()
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        N.check(N.lib().hdr_lpa_workspace_status(ws.data_ptr(), ctypes.byref(n), ctypes.byref(f),
                                                 st.cuda_stream), "hdr_lpa_workspace_status")
        return int(n.value)

    # -- auxiliary outputs ---------------------------------------------------
    def saturation_masks(self):
        """Boolean (h, w) discard masks per sensor, computed on the GPU."""
        masks = []
        st = torch.cuda.current_stream(self.device)
        for k, raw in enumerate(self.raws):
            h, w = int(raw.shape[0]), int(raw.shape[1])
            wpr = (w + 31) // 32
            bits = torch.empty((h, wpr), dtype=torch.int32, device=self.device)
            N.check(N.lib().hdr_saturation_mask(ctypes.byref(self._sensors[k]), bits.data_ptr(),
                                                wpr, st.cuda_stream), "hdr_saturation_mask")
            b = bits.cpu().numpy().view(np.uint32)
            unpacked = np.unpackbits(b.view(np.uint8).reshape(h, wpr, 4)[..., ::1],
                                     axis=-1, bitorder="little").reshape(h, wpr * 32)
            masks.append(unpacked[:, :w].astype(bool))
        return masks

    def radiance_planes(self, weight_mode: str = "variance"):
        """Per sensor (value, inv_den) float32 (h, w) device tensors."""
        st = torch.cuda.current_stream(self.device)
        mode = N.HDR_WEIGHT_SIGMA if weight_mode == "sigma" else N.HDR_WEIGHT_VARIANCE
        res = []
        for k, raw in enumerate(self.raws):
            v = torch.empty(tuple(raw.shape), dtype=torch.float32, device=self.device)
            iv = torch.empty_like(v)
            N.check(N.lib().hdr_radiance_planes(ctypes.byref(self._sensors[k]), mode,
                                                v.data_ptr(), iv.data_ptr(), st.cuda_stream),
                    "hdr_radiance_planes")
            res.append((v, iv))
        return res

    def sample_planes(self):
        """Per sensor (value, sigma) float64 (h, w) device tensors: the
        reference's sample columns per pixel, bit-exact; sigma 0 = no sample."""
        st = torch.cuda.current_stream(self.device)
        res = []
        for k, raw in enumerate(self.raws):
            v = torch.empty(tuple(raw.shape), dtype=torch.float64, device=self.device)
            s = torch.empty_like(v)
            N.check(N.lib().hdr_sample_planes(ctypes.byref(self._sensors[k]), v.data_ptr(),
                                              s.data_ptr(), st.cuda_stream), "hdr_sample_planes")
            res.append((v, s))
        return res

    def materialize_samples(self):
        """Sample columns in the reference's order (sensor-major, raster;
        radiometry.py:303-349), compacted on the device by the library
        (hdr_sample_count / hdr_compact_samples): positions (n, 2) f64,
        channels u8, values f64, sigmas f64, sensor ids i32 as device tensors.
        Values and sigmas are bit-identical to the reference's; positions use
        apply_transform's operation order (T00*x + T01*y + T02)."""
        lib = N.lib()
        st = torch.cuda.current_stream(self.device)
        planes = self.sample_planes()
        counts, wss = [], []
        with torch.cuda.device(self.device):
            for k, (v, s) in enumerate(planes):
                h = int(self.raws[k].shape[0])
                b = ctypes.c_size_t()
                N.check(lib.hdr_sample_count_workspace_bytes(h, ctypes.byref(b)),
                        "hdr_sample_count_workspace_bytes")
                ws = torch.empty(int(b.value), dtype=torch.uint8, device=self.device)
                n = ctypes.c_longlong()
                N.check(lib.hdr_sample_count(ctypes.byref(self._sensors[k]), s.data_ptr(),
                                             ctypes.byref(n), ws.data_ptr(), st.cuda_stream),
                        "hdr_sample_count")
                counts.append(int(n.value))
                wss.append(ws)
            total = sum(counts)
            dev = self.device
            pos = torch.empty((total, 2), dtype=torch.float64, device=dev)
            ch = torch.empty(total, dtype=torch.uint8, device=dev)
            val = torch.empty(total, dtype=torch.float64, device=dev)
            sig = torch.empty(total, dtype=torch.float64, device=dev)
            ids = torch.empty(total, dtype=torch.int32, device=dev)
            off = 0
            for k, (v, s) in enumerate(planes):
                if counts[k]:
                    N.check(lib.hdr_compact_samples(
                        ctypes.byref(self._sensors[k]), int(self.configs[k].sensor_id),  # :335
                        v.data_ptr(), s.data_ptr(), off, pos.data_ptr(), ch.data_ptr(),
                        val.data_ptr(), sig.data_ptr(), ids.data_ptr(), wss[k].data_ptr(),
                        st.cuda_stream), "hdr_compact_samples")
                off += counts[k]
        return pos, ch, val, sig, ids


class CapturedReconstruction:
    """A reconstruction recorded as a CUDA graph (:meth:`DeviceRig.capture`).
    Replays on the caller's current stream."""

    def __init__(self, graph, out, n_kernels, raws):
        self.graph = graph
        self.out = out
        self.n_kernels = n_kernels  # kernel launches of the library inside the graph
        self.raws = raws            # the frame buffers the graph reads

    def replay(self):
        self.graph.replay()
        return self.out

