"""Raster I/O for rigs and results (reference formats: pkg/src/hdrfuse/pnm.py).

* 16-bit binary PGM (``P5``, big-endian samples, maxval 256..65535, ``#``
  comments in the header) for raw CFA frames;
* PFM (``Pf`` grey / ``PF`` RGB, scale sign = endianness, rows stored
  bottom-up) for calibration planes and HDR results.
"""

from __future__ import annotations

import os
from typing import Union

import numpy as np

from .bayer import BayerPattern
from .images import CFAImage, FloatFrame, HDRImage


class PnmParseError(ValueError):
    """Malformed PGM/PFM input (with the byte offset where parsing stopped)."""

    def __init__(self, message, offset=None):
        super().__init__(message if offset is None else f"{message} (byte offset {offset})")
        self.offset = offset


def _header_tokens(buf: bytes, count: int, comments: bool):
    """First ``count`` whitespace-separated tokens; returns (tokens, end offset).
    Exactly one whitespace byte must follow the last token."""
    toks, i, n = [], 0, len(buf)
    while len(toks) < count:
        while i < n and (buf[i:i + 1].isspace() or (comments and buf[i:i + 1] == b"#")):
            if buf[i:i + 1] == b"#":
                j = buf.find(b"\n", i)
                i = n if j < 0 else j + 1
            else:
                i += 1
        j = i
        while j < n and not buf[j:j + 1].isspace():
            j += 1
        if j == i:
            raise PnmParseError("truncated header", i)
        toks.append(buf[i:j])
        i = j
    if i >= n or not buf[i:i + 1].isspace():
        raise PnmParseError("missing whitespace after header", i)
    return toks, i + 1


def read_pgm16(path: Union[str, os.PathLike], pattern: BayerPattern = BayerPattern.RGGB) -> CFAImage:
    buf = open(path, "rb").read()
    if buf[:2] != b"P5":
        raise PnmParseError(f"unsupported magic {buf[:2]!r}, expected P5", 0)
    toks, off = _header_tokens(buf, 4, True)
    try:
        w, h, maxval = int(toks[1]), int(toks[2]), int(toks[3])
    except ValueError:
        raise PnmParseError("non-integer header field", 2) from None
    if w <= 0 or h <= 0:
        raise PnmParseError(f"invalid dimensions {w}x{h}", off)
    if not 256 <= maxval <= 65535:
        raise PnmParseError(f"maxval {maxval} out of range for 16-bit PGM", off)
    need = w * h * 2
    if len(buf) - off < need:
        raise PnmParseError(f"payload has {len(buf) - off} bytes, expected {need}", off)
    data = np.frombuffer(buf, dtype=">u2", count=w * h, offset=off).astype(np.uint16).reshape(h, w)
    if data.size and int(data.max()) > maxval:
        raise PnmParseError(f"sample value {int(data.max())} exceeds maxval {maxval}", off)
    return CFAImage(data, max(8, int(maxval).bit_length()), pattern)


def write_pgm16(img: CFAImage, path: Union[str, os.PathLike]) -> None:
    data = np.asarray(img.data, dtype=np.uint16)
    maxval = (1 << int(img.bit_depth)) - 1
    if maxval < 256:
        raise ValueError("16-bit PGM needs bit_depth >= 9")
    with open(path, "wb") as f:
        f.write(f"P5\n{data.shape[1]} {data.shape[0]}\n{maxval}\n".encode())
        f.write(data.astype(">u2").tobytes())


def read_pfm(path: Union[str, os.PathLike]):
    buf = open(path, "rb").read()
    magic = buf[:2]
    if magic not in (b"PF", b"Pf"):
        raise PnmParseError(f"unsupported magic {magic!r}, expected PF or Pf", 0)
    toks, off = _header_tokens(buf, 4, False)
    try:
        w, h, scale = int(toks[1]), int(toks[2]), float(toks[3])
    except ValueError:
        raise PnmParseError("invalid PFM header", 2) from None
    if w <= 0 or h <= 0:
        raise PnmParseError(f"invalid dimensions {w}x{h}", off)
    if scale == 0 or not np.isfinite(scale):
        raise PnmParseError(f"invalid scale {scale}", off)
    ch = 3 if magic == b"PF" else 1
    need = w * h * ch * 4
    if len(buf) - off < need:
        raise PnmParseError(f"payload has {len(buf) - off} bytes, expected {need}", off)
    dt = "<f4" if scale < 0 else ">f4"
    data = np.frombuffer(buf, dtype=dt, count=w * h * ch, offset=off).astype(np.float32)
    data = data.reshape(h, w, ch)[::-1]  # bottom-up on disk
    if ch == 3:
        return HDRImage(np.ascontiguousarray(data))
    return FloatFrame(np.ascontiguousarray(data[:, :, 0]).astype(np.float64))


def write_pfm(img, path: Union[str, os.PathLike]) -> None:
    data = np.asarray(getattr(img, "data", img))
    if data.ndim == 2:
        magic, arr = "Pf", data[:, :, None]
    elif data.ndim == 3 and data.shape[2] == 3:
        magic, arr = "PF", data
    else:
        raise ValueError(f"cannot write array of shape {data.shape} as PFM")
    h, w = arr.shape[:2]
    with open(path, "wb") as f:
        f.write(f"{magic}\n{w} {h}\n-1.0\n".encode())
        f.write(np.ascontiguousarray(arr[::-1]).astype("<f4").tobytes())
