"""Image file I/O (reference: gridwave/imgio.py:62-162 and 216-228).

Same formats, names, results and errors as the reference:

* ``read_pgm`` -- P2 (ASCII) and P5 (binary), 8- and 16-bit; maxval 1 gives
  a two-level ("binary") image mapped to {0, 255};
* ``write_pgm`` -- P5, maxval 255 for u8/binary, 65535 (big-endian) for u16;
* ``read_f32_raw`` / ``write_f32_raw`` -- raw little-endian float32 plus a
  one-line ``"{w} {h} f32le"`` sidecar;
* ``gen_marker`` -- ``max(mask - h, 0)``.

B200 path: pass ``device=`` (e.g. ``"cuda"``) to the readers and the file
goes into pinned host memory, is copied to HBM as raw bytes and is decoded
there (``iwpp_pgm_decode``: 16-bit byte swap, maxval-1 mapping, the maxval
check).  Writers of device images encode on the device (``iwpp_pgm_encode``)
and copy the payload to pinned memory once.  ``gen_marker`` of a device
image runs ``iwpp_gen_marker``.  Without ``device=`` the readers return
host (numpy) images exactly like the reference.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import ContractViolation, PgmFormatError
from .grid import BG, FG, DEVICE_KINDS, Image2D

_SEP = b" \t\r\n\x0b\x0c"
_SEP_TABLE = np.zeros(256, dtype=bool)
_SEP_TABLE[list(_SEP)] = True


# ---------------------------------------------------------------------------
# PGM header (the reference's token rules, imgio.py:21-59: whitespace and
# '#'-to-end-of-line comments separate tokens; a '#' also ends a token)

class _Scanner:
    def __init__(self, buf):
        self.buf = buf
        self.pos = 0

    def _skip(self):
        b, n = self.buf, len(self.buf)
        while self.pos < n:
            c = b[self.pos]
            if c in _SEP:
                self.pos += 1
            elif c == 35:  # '#': comment to end of line
                while self.pos < n and b[self.pos] not in (10, 13):
                    self.pos += 1
            else:
                return

    def token(self, what: str) -> bytes:
        self._skip()
        b, n = self.buf, len(self.buf)
        if self.pos >= n:
            raise PgmFormatError(f"unexpected end of stream reading {what}", self.pos)
        start = self.pos
        while self.pos < n and b[self.pos] not in _SEP and b[self.pos] != 35:
            self.pos += 1
        return bytes(b[start:self.pos])

    def integer(self, what: str) -> int:
        self._skip()
        start = self.pos
        tok = self.token(what)
        if not tok.isdigit():
            raise PgmFormatError(f"bad {what} token {tok!r}", start)
        return int(tok)


def _parse_header(buf):
    """-> (magic, width, height, maxval, pos after the maxval token)"""
    t = _Scanner(buf)
    magic = t.token("magic")
    if magic not in (b"P2", b"P5"):
        raise PgmFormatError(f"unsupported magic {magic!r}", 0)
    width = t.integer("width")
    height = t.integer("height")
    if width < 1 or height < 1:
        raise PgmFormatError(f"bad dimensions {width}x{height}", t.pos)
    maxval = t.integer("maxval")
    if not 1 <= maxval <= 65535:
        raise PgmFormatError(f"maxval {maxval} out of range", t.pos)
    return magic, width, height, maxval, t.pos


def _kind_of(maxval: int):
    if maxval == 1:
        return "binary", np.uint8
    if maxval <= 255:
        return "u8", np.uint8
    return "u16", np.uint16


def _p2_samples(buf, pos: int, n: int) -> tuple[np.ndarray, int]:
    """The first n ASCII samples after ``pos`` (vectorised token scan).
    Returns (int64 samples, position after the last one).  Errors match the
    reference's sequential reader: the first malformed token among the n,
    else end of stream."""
    body = np.frombuffer(buf, dtype=np.uint8, offset=pos).copy()
    hashes = np.flatnonzero(body == 35)
    if hashes.size:  # blank comments up to the end of their line
        nl = np.flatnonzero((body == 10) | (body == 13))
        ends = np.append(nl, body.size)[np.searchsorted(nl, hashes)]
        d = np.zeros(body.size + 1, dtype=np.int64)
        np.add.at(d, hashes, 1)
        np.add.at(d, ends, -1)
        body[np.cumsum(d)[:-1] > 0] = 32
    sep = _SEP_TABLE[body]
    tok = ~sep
    prev_sep = np.concatenate(([True], sep[:-1]))
    next_sep = np.concatenate((sep[1:], [True]))
    starts = np.flatnonzero(tok & prev_sep)
    ends = np.flatnonzero(tok & next_sep) + 1
    m = min(n, starts.size)
    starts, ends = starts[:m], ends[:m]
    if m:
        lim = ends[-1]
        digit = (body[:lim] >= 48) & (body[:lim] <= 57)
        bad = tok[:lim] & ~digit
        if bad.any():
            first_bad = np.flatnonzero(bad)[0]
            i = int(np.searchsorted(starts, first_bad, side="right")) - 1
            s, e = int(starts[i]), int(ends[i])
            raise PgmFormatError(f"bad sample token {bytes(body[s:e])!r}", pos + s)
    if m < n:
        raise PgmFormatError("unexpected end of stream reading sample", len(buf))
    if not m:
        return np.zeros(0, np.float64), pos
    # value of each token = sum of digit * 10^place, in float64: exact up to
    # 2^53 (far above maxval), and anything larger still compares > maxval
    lim = int(ends[-1])
    is_start = np.zeros(lim, dtype=bool)
    is_start[starts] = True
    tid = np.cumsum(is_start) - 1
    pi = np.flatnonzero(tok[:lim])
    t = tid[pi]
    place = (ends[t] - pi - 1).astype(np.float64)
    with np.errstate(over="ignore"):
        contrib = (body[pi].astype(np.float64) - 48.0) * np.power(10.0, place)
    vals = np.bincount(t, weights=contrib, minlength=m)
    end_pos = pos + lim
    return vals, end_pos


def _p5_extent(buf, pos: int, n: int, per: int) -> int:
    if pos >= len(buf) or buf[pos] not in _SEP:
        raise PgmFormatError("missing separator before raster", pos)
    at = pos + 1
    need = n * per
    if len(buf) - at < need:
        raise PgmFormatError(f"raster truncated: need {need} bytes, have {len(buf) - at}", len(buf))
    return at


def _torch():
    import torch
    return torch


def _pinned_file(path: str):
    """The whole file in a pinned host buffer (torch uint8 tensor)."""
    torch = _torch()
    size = os.path.getsize(path)
    buf = torch.empty(max(size, 1), dtype=torch.uint8, pin_memory=True)
    with open(path, "rb") as f:
        got = f.readinto(memoryview(buf.numpy())[:size]) if size else 0
    return buf[:got]


def read_pgm(path: str, device=None) -> Image2D:
    """Read a P2 or P5 file (imgio.py:62-110).  ``device`` = a CUDA device
    returns a device-resident image decoded in HBM."""
    if device is None:
        with open(path, "rb") as f:
            buf = f.read()
        magic, width, height, maxval, pos = _parse_header(buf)
        kind, dt = _kind_of(maxval)
        n = width * height
        if magic == b"P5":
            per = 1 if maxval <= 255 else 2
            at = _p5_extent(buf, pos, n, per)
            raw = buf[at:at + n * per]
            data = (np.frombuffer(raw, dtype=np.uint8) if per == 1
                    else np.frombuffer(raw, dtype=">u2").astype(np.uint16))
            end = pos
        else:
            data, end = _p2_samples(buf, pos, n)
        if data.max(initial=0) > maxval:
            raise PgmFormatError(f"sample exceeds maxval {maxval}", end)
        img = data.astype(np.int64).reshape(height, width)
        if kind == "binary":
            img = np.where(img != 0, FG, BG)
        return Image2D(width, height, kind, np.ascontiguousarray(img.astype(dt)))
    return _read_pgm_device(path, device)


def _read_pgm_device(path: str, device) -> Image2D:
    from . import _lib
    torch = _torch()
    dev = torch.device(device)
    if dev.type != "cuda":
        raise ContractViolation(f"device reads need a CUDA device, got {device!r}")
    if not os.path.exists(path):  # a missing file is a contract error, device or not
        raise FileNotFoundError(path)
    L = _lib.lib()
    pinned = _pinned_file(path)
    hb = pinned.numpy()
    # the header is short: scan a prefix, the whole buffer for P2 bodies
    magic, width, height, maxval, pos = _parse_header(memoryview(hb))
    kind, dt = _kind_of(maxval)
    n = width * height
    tdt = torch.uint8 if dt == np.uint8 else torch.uint16
    with torch.cuda.device(dev):
        out = torch.empty((height, width), dtype=tdt, device=dev)
        if magic == b"P5":
            per = 1 if maxval <= 255 else 2
            at = _p5_extent(memoryview(hb), pos, n, per)
            raw = torch.empty(n * per, dtype=torch.uint8, device=dev)
            raw.copy_(pinned[at:at + n * per], non_blocking=True)
            mx = ctypes.c_int64(0)
            ws = _lib.workspace(256)
            _lib.check(L.iwpp_pgm_decode(_lib.ptr(out), _lib.ptr(raw), n, per,
                                         1 if kind == "binary" else 0, _lib.ptr(ws),
                                         ctypes.byref(mx), _lib.stream_ptr()), "read_pgm")
            if mx.value > maxval:
                raise PgmFormatError(f"sample exceeds maxval {maxval}", pos)
        else:
            vals, end = _p2_samples(hb.tobytes(), pos, n)
            if vals.max(initial=0) > maxval:
                raise PgmFormatError(f"sample exceeds maxval {maxval}", end)
            if kind == "binary":
                vals = np.where(vals != 0, FG, BG)
            out.copy_(torch.from_numpy(np.ascontiguousarray(vals.astype(dt)).reshape(height, width)))
    return Image2D(width, height, kind, out)


def _atomic_write(path: str, chunks) -> None:
    tmp = path + ".tmp"
    with open(tmp, "wb") as f:
        for c in chunks:
            f.write(c)
    os.replace(tmp, path)


def _device_payload(img: Image2D, per: int) -> memoryview:
    """Device image -> its P5 payload bytes in pinned host memory."""
    from . import _lib
    torch = _torch()
    L = _lib.lib()
    n = img.width * img.height
    src = img.data.contiguous()
    with torch.cuda.device(src.device):
        if per == 2:
            raster = torch.empty(2 * n, dtype=torch.uint8, device=src.device)
            _lib.check(L.iwpp_pgm_encode(_lib.ptr(raster), _lib.ptr(src), n, 2,
                                         _lib.stream_ptr()), "write_pgm")
        else:
            raster = src.view(torch.uint8).reshape(-1)
        host = torch.empty(raster.numel(), dtype=torch.uint8, pin_memory=True)
        host.copy_(raster)
    return memoryview(host.numpy())


def write_pgm(img: Image2D, path: str) -> None:
    """Write a P5 file (imgio.py:113-130): maxval 255 for u8/binary, 65535
    (big-endian) for u16.  Float and int32 images have no PGM form."""
    if img.elem_kind == "f32":
        raise ContractViolation("f32 images cannot be written as PGM")
    if img.elem_kind == "i32":
        raise ContractViolation("i32 images cannot be written as PGM")
    maxval = 65535 if img.elem_kind == "u16" else 255
    header = f"P5\n{img.width} {img.height}\n{maxval}\n".encode()
    if img.on_device:
        payload = _device_payload(img, 2 if maxval == 65535 else 1)
    elif maxval == 65535:
        payload = img.data.astype(">u2").tobytes()
    else:
        payload = img.data.astype(np.uint8).tobytes()
    _atomic_write(path, (header, payload))


# ---------------------------------------------------------------------------
# raw float maps (imgio.py:136-162)

def write_f32_raw(img: Image2D, path: str) -> None:
    """Raw little-endian float32, row-major, plus ``path + '.hdr'`` holding
    ``'{width} {height} f32le'``."""
    if img.elem_kind != "f32":
        raise ContractViolation("write_f32_raw requires an f32 image")
    if img.on_device:
        torch = _torch()
        host = torch.empty(img.width * img.height, dtype=torch.float32, pin_memory=True)
        host.copy_(img.data.reshape(-1))
        payload = memoryview(host.numpy()).cast("B")
    else:
        payload = img.data.astype("<f4").tobytes()
    _atomic_write(path, (payload,))
    with open(path + ".hdr", "w") as f:
        f.write(f"{img.width} {img.height} f32le\n")


def read_f32_raw(path: str, device=None) -> Image2D:
    with open(path + ".hdr") as f:
        fields = f.read().split()
    if len(fields) != 3 or fields[2] != "f32le":
        raise ContractViolation(f"unrecognized raw float header {fields!r}")
    w, h = int(fields[0]), int(fields[1])
    if device is None:
        raw = np.fromfile(path, dtype="<f4")
        if raw.size != w * h:
            raise ContractViolation(f"raw float file holds {raw.size} samples, header says {w * h}")
        return Image2D(w, h, "f32", np.ascontiguousarray(raw.astype(np.float32).reshape(h, w)))
    torch = _torch()
    dev = torch.device(device)
    pinned = _pinned_file(path)
    count = pinned.numel() // 4
    if count != w * h:
        raise ContractViolation(f"raw float file holds {count} samples, header says {w * h}")
    out = torch.empty((h, w), dtype=torch.float32, device=dev)
    out.view(torch.uint8).reshape(-1).copy_(pinned[:4 * count])
    return Image2D(w, h, "f32", out)


# ---------------------------------------------------------------------------
# markers (imgio.py:216-228)

def gen_marker(mask: Image2D, h: int) -> Image2D:
    """Marker for h-reconstruction: max(mask - h, 0) per cell, for the
    integer and float kinds (not binary)."""
    if mask.elem_kind == "binary":
        raise ContractViolation("h-marker is undefined for binary images")
    if h < 0:
        raise ContractViolation("h must be >= 0")
    if mask.on_device:
        from . import _lib
        torch = _torch()
        L = _lib.lib()
        src = mask.data.contiguous()
        out = torch.empty_like(src)
        with torch.cuda.device(src.device):
            _lib.check(L.iwpp_gen_marker(_lib.ptr(out), _lib.ptr(src), src.numel(),
                                         DEVICE_KINDS[mask.elem_kind], float(h),
                                         _lib.stream_ptr()), "gen_marker")
        return Image2D(mask.width, mask.height, mask.elem_kind, out)
    a = mask.data
    if mask.elem_kind == "f32":
        out = np.maximum(a - np.float32(h), np.float32(0)).astype(np.float32)
    else:
        out = np.maximum(a.astype(np.int64) - h, 0).astype(a.dtype)
    return Image2D(mask.width, mask.height, mask.elem_kind, out)


def quantize_distance(dist: Image2D) -> Image2D:
    """The CLI's quantized distance view (cli.py:98-101): nearest integer
    (half to even), saturating at 255, as u8."""
    if dist.elem_kind != "f32":
        raise ContractViolation("quantize_distance requires an f32 image")
    if dist.on_device:
        from . import _lib
        torch = _torch()
        L = _lib.lib()
        src = dist.data.contiguous()
        out = torch.empty(src.shape, dtype=torch.uint8, device=src.device)
        with torch.cuda.device(src.device):
            _lib.check(L.iwpp_quantize_u8(_lib.ptr(out), _lib.ptr(src), src.numel(),
                                          _lib.stream_ptr()), "quantize")
        return Image2D(dist.width, dist.height, "u8", out)
    q = np.minimum(np.rint(dist.data), 255).astype(np.uint8)
    return Image2D(dist.width, dist.height, "u8", q)
