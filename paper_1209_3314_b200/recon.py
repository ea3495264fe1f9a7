"""Grayscale morphological reconstruction by dilation on B200
(reference: gridwave/recon.py).

Same entry points, arguments, return types and exceptions as the reference:
``recon_sr``, ``recon_qb``, ``recon_fh``, ``recon_parallel``, ``recon_tiled``
(recon.py:164-342).  The reconstruction has a unique fixed point
(engine.py:9-18), so all five route to one device engine
(libiwpp_b200.so: ``iwpp_recon``) and return bit-identical images; they
differ only in which reference schedule they name.

Inputs may live on the host (numpy, as in the reference) or on the device
(CUDA torch tensors).  Results are returned where the inputs live; inputs
are never mutated (recon.py:63-64, test_recon.py:257-265).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .engine import EngineConfig, RunStats
from .errors import ContractViolation
from .grid import DEVICE_KINDS, SE8, Coord, Image2D, StructuringElement, unpack


@dataclass
class ReconInput:
    """Marker/mask pair plus connectivity (recon.py:37-64).

    Contract: same dimensions, same element kind, marker <= mask pointwise.
    Host arrays are checked on the host like the reference; device tensors
    are checked by a device kernel (``iwpp_check_le``).
    """

    marker: Image2D
    mask: Image2D
    se: StructuringElement = field(default_factory=lambda: SE8)

    def __post_init__(self):
        m, i = self.marker, self.mask
        if m.dims != i.dims:
            raise ContractViolation(f"marker dims {m.dims} != mask dims {i.dims}")
        if m.elem_kind != i.elem_kind:
            raise ContractViolation(
                f"marker kind {m.elem_kind!r} != mask kind {i.elem_kind!r}")
        if m.on_device != i.on_device:
            raise ContractViolation("marker and mask must both be host or both be device arrays")
        if m.on_device:
            if _count_violations(m, i):
                raise ContractViolation("marker exceeds mask somewhere")
        elif not np.all(m.data <= i.data):
            raise ContractViolation("marker exceeds mask somewhere")

    def working_copy(self) -> "ReconInput":
        w = object.__new__(ReconInput)  # already validated: skip __post_init__
        w.marker, w.mask, w.se = self.marker.copy(), self.mask, self.se
        return w


def _count_violations(m: Image2D, i: Image2D) -> int:
    if m.elem_kind not in DEVICE_KINDS:
        return int((m.data > i.data).sum())
    L = _lib.lib()
    n = _lib.ctypes.c_int64(0)
    with _lib.device_of(m.data, i.data):
        ws = _lib.workspace(256)
        _lib.check(L.iwpp_check_le(_lib.ptr(m.data), _lib.ptr(i.data), m.width * m.height,
                                   DEVICE_KINDS[m.elem_kind], _lib.ptr(ws), _lib.ctypes.byref(n),
                                   _lib.stream_ptr()), "check_le")
    return int(n.value)


# ---------------------------------------------------------------------------
# the device engine

ENGINE_AUTO, ENGINE_SMEM, ENGINE_REG, ENGINE_ROUNDS = 0, 1, 2, 3  # iwpp_recon_opts.engine

def _opts(cfg: EngineConfig | None, sweeps: int = -1, tile_sweeps: int = -1,
          halo_sweep_threshold: int = -1, max_blocks: int = 0,
          pipeline_rows: int = 0, engine: int = 0) -> _lib.ReconOpts:
    o = _lib.ReconOpts()
    o.sweeps = sweeps
    o.max_blocks = max_blocks
    o.check_contract = 0
    o.tile_sweeps = tile_sweeps
    o.halo_sweep_threshold = halo_sweep_threshold
    o.pipeline_rows = pipeline_rows
    o.engine = engine
    if cfg is not None and cfg.queue.gbq_capacity is not None:
        o.queue_capacity = int(cfg.queue.gbq_capacity)
    else:
        o.queue_capacity = 0
    return o


def reconstruct(marker, mask, conn: int = 8, cfg: EngineConfig | None = None,
                sweeps: int = -1, stats: dict | None = None, tile_sweeps: int = -1,
                halo_sweep_threshold: int = -1, max_blocks: int = 0, pipeline_rows: int = 0,
                engine: int = 0, kind: str | None = None):
    """Reconstruction of raw arrays (numpy -> numpy, CUDA tensor -> tensor).

    The marker is not modified.  ``stats`` (a dict) receives the device
    counters when given (this synchronizes the stream).  The remaining
    keywords are engine tuning knobs (results never depend on them);
    ``pipeline_rows`` sets the slab height of the host path's transfer /
    compute pipeline (0 = auto, < 0 = off); ``engine`` picks the tile engine
    (0 = auto, 1 = shared-memory queue engine, 2 = register engine on the
    tile queue, 3 = register engine in level-synchronous tile rounds; 2 and 3
    are u8 only).
    ``kind="binary"`` (u8 arrays holding only 0 / 255, grid.py binary) runs
    the one-bit-per-pixel engine.
    """
    L = _lib.lib()
    from .grid import np_dtype_of, is_device_array
    dt = np_dtype_of(marker)
    if is_device_array(marker) != is_device_array(mask):
        raise ContractViolation("marker and mask must both be host or both be device arrays")
    if len(marker.shape) != 2 or tuple(marker.shape) != tuple(mask.shape):
        raise ContractViolation(f"marker shape {tuple(marker.shape)} != mask shape "
                                f"{tuple(mask.shape)} (both must be 2-D)")
    if np_dtype_of(mask) != dt:
        raise ContractViolation(f"marker dtype {dt} != mask dtype {np_dtype_of(mask)}")
    code = {np.dtype(np.uint8): 0, np.dtype(np.uint16): 1, np.dtype(np.int32): 2,
            np.dtype(np.float32): 3}.get(dt)
    if kind == "binary" and code == 0:
        code = 4
    if code is None:
        raise ContractViolation(f"no device engine for dtype {dt}")
    if conn not in (4, 8):
        raise ContractViolation(f"connectivity must be 4 or 8, got {conn}")
    H, W = marker.shape
    st = _lib.Stats()
    sp = _lib.ctypes.byref(st) if stats is not None else None
    opts = _opts(cfg, sweeps, tile_sweeps, halo_sweep_threshold, max_blocks, pipeline_rows,
                 engine)
    with _lib.device_of(marker, mask):
        if is_device_array(marker):
            J = marker.clone()
            I = mask.contiguous()
            nbytes = L.iwpp_recon_workspace_bytes(W, H, code, conn)
            ws = _lib.workspace(nbytes)
            _lib.check(L.iwpp_recon(_lib.ptr(J), _lib.ptr(I), W, H, code, conn, _lib.ptr(ws),
                                    ws.numel(), _lib.ctypes.byref(opts), sp, _lib.stream_ptr()),
                       "recon")
        else:
            m = np.ascontiguousarray(marker)
            i = np.ascontiguousarray(mask)
            J = np.empty_like(m)
            nbytes = L.iwpp_recon_host_workspace_bytes(W, H, code, conn)
            ws = _lib.workspace(nbytes)
            _lib.check(L.iwpp_recon_host(_lib.ptr(J), _lib.ptr(m), _lib.ptr(i), W, H, code, conn,
                                         _lib.ptr(ws), ws.numel(), _lib.ctypes.byref(opts), sp,
                                         _lib.stream_ptr()), "recon")
    if stats is not None:
        stats.update(st.as_dict())
    return J


def _run(inp: ReconInput, cfg: EngineConfig | None = None, sweeps: int = -1) -> Image2D:
    if inp.marker.elem_kind not in DEVICE_KINDS:
        raise ContractViolation(f"no B200 engine for elem_kind {inp.marker.elem_kind!r}")
    want_stats = cfg is not None
    d = {} if want_stats else None
    J = reconstruct(inp.marker.data, inp.mask.data, inp.se.connectivity, cfg, sweeps, d,
                    kind=inp.marker.elem_kind)
    if want_stats:
        cfg.stats.add(d)
    return Image2D(inp.marker.width, inp.marker.height, inp.marker.elem_kind, J)


# ---------------------------------------------------------------------------
# reference entry points (recon.py:164-342)

def recon_sr(inp: ReconInput) -> Image2D:
    """recon.py:164-171 (sweeps to stability) -- same fixed point."""
    return _run(inp)


def recon_fh(inp: ReconInput) -> Image2D:
    """recon.py:174-182 (fast hybrid) -- sweeps + wavefront on the device."""
    return _run(inp)


def recon_qb(inp: ReconInput) -> Image2D:
    """recon.py:185-208 (queue-based from regional maxima) -- same fixed
    point; the device engine seeds itself."""
    return _run(inp)


def recon_parallel(inp: ReconInput, cfg: EngineConfig | None = None) -> Image2D:
    """recon.py:328-342.  ``cfg.stats`` receives the device counters."""
    cfg = cfg or EngineConfig()
    cfg.validate()
    return _run(inp, cfg)


def recon_tiled(inp: ReconInput, tile_dims: tuple[int, int] = (64, 64), cfg=None) -> Image2D:
    """recon.py:308-325.  On one device the tile engine's own 64x64 tiles
    replace ``tile_dims`` (result identical: unique fixed point).  With a
    torch.distributed group initialised, see ``tiles.recon_slabs``."""
    if tile_dims[0] < 1 or tile_dims[1] < 1:
        raise ContractViolation("tile dimensions must be >= 1")
    out = _run(inp)
    if cfg is not None:
        cfg.bp_waves = max(getattr(cfg, "bp_waves", 0), 1)
    return out


# ---------------------------------------------------------------------------
# scan passes / regional maxima (host helpers kept for API parity)

def regional_maxima(img: Image2D, se: StructuringElement = SE8) -> list[Coord]:
    """Cells on plateaus with no strictly greater neighbour, raster order
    (recon.py:211-254).  Host-side helper (not on the hot path)."""
    from scipy import ndimage

    a = img.numpy()
    struct = np.ones((3, 3), bool) if se.connectivity == 8 else \
        np.array([[0, 1, 0], [1, 1, 1], [0, 1, 0]], bool)
    # a plateau is a regional maximum iff none of its cells has a greater
    # neighbour: label equal-valued components, then veto components that
    # touch a greater neighbour
    H, W = a.shape
    greater = np.zeros(a.shape, bool)
    P = np.pad(a, 1, mode="edge")
    for dx, dy in se.offsets:
        nb = P[1 + dy:1 + dy + H, 1 + dx:1 + dx + W]
        valid = np.ones(a.shape, bool)
        if dy < 0:
            valid[0, :] = False
        if dy > 0:
            valid[-1, :] = False
        if dx < 0:
            valid[:, 0] = False
        if dx > 0:
            valid[:, -1] = False
        greater |= valid & (nb > a)
    keep = np.zeros(a.shape, bool)
    for v in np.unique(a):
        lab, k = ndimage.label(a == v, structure=struct)
        if k == 0:
            continue
        bad = np.unique(lab[greater & (lab > 0)])
        ok = np.ones(k + 1, bool)
        ok[0] = False
        ok[bad] = False
        keep |= ok[lab]
    ys, xs = np.nonzero(keep)
    return [Coord(int(x), int(y)) for y, x in zip(ys, xs)]


def seed_scan(J, I, conn: int = 8):
    """Full-neighbourhood active pixels (K.193-217) on the device; returns
    packed indices sorted to raster order."""
    L = _lib.lib()
    torch = _lib._torch()
    from .grid import np_dtype_of, is_device_array
    host = not is_device_array(J)
    dJ = torch.from_numpy(np.ascontiguousarray(J)).cuda() if host else J.contiguous()
    dI = torch.from_numpy(np.ascontiguousarray(I)).cuda() if host else I.contiguous()
    code = DEVICE_KINDS[{np.dtype(np.uint8): "u8", np.dtype(np.uint16): "u16",
                         np.dtype(np.int32): "i32"}[np_dtype_of(J)]]
    H, W = J.shape
    out = torch.empty(max(W * H, 1), dtype=torch.int64, device=dJ.device)
    n = _lib.ctypes.c_int64(0)
    ws = _lib.workspace(256)
    _lib.check(L.iwpp_recon_seed_scan(_lib.ptr(dJ), _lib.ptr(dI), W, H, code, conn,
                                      _lib.ptr(out), _lib.ctypes.byref(n), _lib.ptr(ws),
                                      _lib.stream_ptr()), "seed_scan")
    s = torch.sort(out[:n.value]).values
    return s.cpu().numpy() if host else s


def seeds_as_coords(packed, width: int) -> list[Coord]:
    return [unpack(int(p), width) for p in packed]


RunStats = RunStats
