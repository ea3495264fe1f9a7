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
from .engine import EngineConfig, PropagationRule, RunStats
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


class ReconRule(PropagationRule):
    """The reconstruction rule (recon.py:67-128) over packed indices: p
    raises neighbour q to min(J(p), I(q)) when J(q) < J(p) and q is below
    its mask.  ``tiles.run_pipeline`` runs it on the device tile engine;
    the per-cell hooks below state the rule for host-side inspection and
    small checks (numpy arrays)."""

    def __init__(self, J, I, se: StructuringElement, bounds=None):
        h, w = J.shape
        super().__init__(w, h, se, bounds)
        self.J, self.I = J, I

    def read(self, q):
        return self.J.reshape(-1)[q]

    def write(self, q, value):
        self.J.reshape(-1)[q] = value

    def condition(self, p, q):
        Jf, If = self.J.reshape(-1), self.I.reshape(-1)
        return Jf[q] < Jf[p] and If[q] != Jf[q]

    def propose(self, p, q):
        return min(self.J.reshape(-1)[p], self.I.reshape(-1)[q])

    def improves(self, q, old, new):
        return old < new

    def condition_from(self, v, p, q):
        Jf, If = self.J.reshape(-1), self.I.reshape(-1)
        return Jf[q] < v and If[q] != Jf[q]

    def propose_from(self, v, p, q):
        return min(v, self.I.reshape(-1)[q])

    def rebound(self, bounds) -> "ReconRule":
        return ReconRule(self.J, self.I, self.se, bounds)


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
          pipeline_rows: int = 0, engine: int = 0,
          max_rounds: int | None = None) -> _lib.ReconOpts:
    o = _lib.ReconOpts()
    # EngineConfig.max_rounds (engine.py:311-317): the level-synchronous
    # tile-rounds engine counts rounds; EngineError past the cap
    o.max_rounds = -1 if max_rounds is None else int(max_rounds)
    if max_rounds is not None and engine == ENGINE_AUTO:
        engine = ENGINE_ROUNDS
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
                engine: int = 0, kind: str | None = None, max_rounds: int | None = None):
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
                 engine, max_rounds)
    with _lib.device_of(marker, mask):
        if is_device_array(marker):
            M = marker.contiguous()
            J = M.new_empty(M.shape)
            opts.marker = _lib.ptr(M)  # copied into J by the engine (not modified)
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
                    kind=inp.marker.elem_kind,
                    max_rounds=cfg.max_rounds if cfg is not None else None)
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
    """recon.py:308-325: the rule over the pipeline (``tiles.run_pipeline``)
    on a working copy of the marker.  One device: the tile engine's own
    32x32 tiles replace ``tile_dims`` (result identical: unique fixed point,
    tiles.py:7-9).  Under an initialised torch.distributed group (one rank
    per GPU, every rank passing the full image) the pipeline runs as
    horizontal slabs, one per rank, with border-row exchange waves
    (``distributed.recon_slabs``); every rank returns the full result."""
    from .tiles import run_pipeline

    if inp.marker.elem_kind not in DEVICE_KINDS:
        raise ContractViolation(f"no B200 engine for elem_kind {inp.marker.elem_kind!r}")
    work = inp.working_copy()
    rule = ReconRule(work.marker.data, work.mask.data, work.se)
    rule.elem_kind = work.marker.elem_kind
    run_pipeline(work.marker, rule, lambda: None, tile_dims, cfg)
    return work.marker


# ---------------------------------------------------------------------------
# the reference's individual scan passes (recon.py:134-161, 260-305) on the
# device, cell for cell (libiwpp_b200.so: iwpp_recon_pass)

PASS_RASTER, PASS_ANTIRASTER, PASS_ROWS_FWD, PASS_COLS_FWD, PASS_ROWS_BWD, PASS_COLS_BWD = range(6)
_PASS_CODES = {np.dtype(np.uint8): 0, np.dtype(np.uint16): 1, np.dtype(np.int32): 2,
               np.dtype(np.float32): 3}


def _run_pass(J, I, conn: int, pas: int, collect: bool = False):
    """One pass in place on J (numpy or CUDA tensor); returns (changed,
    seeds or None) with seeds packed y*W+x in the order the sweep met them."""
    from .grid import np_dtype_of, is_device_array
    L = _lib.lib()
    torch = _lib._torch()
    code = _PASS_CODES.get(np_dtype_of(J))
    if code is None:
        raise ContractViolation(f"no device pass for dtype {np_dtype_of(J)}")
    H, W = J.shape
    host = not is_device_array(J)
    with _lib.device_of(J, I):
        dJ = torch.from_numpy(np.ascontiguousarray(J)).cuda() if host else J
        dI = torch.from_numpy(np.ascontiguousarray(I)).cuda() if host else I.contiguous()
        work = dJ if dJ.is_contiguous() else dJ.contiguous()
        seeds = torch.empty(max(W * H, 1) if collect else 1, dtype=torch.int64, device=work.device)
        n = _lib.ctypes.c_int64(0)
        ch = _lib.ctypes.c_int(0)
        ws = _lib.workspace(L.iwpp_recon_pass_workspace_bytes(W, H, code))
        _lib.check(L.iwpp_recon_pass(_lib.ptr(work), _lib.ptr(dI), W, H, code, conn, pas,
                                     _lib.ptr(seeds) if collect else None, _lib.ctypes.byref(n),
                                     _lib.ctypes.byref(ch), _lib.ptr(ws), _lib.stream_ptr()),
                   "recon_pass")
        if work is not dJ:
            dJ.copy_(work)
        if host:
            J[...] = dJ.cpu().numpy()
    out = seeds[:n.value] if collect else None
    if collect and host:
        out = out.cpu().numpy()
    return bool(ch.value), out


def raster_pass(inp: ReconInput) -> bool:
    """recon.py:134-139 (K.38-74): one in-place top-left to bottom-right
    sweep of inp.marker; returns whether any cell changed."""
    return _run_pass(inp.marker.data, inp.mask.data, inp.se.connectivity, PASS_RASTER)[0]


def _antiraster_packed(inp: ReconInput, collect_seeds: bool):
    """recon.py:151-161: (changed, packed seeds) of the mirror sweep."""
    ch, seeds = _run_pass(inp.marker.data, inp.mask.data, inp.se.connectivity, PASS_ANTIRASTER,
                          collect_seeds)
    if seeds is None:
        seeds = np.empty(0, np.int64)
    return ch, seeds


def antiraster_pass(inp: ReconInput, collect_seeds: bool = False):
    """recon.py:142-148 (K.77-112): the bottom-right to top-left sweep;
    returns (changed, seeds as Coord) -- the cells that may still raise a
    scan-order successor, in the order the sweep met them (empty unless
    requested)."""
    ch, packed = _antiraster_packed(inp, collect_seeds)
    w = inp.marker.width
    seq = packed.tolist() if not isinstance(packed, np.ndarray) else packed
    return ch, [unpack(int(p), w) for p in seq]


def parallel_sweeps(J, I, se: StructuringElement, n_workers: int = 1, pool=None,
                    bounds=None) -> None:
    """recon.py:275-305: rows forward, columns forward, rows backward,
    columns backward (K.115-190), in place on J.  With several bands the
    reference's diagonal reads race across band edges (results vary with
    timing, recon.py:280-286); the device runs the single-band order, one of
    those outcomes, exactly.  ``bounds`` = (x0, y0, x1, y1) restricts the
    sweeps to a window (neighbours outside it are not read)."""
    if n_workers < 1:
        raise ContractViolation("n_workers must be >= 1")
    H, W = J.shape
    x0, y0, x1, y1 = bounds if bounds is not None else (0, 0, W, H)
    win = (x0, y0, x1, y1) != (0, 0, W, H)
    Jw, Iw = (J[y0:y1, x0:x1], I[y0:y1, x0:x1]) if win else (J, I)
    if win:
        Jw = Jw.copy() if isinstance(Jw, np.ndarray) else Jw.contiguous()
    for pas in (PASS_ROWS_FWD, PASS_COLS_FWD, PASS_ROWS_BWD, PASS_COLS_BWD):
        _run_pass(Jw, Iw, se.connectivity, pas)
    if win:
        J[y0:y1, x0:x1] = Jw


# ---------------------------------------------------------------------------
# regional maxima (host helper kept for API parity)

def regional_maxima(img: Image2D, se: StructuringElement = SE8) -> list[Coord]:
    """Cells on plateaus with no strictly greater neighbour, raster order
    (recon.py:211-254).  Host-side helper (not on the hot path).

    One pass for every value at once: the equal-valued neighbour pairs are
    the edges of a graph whose connected components are the plateaus
    (scipy.sparse.csgraph), and a plateau is vetoed iff one of its cells
    has a strictly greater neighbour -- O(pixels), whatever the number of
    distinct values."""
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components

    a = img.numpy()
    H, W = a.shape
    n = H * W
    idx = np.arange(n, dtype=np.int64).reshape(H, W)
    greater = np.zeros(a.shape, bool)
    src, dst = [], []
    for dx, dy in se.offsets:
        # cells p whose neighbour p + (dx, dy) lies on the image
        ys = slice(max(0, -dy), H - max(0, dy))
        xs = slice(max(0, -dx), W - max(0, dx))
        nys = slice(max(0, dy), H - max(0, -dy))
        nxs = slice(max(0, dx), W - max(0, -dx))
        c, nb = a[ys, xs], a[nys, nxs]
        greater[ys, xs] |= nb > c
        eq = c == nb
        src.append(idx[ys, xs][eq])
        dst.append(idx[nys, nxs][eq])
    src = np.concatenate(src) if src else np.zeros(0, np.int64)
    dst = np.concatenate(dst) if dst else np.zeros(0, np.int64)
    g = coo_matrix((np.ones(src.size, np.int8), (src, dst)), shape=(n, n))
    k, lab = connected_components(g, directed=False)
    vetoed = np.bincount(lab, weights=greater.ravel(), minlength=k) > 0
    keep = ~vetoed[lab]
    ys, xs = np.divmod(np.nonzero(keep)[0], W)
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
