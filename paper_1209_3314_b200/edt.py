"""Euclidean distance transform by nearest-source propagation on B200
(reference: gridwave/edt.py).

The reference pins one canonical schedule: two-phase rounds in which every
offer uses the source its sender held at the start of the round, and a
cell adopts a source iff it is strictly closer or equally close from a
smaller packed index (edt.py:1-14, K.320-336, K.403-433).  The device
engine (libiwpp_b200.so: ``iwpp_edt``) runs exactly that schedule --
level-synchronous rounds with a grid barrier -- so source maps, squared
distances and float32 distances are bit-identical to the reference.
``mode="sequential"`` and ``mode="parallel"`` therefore give the same
result here as they do in the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .engine import EngineConfig, PropagationRule
from .errors import ContractViolation, NoBackgroundError
from .grid import SE8, Coord, Image2D, StructuringElement, is_device_array, pack, unpack

#: squared distance reported for cells without a source (K.19)
FAR = 1 << 62
#: source-map sentinel for "no source yet" (edt.py:40-42)
INF = -1


@dataclass
class VoronoiMap:
    """Per-cell packed index of the nearest background cell (edt.py:45-80).
    ``vr`` is int64 (height, width), numpy or CUDA tensor; INF = -1."""

    width: int
    height: int
    vr: object

    @property
    def dims(self):
        return self.width, self.height

    @property
    def on_device(self) -> bool:
        return is_device_array(self.vr)

    def copy(self) -> "VoronoiMap":
        return VoronoiMap(self.width, self.height,
                          self.vr.clone() if self.on_device else self.vr.copy())

    def source(self, p: Coord) -> Coord | None:
        v = int(self.vr[p[1], p[0]])
        return None if v == INF else unpack(v, self.width)

    def squared_distances(self):
        """Exact int64 squared distances, FAR where unassigned (device
        kernel; returns the same residency as ``vr``)."""
        L = _lib.lib()
        torch = _lib._torch()
        host = not self.on_device
        with _lib.device_of(self.vr):
            vr = torch.from_numpy(np.ascontiguousarray(self.vr)).cuda() if host else self.vr.contiguous()
            d2 = torch.empty_like(vr)
            ws = _lib.workspace(256)
            rc = L.iwpp_edt_finalize(_lib.ptr(vr), self.width, self.height, None, _lib.ptr(d2),
                                     _lib.ptr(ws), _lib.stream_ptr())
        if rc not in (_lib.IWPP_OK, _lib.IWPP_E_NO_BACKGROUND):
            _lib.check(rc, "squared_distances")
        return d2.cpu().numpy() if host else d2


class DistanceRule(PropagationRule):
    """Source adoption (edt.py:83-153): p offers its source to q; q takes it
    when strictly closer, or equally close from a smaller packed index
    (K.320-336).  Synchronous: offers use the round-start sources.
    ``tiles.run_pipeline`` runs it on the device round engine; the hooks
    below state the rule for host-side inspection (numpy ``vr``)."""

    synchronous = True

    def __init__(self, vr, se: StructuringElement, bounds=None):
        h, w = vr.shape
        super().__init__(w, h, se, bounds)
        self.vr = vr

    def sqdist(self, q: int, src: int) -> int:
        if src < 0:
            return FAR
        w = self.width
        return (q % w - src % w) ** 2 + (q // w - src // w) ** 2

    def closer(self, q: int, cand: int, held: int) -> bool:
        if cand < 0:
            return False
        if held < 0:
            return True
        dc, dh = self.sqdist(q, cand), self.sqdist(q, held)
        return dc < dh or (dc == dh and cand < held)

    def read(self, q):
        return int(self.vr.reshape(-1)[q])

    def write(self, q, value):
        self.vr.reshape(-1)[q] = value

    def condition(self, p, q):
        return self.closer(q, self.read(p), self.read(q))

    def propose(self, p, q):
        return self.read(p)

    def improves(self, q, old, new):
        return self.closer(q, int(new), int(old))

    def condition_from(self, v, p, q):
        return self.closer(q, int(v), self.read(q))

    def propose_from(self, v, p, q):
        return int(v)

    def rebound(self, bounds) -> "DistanceRule":
        return DistanceRule(self.vr, self.se, bounds)


def _require_binary(mask: Image2D):
    if mask.elem_kind != "binary":
        raise ContractViolation(
            f"distance transform needs a binary mask, got {mask.elem_kind!r}")


def _conn(se: StructuringElement) -> int:
    return se.connectivity


def _max_rounds(cfg: EngineConfig | None, mode: str) -> int:
    # the reference applies max_rounds only through run_parallel
    if mode == "parallel" and cfg is not None and cfg.max_rounds is not None:
        return int(cfg.max_rounds)
    return -1


def _check_mode(mode: str):
    if mode not in ("sequential", "parallel"):
        raise ContractViolation(f"unknown mode {mode!r}")


def _edt_arrays(mask, conn: int, max_rounds: int = -1, stats: dict | None = None,
                want_dist: bool = True):
    """(vr, dist, status) for a raw mask (numpy -> numpy, tensor -> tensor)."""
    L = _lib.lib()
    H, W = mask.shape
    st = _lib.Stats()
    with _lib.device_of(mask):
        vr, dist, rc = _edt_arrays_on(L, mask, W, H, conn, max_rounds, st, want_dist)
    if stats is not None:
        stats.update(st.as_dict())
    return vr, dist, rc


def _edt_arrays_on(L, mask, W, H, conn, max_rounds, st, want_dist):
    if is_device_array(mask):
        torch = _lib._torch()
        m = mask.contiguous()
        vr = torch.empty((H, W), dtype=torch.int64, device=m.device)
        dist = torch.empty((H, W), dtype=torch.float32, device=m.device) if want_dist else None
        ws = _lib.workspace(L.iwpp_edt_workspace_bytes(W, H, conn))
        rc = L.iwpp_edt(_lib.ptr(m), W, H, conn, _lib.ptr(vr),
                        _lib.ptr(dist) if dist is not None else None, _lib.ptr(ws), ws.numel(),
                        max_rounds, _lib.ctypes.byref(st), _lib.stream_ptr())
    else:
        m = np.ascontiguousarray(mask, dtype=np.uint8)
        vr = np.empty((H, W), np.int64)
        dist = np.empty((H, W), np.float32) if want_dist else None
        ws = _lib.workspace(L.iwpp_edt_host_workspace_bytes(W, H, conn))
        rc = L.iwpp_edt_host(_lib.ptr(m), W, H, conn, _lib.ptr(vr),
                             _lib.ptr(dist) if dist is not None else None, _lib.ptr(ws),
                             ws.numel(), max_rounds, _lib.ctypes.byref(st), _lib.stream_ptr())
    return vr, dist, rc


def edt(mask: Image2D, se: StructuringElement = SE8, mode: str = "sequential",
        cfg: EngineConfig | None = None):
    """edt.py:284-294: init, propagate, finalize -> (VoronoiMap, f32 Image2D).
    Raises NoBackgroundError on an all-foreground mask."""
    _require_binary(mask)
    _check_mode(mode)
    if cfg is not None:
        cfg.validate()
    d = {}
    vr, dist, rc = _edt_arrays(mask.data, _conn(se), _max_rounds(cfg, mode), d)
    if cfg is not None and mode == "parallel":
        cfg.stats.add(d)
    _lib.check(rc, "edt")
    return (VoronoiMap(mask.width, mask.height, vr),
            Image2D(mask.width, mask.height, "f32", dist))


def init_packed(mask: Image2D, se: StructuringElement = SE8):
    """edt.py:187-196: (VoronoiMap, packed contour seeds in raster order).
    Device kernels (``iwpp_edt_init``): K.edt_assign + K.edt_contour_seeds."""
    _require_binary(mask)
    L = _lib.lib()
    torch = _lib._torch()
    host = not mask.on_device
    H, W = mask.height, mask.width
    with _lib.device_of(mask.data):
        m = torch.from_numpy(np.ascontiguousarray(mask.data)).cuda() if host else mask.data.contiguous()
        vr = torch.empty((H, W), dtype=torch.int64, device=m.device)
        seeds = torch.empty(H * W, dtype=torch.int64, device=m.device)
        n = _lib.ctypes.c_int64(0)
        ws = _lib.workspace(L.iwpp_edt_init_workspace_bytes(W, H))
        _lib.check(L.iwpp_edt_init(_lib.ptr(m), W, H, se.connectivity, _lib.ptr(vr), _lib.ptr(seeds),
                                   _lib.ctypes.byref(n), _lib.ptr(ws), ws.numel(), _lib.stream_ptr()),
                   "edt_init")
        seeds = seeds[:n.value]
        if host:
            return VoronoiMap(W, H, vr.cpu().numpy()), seeds.cpu().numpy()
    return VoronoiMap(W, H, vr), seeds


def edt_init(mask: Image2D, se: StructuringElement = SE8):
    """edt.py:199-202: as init_packed with seeds as coordinate pairs."""
    vmap, seeds = init_packed(mask, se)
    s = seeds.tolist() if not isinstance(seeds, np.ndarray) else seeds
    return vmap, [unpack(int(p), mask.width) for p in s]


def _norm_seeds(seeds, width: int) -> np.ndarray:
    if isinstance(seeds, np.ndarray):
        return seeds.astype(np.int64)
    if is_device_array(seeds):
        return seeds
    out = np.empty(len(seeds), dtype=np.int64)
    for i, s in enumerate(seeds):
        out[i] = pack(s[0], s[1], width) if isinstance(s, (tuple, Coord)) else int(s)
    return out


def edt_propagate(vmap: VoronoiMap, seeds, se: StructuringElement = SE8,
                  mode: str = "sequential", cfg: EngineConfig | None = None) -> VoronoiMap:
    """edt.py:248-269: propagate to the fixed point, in place on ``vmap``."""
    _check_mode(mode)
    if cfg is not None:
        cfg.validate()
    L = _lib.lib()
    torch = _lib._torch()
    W, H = vmap.width, vmap.height
    packed = _norm_seeds(seeds, W)
    host = not vmap.on_device
    with _lib.device_of(vmap.vr, packed):
        vr = torch.from_numpy(np.ascontiguousarray(vmap.vr)).cuda() if host else vmap.vr
        dev = vr.device
        sd = torch.as_tensor(packed, dtype=torch.int64).to(dev) if not is_device_array(packed) \
            else packed.to(torch.int64).contiguous()
        n = sd.numel()
        if n == 0:
            sd = torch.zeros(1, dtype=torch.int64, device=dev)
        st = _lib.Stats()
        ws = _lib.workspace(L.iwpp_edt_workspace_bytes(W, H, se.connectivity))
        rc = L.iwpp_edt_propagate(_lib.ptr(vr), W, H, se.connectivity, _lib.ptr(sd), n,
                                  _lib.ptr(ws), ws.numel(), _max_rounds(cfg, mode),
                                  _lib.ctypes.byref(st), _lib.stream_ptr())
        if cfg is not None and mode == "parallel":
            cfg.stats.add(st.as_dict())
        _lib.check(rc, "edt_propagate")
        if host:
            vmap.vr[...] = vr.cpu().numpy()
    return vmap


def finalize_distance_map(vmap: VoronoiMap) -> Image2D:
    """edt.py:272-281: float32(sqrt(float64(d2))); NoBackgroundError if any
    cell still holds INF."""
    L = _lib.lib()
    torch = _lib._torch()
    host = not vmap.on_device
    with _lib.device_of(vmap.vr):
        vr = torch.from_numpy(np.ascontiguousarray(vmap.vr)).cuda() if host else vmap.vr.contiguous()
        dist = torch.empty(vr.shape, dtype=torch.float32, device=vr.device)
        ws = _lib.workspace(256)
        rc = L.iwpp_edt_finalize(_lib.ptr(vr), vmap.width, vmap.height, _lib.ptr(dist), None,
                                 _lib.ptr(ws), _lib.stream_ptr())
    if rc == _lib.IWPP_E_NO_BACKGROUND:
        raise NoBackgroundError("no background reachable: distance map undefined")
    _lib.check(rc, "finalize_distance_map")
    return Image2D(vmap.width, vmap.height, "f32", dist.cpu().numpy() if host else dist)


def edt_tiled(mask: Image2D, se: StructuringElement = SE8,
              tile_dims: tuple[int, int] = (64, 64), cfg=None):
    """edt.py:297-310: the rule over the pipeline (``tiles.run_pipeline``),
    cell-for-cell identical to the untiled modes.  One device: init +
    device rounds.  Under an initialised torch.distributed group (one rank
    per GPU, every rank passing the full mask) the rounds run as horizontal
    slabs with one boundary-row exchange per round
    (``distributed.edt_slabs``); every rank returns the full result."""
    from .tiles import PipelineConfig, _dist_world, partition, run_pipeline

    _require_binary(mask)
    world, _ = _dist_world()
    if world > 1:
        from .distributed import edt_slabs
        cfg = cfg or PipelineConfig()
        partition(mask, *tile_dims)
        vr, dist = edt_slabs(mask.data, _conn(se))
        cfg.bp_waves = 1
        return (VoronoiMap(mask.width, mask.height, vr),
                Image2D(mask.width, mask.height, "f32", dist))
    vmap, seeds = init_packed(mask, se)
    rule = DistanceRule(vmap.vr, se)
    run_pipeline(vmap, rule, lambda: seeds, tile_dims, cfg)
    return vmap, finalize_distance_map(vmap)


def edt_exact_bruteforce(mask: Image2D) -> Image2D:
    """edt.py:313-323 / oracles.py:57-73: exact distances, the minimum over
    every background cell.  The device computes that same integer minimum by
    the separable exact transform (``iwpp_edt_exact``: column distances, then
    the lower envelope of parabolas per row), linear instead of quadratic."""
    _require_binary(mask)
    d2, dist = exact_sqdist(mask.data, want_dist=True)
    return Image2D(mask.width, mask.height, "f32", dist)


def exact_sqdist(mask, want_dist: bool = False):
    """(d2 int64, dist f32 or None) of the exact EDT of a raw 0/nonzero mask
    (numpy -> numpy, tensor -> tensor).  NoBackgroundError without background."""
    L = _lib.lib()
    torch = _lib._torch()
    host = not is_device_array(mask)
    H, W = mask.shape
    with _lib.device_of(mask):
        m = torch.from_numpy(np.ascontiguousarray(mask, dtype=np.uint8)).cuda() if host \
            else mask.contiguous()
        d2 = torch.empty((H, W), dtype=torch.int64, device=m.device)
        dist = torch.empty((H, W), dtype=torch.float32, device=m.device) if want_dist else None
        ws = _lib.workspace(L.iwpp_edt_exact_workspace_bytes(W, H))
        _lib.check(L.iwpp_edt_exact(_lib.ptr(m), W, H, _lib.ptr(d2),
                                    _lib.ptr(dist) if dist is not None else None, _lib.ptr(ws),
                                    ws.numel(), _lib.stream_ptr()), "edt_exact")
        if host:
            return d2.cpu().numpy(), dist.cpu().numpy() if dist is not None else None
    return d2, dist
