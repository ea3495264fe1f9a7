"""Randomized self-checks on the B200 (reference: gridwave/verify.py).

Same suites, flags, determinism and report lines as the reference
("recon: 4/4 pass").  Every suite compares one device result with a
differently-scheduled device twin or with a property / closed form that
does not share the code under test:

* ``recon``  -- register vs shared-memory BFS tile engine vs the host
                pipeline; the one-bit engine vs the u8 engines on binary
                inputs; the u16 / int32 engines on a strictly increasing
                remap of the same instance (reconstruction commutes with
                it); and the fixed-point properties marker <= J <= mask
                with an empty seed scan (no pixel can still raise a
                neighbour), checked by separate kernels;
* ``edt``    -- raster-frontier vs temporally blocked vs frontier-queue vs
                CAS engines, init+propagate vs edt vs edt_tiled; the closed
                form for a single source; the lower bound against the
                exact (brute-force) distance at 16 x 16;
* ``queue``  -- bounded queues: a random small capacity overflows, rescans
                and re-executes to the same image; the three EDT frontier
                queues (naive / prefix-sum / block) enqueue exactly the
                same items;
* ``tiling`` -- recon_tiled vs recon_fh, virtual multi-GPU slabs (wave
                protocol, border exchange) vs one device for recon and
                EDT, and the disjoint cover of ``partition``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .distributed import (SlabEDT, SlabRecon, device_solver, mask_ext_rows, run_edt_slabs_local,
                          run_slabs_local, slab_bounds)
from .edt import edt, edt_exact_bruteforce, edt_propagate, edt_tiled, init_packed
from .engine import EngineConfig, QueueConfig, QueueStrategy
from .grid import BG, FG, Image2D, StructuringElement
from .recon import ReconInput, reconstruct, recon_fh, recon_tiled, seed_scan
from .tiles import PipelineConfig, partition

SUITES = ("recon", "edt", "queue", "tiling")
# EDT engine modes (iwpp_edt_set_engine): raster, blocked, queue, CAS
_EDT_TWINS = (7, 4, 3, 1)
_EDT_QUEUES = {QueueStrategy.NAIVE: 6, QueueStrategy.PREFIX_SUM: 5, QueueStrategy.PER_WORKER: 3}


@dataclass
class SuiteResult:
    name: str
    passed: int
    failed: int

    @property
    def ok(self) -> bool:
        return self.failed == 0

    def line(self) -> str:
        return f"{self.name}: {self.passed}/{self.passed + self.failed} pass"


def _t():
    return _lib._torch()


def _dev(a):
    return _t().from_numpy(np.ascontiguousarray(a)).cuda()


def _gray_pair(rng, w, h):
    I = rng.integers(0, 256, (h, w)).astype(np.uint8)
    J = np.maximum(I.astype(np.int32) - 40, 0).astype(np.uint8)
    return J, I


def _random_mask(rng, w, h, pct):
    return (rng.random((h, w)) < pct / 100.0).astype(np.uint8) * FG


def _eq(a, b) -> bool:
    t = _t()
    a = a.cpu().numpy() if isinstance(a, t.Tensor) else a
    b = b.cpu().numpy() if isinstance(b, t.Tensor) else b
    return bool(np.array_equal(a, b))


def _le(a, b, kind) -> bool:
    from .recon import _count_violations
    return _count_violations(Image2D(a.shape[1], a.shape[0], kind, a),
                             Image2D(b.shape[1], b.shape[0], kind, b)) == 0


def _dilation_recon(marker, I, conn):
    """recon_by_dilation (the reference's oracles.py restated with torch
    pooling ops on the device, none of this package's kernels): repeat
    J <- min(I, max(J, dilate(J))) until nothing changes.  Small images only
    (one pass per unit of propagation distance)."""
    torch = _t()
    F = torch.nn.functional
    J, M = marker.to(torch.float32)[None, None], I.to(torch.float32)[None, None]
    for _ in range(4 * (J.shape[-1] + J.shape[-2]) * 8):
        if conn == 8:
            D = F.max_pool2d(J, 3, 1, 1)
        else:
            P = F.pad(J, (1, 1, 1, 1), value=-1.0)
            D = torch.maximum(torch.maximum(P[..., 1:-1, :-2], P[..., 1:-1, 2:]),
                              torch.maximum(P[..., :-2, 1:-1], P[..., 2:, 1:-1]))
            D = torch.maximum(D, J)
        N = torch.minimum(M, D)
        if torch.equal(N, J):
            break
        J = N
    return J[0, 0].to(marker.dtype)


def _fixed_point_ok(marker, J, I, conn, kind="u8") -> bool:
    """marker <= J <= mask, no seed left (a separate scan kernel), and -- up
    to 64K pixels -- J equals an independent iterated-dilation
    reconstruction, which also proves minimality (J = mask passes the first
    two checks)."""
    n = int(seed_scan(J, I, conn).numel())
    ok = _le(marker, J, kind) and _le(J, I, kind) and n == 0
    if ok and J.numel() <= 65536 and kind in ("u8", "binary"):
        ok = bool(_t().equal(_dilation_recon(marker, I, conn), J))
    return ok


class _edt_engine:
    def __init__(self, mode):
        self.mode = mode

    def __enter__(self):
        _lib.check(_lib.lib().iwpp_edt_set_engine(self.mode), "set_engine")

    def __exit__(self, *exc):
        _lib.check(_lib.lib().iwpp_edt_set_engine(0), "set_engine")


def verify_recon(cases: int, seed: int, size: tuple[int, int]) -> SuiteResult:
    rng = np.random.default_rng(seed)
    w, h = size
    passed = failed = 0
    for i in range(cases):
        conn = 8 if i % 2 == 0 else 4
        if i % 4 == 3:
            mask = (rng.random((h, w)) < 0.45).astype(np.uint8) * FG
            marker = np.where((rng.random((h, w)) < 0.06) & (mask == FG), FG, BG).astype(np.uint8)
            dJ, dI = _dev(marker), _dev(mask)
            a = reconstruct(dJ, dI, conn, kind="binary")
            ok = (_eq(a, reconstruct(dJ, dI, conn, engine=2))
                  and _eq(a, reconstruct(dJ, dI, conn, engine=1))
                  and _fixed_point_ok(dJ, a, dI, conn))
        else:
            J, I = _gray_pair(rng, w, h)
            dJ, dI = _dev(J), _dev(I)
            a = reconstruct(dJ, dI, conn, engine=2)
            host = reconstruct(J, I, conn, pipeline_rows=64)
            # strictly increasing remaps: u16 x 257, int32 x 1000 - 7
            a16 = reconstruct(_dev(J.astype(np.uint16) * 257), _dev(I.astype(np.uint16) * 257), conn)
            a32 = reconstruct(_dev(J.astype(np.int32) * 1000 - 7), _dev(I.astype(np.int32) * 1000 - 7),
                              conn)
            an = a.cpu().numpy()
            ok = (_eq(a, reconstruct(dJ, dI, conn, engine=1)) and _eq(a, host)
                  and _eq(a16, an.astype(np.uint16) * 257)
                  and _eq(a32, an.astype(np.int32) * 1000 - 7)
                  and _fixed_point_ok(dJ, a, dI, conn))
        passed, failed = passed + ok, failed + (not ok)
    return SuiteResult("recon", passed, failed)


def verify_edt(cases: int, seed: int, size: tuple[int, int]) -> SuiteResult:
    rng = np.random.default_rng(seed)
    w, h = size
    passed = failed = 0
    for i in range(cases):
        se = StructuringElement(8 if i % 2 == 0 else 4)
        if i % 5 == 4:
            a = np.full((h, w), FG, np.uint8)
            y0, x0 = int(rng.integers(0, h)), int(rng.integers(0, w))
            a[y0, x0] = BG
            vmap, _ = edt(Image2D(w, h, "binary", _dev(a)), se)
            ys, xs = np.mgrid[0:h, 0:w]
            ok = _eq(vmap.squared_distances(), ((ys - y0) ** 2 + (xs - x0) ** 2).astype(np.int64))
        else:
            m = _random_mask(rng, w, h, 25 + (i % 3) * 25)
            if not (m == BG).any():
                m[0, 0] = BG
            mask = Image2D(w, h, "binary", _dev(m))
            outs = []
            for mode in _EDT_TWINS:
                with _edt_engine(mode):
                    vm, d = edt(mask, se, mode="parallel")
                outs.append((vm.vr, d.data))
            vp, seeds = init_packed(mask, se)
            edt_propagate(vp, seeds, se)
            vt, _ = edt_tiled(mask, se, (max(w // 4, 1), max(h // 4, 1)))
            small = _random_mask(rng, 16, 16, 50)
            small[0, 0] = BG
            sm = Image2D(16, 16, "binary", _dev(small))
            vs, ds = edt(sm, se)
            exact = edt_exact_bruteforce(sm)
            ok = (all(_eq(v, outs[0][0]) and _eq(d, outs[0][1]) for v, d in outs)
                  and _eq(vp.vr, outs[0][0]) and _eq(vt.vr, outs[0][0])
                  and bool((ds.data >= exact.data).all()))
        passed, failed = passed + ok, failed + (not ok)
    return SuiteResult("edt", passed, failed)


def verify_queue(cases: int, seed: int, size: tuple[int, int]) -> SuiteResult:
    rng = np.random.default_rng(seed)
    w, h = size
    passed = failed = 0
    for i in range(cases):
        cw, ch = int(rng.integers(max(w // 2, 1), w + 1)), int(rng.integers(max(h // 2, 1), h + 1))
        J, I = _gray_pair(rng, cw, ch)
        dJ, dI = _dev(J), _dev(I)
        conn = 8 if i % 2 == 0 else 4
        cap = int(rng.integers(1, 120))
        want = reconstruct(dJ, dI, conn)
        cfg = EngineConfig(queue=QueueConfig(gbq_capacity=cap))
        st: dict = {}
        got = reconstruct(dJ, dI, conn, cfg=cfg, stats=st)
        ok = _eq(got, want) and st["overflow_count"] >= 0
        m = Image2D(cw, ch, "binary", _dev(_random_mask(rng, cw, ch, 50)))
        visits = set()
        ref = None
        for strat, mode in _EDT_QUEUES.items():
            c = EngineConfig(queue=QueueConfig(strategy=strat))
            with _edt_engine(mode):
                vm, sd = init_packed(m, StructuringElement(conn))
                edt_propagate(vm, sd, StructuringElement(conn), mode="parallel", cfg=c)
            visits.add((c.stats.rounds, c.stats.queued_total))
            ok = ok and (ref is None or _eq(vm.vr, ref))
            ref = vm.vr if ref is None else ref
        ok = ok and len(visits) == 1
        passed, failed = passed + ok, failed + (not ok)
    return SuiteResult("queue", passed, failed)


def verify_tiling(cases: int, seed: int, size: tuple[int, int]) -> SuiteResult:
    rng = np.random.default_rng(seed)
    w, h = size
    passed = failed = 0
    t = _t()
    for i in range(cases):
        conn = 8 if i % 2 == 0 else 4
        se = StructuringElement(conn)
        tile = [(16, 16), (32, 32), (w, h)][i % 3]
        G = 2 + i % 3
        J, I = _gray_pair(rng, w, h)
        inp = ReconInput(Image2D(w, h, "u8", _dev(J)), Image2D(w, h, "u8", _dev(I)), se)
        cfg = PipelineConfig(n_workers=(i % 3) + 1)
        want = recon_fh(inp).data
        ok = _eq(recon_tiled(inp, tile, cfg).data, want)
        slabs = []
        for r in range(G):
            y0, y1 = slab_bounds(h, G, r)
            slabs.append(SlabRecon(_dev(J[y0:y1]), _dev(I[y0:y1]), r > 0, r + 1 < G, conn,
                                   device_solver))
        run_slabs_local(slabs)
        ok = ok and _eq(t.cat([s.result() for s in slabs]), want)
        m = _random_mask(rng, w, h, 50)
        m[0, 0] = BG
        mask = Image2D(w, h, "binary", _dev(m))
        vt, _ = edt_tiled(mask, se, tile)
        vs, _ = edt(mask, se, mode="sequential")
        ok = ok and _eq(vt.vr, vs.vr)
        es = []
        for r in range(G):
            y0, y1 = slab_bounds(h, G, r)
            es.append(SlabEDT(mask_ext_rows(m, y0, y1).cuda(), y0, h, r > 0, r + 1 < G, conn))
        run_edt_slabs_local(es)
        ok = ok and _eq(t.cat([e.finalize()[0] for e in es]), vs.vr)
        grid = partition(inp.mask, *tile)
        member = np.zeros((h, w), np.int32)
        for tl in grid.tiles:
            member[tl.y0:tl.y1, tl.x0:tl.x1] += 1
        ok = ok and bool((member == 1).all())
        passed, failed = passed + ok, failed + (not ok)
    return SuiteResult("tiling", passed, failed)


_RUNNERS = {"recon": verify_recon, "edt": verify_edt, "queue": verify_queue,
            "tiling": verify_tiling}


def run_suites(suite: str, cases: int, seed: int, size: tuple[int, int]) -> list[SuiteResult]:
    names = SUITES if suite == "all" else (suite,)
    return [_RUNNERS[n](cases, seed, size) for n in names]
