"""Multi-GPU slab execution: one process per GPU, horizontal
slabs, border rows exchanged with the up/down neighbours, global
termination by an all-reduce.

This mirrors the reference's tiled pipeline (tiles.py:375-431): TP = each
rank propagates its slab to the local fixed point; BP = the changed border
rows cross the slab cuts; waves repeat until no border changes anywhere.
Reconstruction's fixed point is unique (tiles.py:7-9), so the slab result
equals the single-device result cell for cell.

Slab layout (per rank, device buffers): ``J_ext``/``I_ext`` hold the rank's
rows plus one halo row above and below.  Halo rows carry the neighbour's
current border values in both J and I (J == I: never raised, never
clamped), so the engine treats them as fixed sources.  A missing neighbour
(image edge) is a min(T) row in both (never a source either).

The protocol is written against a tiny transport interface so the same
driver runs (a) one slab per rank over torch.distributed (NCCL on B200s,
gloo on CPU for the tests) and (b) several virtual slabs in one process
(the single-GPU parity tests).  The local solver is injected: the CUDA
engine (``device_solver``) in production; tests may pass a CPU checker.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ContractViolation

# sentinel (smallest) value per dtype, as stored in J/I halo rows
_LO = {np.dtype(np.uint8): 0, np.dtype(np.uint16): 0, np.dtype(np.int32): -(2**31)}


def slab_bounds(H: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [y0, y1) of ``rank`` for H rows split into ``world`` near-equal
    horizontal slabs (the reference's _bands, recon.py:260-272)."""
    if world < 1 or not 0 <= rank < world:
        raise ContractViolation("bad slab rank/world")
    base, rem = divmod(H, world)
    y0 = rank * base + min(rank, rem)
    return y0, y0 + base + (1 if rank < rem else 0)


@dataclass
class WaveStats:
    waves: int = 0
    halo_changes: int = 0


class SlabRecon:
    """One rank's slab of a reconstruction: ext buffers + protocol steps.

    ``xp`` is the array module of the buffers (torch for device slabs,
    numpy for CPU checker slabs); only element-wise copies and compares
    are used here.
    """

    def __init__(self, J_rows, I_rows, has_up: bool, has_down: bool, conn: int, solver):
        h, W = J_rows.shape
        self.h, self.W, self.conn, self.solver = h, W, conn, solver
        self.has_up, self.has_down = has_up, has_down
        self.is_torch = not isinstance(J_rows, np.ndarray)
        dt = np.dtype(np.uint8) if not self.is_torch else _np_dtype(J_rows)
        lo = _LO[dt]
        if self.is_torch:
            import torch
            self.J = torch.full((h + 2, W), lo, dtype=J_rows.dtype, device=J_rows.device)
            self.I = torch.full((h + 2, W), lo, dtype=I_rows.dtype, device=I_rows.device)
        else:
            dt = J_rows.dtype
            lo = _LO[np.dtype(dt)]
            self.J = np.full((h + 2, W), lo, dtype=dt)
            self.I = np.full((h + 2, W), lo, dtype=dt)
        self.J[1:h + 1] = J_rows
        self.I[1:h + 1] = I_rows
        self.first = True

    def reset(self, J_rows):
        """Start over from a new marker (same mask): the rows are copied in,
        the halo rows return to the min(T) sentinel until the next exchange
        (no reallocation, the mask rows stay)."""
        h = self.h
        lo = _LO[_np_dtype(self.J) if self.is_torch else np.dtype(self.J.dtype)]
        self.J[1:h + 1] = J_rows
        for r in (0, h + 1):
            self.J[r] = lo
            self.I[r] = lo
        self.first = True

    # -- protocol pieces --------------------------------------------------
    def border_rows(self):
        """(my first row, my last row) to send up / down."""
        return self.J[1], self.J[self.h]

    def set_halos(self, from_up, from_down):
        """Install the neighbours' border rows; returns (top changed,
        bottom changed).  Values only grow, so any difference is a rise."""
        top = bot = False
        if self.has_up and from_up is not None:
            top = bool((from_up != self.J[0]).any())
            self.J[0] = from_up
            self.I[0] = from_up  # J == I: a fixed source, never raised or clamped
        if self.has_down and from_down is not None:
            bot = bool((from_down != self.J[self.h + 1]).any())
            self.J[self.h + 1] = from_down
            self.I[self.h + 1] = from_down
        self._top, self._bot = top, bot
        return top, bot

    def solve(self):
        """Propagate to the slab's fixed point (first wave: everything;
        later waves: only the tile rows at changed halos)."""
        if self.first:
            rows = 0
        else:
            rows = (1 if self._top else 0) | (2 if self._bot else 0)
            if rows == 0:
                return
        self.solver(self.J, self.I, self.conn, rows)
        self.first = False

    def result(self):
        return self.J[1:self.h + 1]


def _np_dtype(t):
    import torch
    return {torch.uint8: np.dtype(np.uint8), torch.uint16: np.dtype(np.uint16),
            torch.int32: np.dtype(np.int32)}[t.dtype]


# ---------------------------------------------------------------------------
# solvers

def device_solver(J, I, conn: int, rows: int):
    """The CUDA tile engine on an ext slab (torch device tensors)."""
    from . import _lib
    L = _lib.lib()
    code = {np.dtype(np.uint8): 0, np.dtype(np.uint16): 1, np.dtype(np.int32): 2}[_np_dtype(J)]
    H, W = J.shape
    ws = _lib.workspace(L.iwpp_recon_workspace_bytes(W, H, code, conn))
    o = _lib.ReconOpts()
    o.sweeps, o.max_blocks, o.check_contract, o.queue_capacity = 0, 0, 0, 0
    o.tile_sweeps, o.halo_sweep_threshold, o.slab_rows = -1, -1, rows
    _lib.check(L.iwpp_recon(_lib.ptr(J), _lib.ptr(I), W, H, code, conn, _lib.ptr(ws),
                            ws.numel(), _lib.ctypes.byref(o), None, _lib.stream_ptr()), "slab")


# ---------------------------------------------------------------------------
# drivers

def run_slabs_local(slabs: list[SlabRecon], max_waves: int | None = None) -> WaveStats:
    """Several slabs in one process (virtual ranks), wave-synchronous."""
    st = WaveStats()
    n = len(slabs)
    pending = [(None, None)] * n
    # initial exchange: neighbours' marker rows
    for i, s in enumerate(slabs):
        up = slabs[i - 1].border_rows()[1] if i > 0 else None
        dn = slabs[i + 1].border_rows()[0] if i + 1 < n else None
        pending[i] = (_copy(up), _copy(dn))
    for i, s in enumerate(slabs):
        s.set_halos(*pending[i])
    while True:
        if max_waves is not None and st.waves >= max_waves:
            raise ContractViolation(f"no stability within {max_waves} waves")
        for s in slabs:
            s.solve()
        st.waves += 1
        for i, s in enumerate(slabs):
            up = slabs[i - 1].border_rows()[1] if i > 0 else None
            dn = slabs[i + 1].border_rows()[0] if i + 1 < n else None
            pending[i] = (_copy(up), _copy(dn))
        changed = 0
        for i, s in enumerate(slabs):
            t, b = s.set_halos(*pending[i])
            changed += int(t) + int(b)
        st.halo_changes += changed
        if changed == 0:
            return st


def _copy(x):
    if x is None:
        return None
    return x.clone() if hasattr(x, "clone") else x.copy()


def run_slab_dist(slab: SlabRecon, group=None, max_waves: int | None = None) -> WaveStats:
    """One slab per rank over torch.distributed (NCCL between B200s; gloo
    for CPU tests).  Border rows go to rank-1 / rank+1 with point-to-point
    send/recv; the wave loop ends when an all-reduce of halo changes is 0."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    st = WaveStats()

    def exchange():
        first, last = slab.border_rows()
        ops, up, dn = [], None, None
        if rank > 0:
            up = torch.empty_like(first)
            ops.append(dist.P2POp(dist.isend, first.contiguous(), rank - 1, group))
            ops.append(dist.P2POp(dist.irecv, up, rank - 1, group))
        if rank + 1 < world:
            dn = torch.empty_like(last)
            ops.append(dist.P2POp(dist.isend, last.contiguous(), rank + 1, group))
            ops.append(dist.P2POp(dist.irecv, dn, rank + 1, group))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        return slab.set_halos(up, dn)

    exchange()
    dev = slab.J.device
    while True:
        if max_waves is not None and st.waves >= max_waves:
            raise ContractViolation(f"no stability within {max_waves} waves")
        slab.solve()
        st.waves += 1
        t, b = exchange()
        flag = torch.tensor([int(t) + int(b)], device=dev, dtype=torch.int64)
        dist.all_reduce(flag, group=group)
        st.halo_changes += int(flag.item())
        if int(flag.item()) == 0:
            return st


def recon_slabs(marker, mask, conn: int = 8, group=None, max_waves: int | None = None):
    """Distributed reconstruction: every rank passes the FULL image (host
    numpy or device tensor), computes its slab on its GPU, and receives the
    full result (all-gather).  Returns (result, WaveStats)."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    H, W = marker.shape
    y0, y1 = slab_bounds(H, world, rank)
    dev = torch.device("cuda", torch.cuda.current_device())
    Jt = torch.as_tensor(marker)[y0:y1].to(dev)
    It = torch.as_tensor(mask)[y0:y1].to(dev)
    slab = SlabRecon(Jt, It, rank > 0, rank + 1 < world, conn, device_solver)
    st = run_slab_dist(slab, group, max_waves)
    full = torch.empty((H, W), dtype=Jt.dtype, device=dev)
    parts = [full[slice(*slab_bounds(H, world, r))] for r in range(world)]
    if all(p.shape == parts[0].shape for p in parts):
        dist.all_gather(parts, slab.result().contiguous(), group=group)
    else:  # ragged slabs: gather padded rows
        hmax = max(p.shape[0] for p in parts)
        buf = torch.zeros((hmax, W), dtype=Jt.dtype, device=dev)
        buf[:y1 - y0] = slab.result()
        outs = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(outs, buf, group=group)
        for r, p in enumerate(parts):
            p.copy_(outs[r][:p.shape[0]])
    if isinstance(marker, np.ndarray):
        return full.cpu().numpy(), st
    return full, st


# ---------------------------------------------------------------------------
# EDT: one exchange per round (the synchronous rule, tiles.py:10-15)

class SlabEDT:
    """One rank's slab of a distance transform on the device: the slab
    engine advances one two-phase round per call; the neighbours' boundary
    frontier rows (sources, all-ones = none) are the halo items of the
    round."""

    def __init__(self, mask_ext, y0: int, H: int, has_up: bool, has_down: bool, conn: int):
        import torch
        from . import _lib
        self._lib, self.L = _lib, _lib.lib()
        h2, W = mask_ext.shape
        self.h, self.W, self.y0, self.H, self.conn = h2 - 2, W, y0, H, conn
        self.has_up, self.has_down = has_up, has_down
        dev = self.device = mask_ext.device
        self.ws = torch.empty(self.L.iwpp_edt_slab_workspace_bytes(W, self.h), dtype=torch.uint8,
                              device=dev)
        self.out = [torch.empty(W, dtype=torch.int64, device=dev) for _ in range(2)]
        self.rounds = 0
        self._lib.check(self.L.iwpp_edt_slab_init(
            _lib.ptr(mask_ext.contiguous()), W, self.h, y0, H, conn, int(has_up), int(has_down),
            _lib.ptr(self.ws), _lib.ptr(self.out[0]), _lib.ptr(self.out[1]), _lib.stream_ptr()),
            "edt_slab_init")

    def boundary_rows(self):
        """(first-row, last-row) frontier sources of the coming round."""
        return self.out[0], self.out[1]

    def round(self, halo_up, halo_dn) -> int:
        """Run one round; returns this slab's next frontier size."""
        import torch
        _lib = self._lib
        new = [torch.empty_like(self.out[0]), torch.empty_like(self.out[1])]
        n = _lib.ctypes.c_int64(0)
        _lib.check(self.L.iwpp_edt_slab_round(
            _lib.ptr(self.ws), self.W, self.h, self.y0, self.conn, self.rounds,
            _lib.ptr(halo_up) if halo_up is not None else None,
            _lib.ptr(halo_dn) if halo_dn is not None else None,
            _lib.ptr(new[0]), _lib.ptr(new[1]), _lib.ctypes.byref(n), _lib.stream_ptr()),
            "edt_slab_round")
        self.out = new
        self.rounds += 1
        return int(n.value)

    def finalize(self):
        import torch
        _lib = self._lib
        dev = self.ws.device
        vr = torch.empty((self.h, self.W), dtype=torch.int64, device=dev)
        dist = torch.empty((self.h, self.W), dtype=torch.float32, device=dev)
        _lib.check(self.L.iwpp_edt_slab_finalize(_lib.ptr(self.ws), self.W, self.h, self.y0,
                                                 self.rounds, _lib.ptr(vr), _lib.ptr(dist),
                                                 _lib.stream_ptr()), "edt_slab_finalize")
        return vr, dist


def mask_ext_rows(mask, y0: int, y1: int):
    """(h + 2) x W slab of a full mask with the neighbours' rows (zeros past
    the image edge; the engine ignores them there)."""
    import torch
    m = torch.as_tensor(mask)
    H, W = m.shape
    ext = torch.zeros((y1 - y0 + 2, W), dtype=torch.uint8)
    ext[1:-1] = m[y0:y1]
    if y0 > 0:
        ext[0] = m[y0 - 1]
    if y1 < H:
        ext[-1] = m[y1]
    return ext


def run_edt_slabs_local(slabs: list[SlabEDT], max_rounds: int | None = None) -> int:
    """Virtual ranks in one process: round-synchronous, one boundary-row
    exchange per round.  Returns the number of rounds."""
    n = len(slabs)
    while True:
        if max_rounds is not None and slabs[0].rounds >= max_rounds:
            from .errors import EngineError
            raise EngineError(f"no fixed point within {max_rounds} rounds")
        halos = []
        for i in range(n):
            up = slabs[i - 1].boundary_rows()[1] if i > 0 else None
            dn = slabs[i + 1].boundary_rows()[0] if i + 1 < n else None
            halos.append((up, dn))
        total = sum(s.round(*hl) for s, hl in zip(slabs, halos))
        if total == 0:
            return slabs[0].rounds


def run_edt_slab_dist(slab: SlabEDT, group=None, max_rounds: int | None = None) -> int:
    """One slab per rank: per round, boundary rows to rank-1 / rank+1
    (send/recv), then an all-reduce of the next frontier sizes."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = slab.device
    while True:
        if max_rounds is not None and slab.rounds >= max_rounds:
            from .errors import EngineError
            raise EngineError(f"no fixed point within {max_rounds} rounds")
        first, last = slab.boundary_rows()
        ops, up, dn = [], None, None
        if rank > 0:
            up = torch.empty_like(first)
            ops.append(dist.P2POp(dist.isend, first, rank - 1, group))
            ops.append(dist.P2POp(dist.irecv, up, rank - 1, group))
        if rank + 1 < world:
            dn = torch.empty_like(last)
            ops.append(dist.P2POp(dist.isend, last, rank + 1, group))
            ops.append(dist.P2POp(dist.irecv, dn, rank + 1, group))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        nxt = slab.round(up, dn)
        t = torch.tensor([nxt], device=dev, dtype=torch.int64)
        dist.all_reduce(t, group=group)
        if int(t.item()) == 0:
            return slab.rounds


def finalize_agreed(slab, group=None):
    """slab.finalize() on every rank, with the ranks agreeing on the outcome
    before anyone moves on: a rank whose finalize raises (no background,
    key-range overflow) would otherwise leave the others blocked in the
    all-gather that follows.  The error codes are all-reduced (max) and
    every rank raises the same exception."""
    import torch
    import torch.distributed as dist
    from .errors import EngineError, NoBackgroundError

    out, code, msg = None, 0, ""
    try:
        out = slab.finalize()
    except NoBackgroundError as e:
        code, msg = 1, str(e)
    except EngineError as e:
        code, msg = 2, str(e)
    except RuntimeError as e:  # IWPP_E_OVERFLOW: a d2 beyond the 32-bit key field
        code, msg = 3, str(e)
    flag = torch.tensor([code], dtype=torch.int64, device=slab.device)
    dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
    code = int(flag.item())
    if code == 1:
        raise NoBackgroundError(msg or "no background reachable: distance map undefined")
    if code == 2:
        raise EngineError(msg or "engine limit reached on another slab")
    if code == 3:
        raise RuntimeError(msg or "a squared distance exceeded the 32-bit key range (another slab)")
    return out


def edt_slabs(mask, conn: int = 8, group=None, max_rounds: int | None = None,
              engine: str = "auto"):
    """Distributed EDT: every rank passes the full binary mask; returns the
    full (vr int64, dist f32) on every rank (all-gather).

    engine="device" runs all rounds in one kernel per GPU with the
    boundary items and counts going through NVLink mailboxes
    (run_edt_slab_device); engine="host" runs the per-round host loop
    (NCCL send/recv + all-reduce per round, run_edt_slab_dist); "auto"
    takes the device protocol when the symmetric-memory rendezvous works."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    H, W = mask.shape
    y0, y1 = slab_bounds(H, world, rank)
    dev = torch.device("cuda", torch.cuda.current_device())
    dslab = None
    if engine in ("auto", "device"):
        try:  # the mailbox rendezvous (symmetric memory over NVLink)
            dslab = DeviceSlabEDT(mask_ext_rows(mask, y0, y1).to(dev), y0, H, conn, group)
        except Exception:  # noqa: BLE001 - no symmetric memory / peer access here
            if engine == "device":
                raise
        # every rank takes the same protocol
        ok = torch.tensor([1 if dslab is not None else 0], dtype=torch.int64, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if int(ok.item()) == 0:
            dslab = None
    if dslab is not None:
        dslab.run(max_rounds)
        vr, dist_ = finalize_agreed(dslab, group)
    else:
        slab = SlabEDT(mask_ext_rows(mask, y0, y1).to(dev), y0, H, rank > 0, rank + 1 < world, conn)
        run_edt_slab_dist(slab, group, max_rounds)
        vr, dist_ = finalize_agreed(slab, group)
    outs = []
    for t in (vr, dist_):
        hmax = max(b - a for a, b in (slab_bounds(H, world, r) for r in range(world)))
        buf = torch.zeros((hmax, W), dtype=t.dtype, device=dev)
        buf[:y1 - y0] = t
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf, group=group)
        full = torch.cat([parts[r][:slab_bounds(H, world, r)[1] - slab_bounds(H, world, r)[0]]
                          for r in range(world)])
        outs.append(full.cpu().numpy() if isinstance(mask, np.ndarray) else full)
    return outs[0], outs[1]


# ---------------------------------------------------------------------------
# EDT, device-resident rounds (iwpp_edt_mg_*: one persistent kernel per GPU,
# boundary items and frontier counts through per-rank mailboxes)

def _mg_setup(L, mask_ext, W, h, y0, H, conn, rank, world, mailboxes, dev):
    import torch
    from . import _lib
    ws = torch.empty(L.iwpp_edt_mg_workspace_bytes(W, h), dtype=torch.uint8, device=dev)
    up = _lib.ptr(mailboxes[rank - 1]) if rank > 0 else None
    dn = _lib.ptr(mailboxes[rank + 1]) if rank + 1 < world else None
    _lib.check(L.iwpp_edt_mg_init(_lib.ptr(mask_ext), W, h, y0, H, conn, int(rank > 0),
                                  int(rank + 1 < world), _lib.ptr(ws), up, dn, _lib.stream_ptr()),
               "edt_mg_init")
    d = _lib.MgSlab()
    d.workspace, d.W, d.h, d.y0, d.H = _lib.ptr(ws), W, h, y0, H
    d.has_up, d.has_down, d.rank, d.world = int(rank > 0), int(rank + 1 < world), rank, world
    for g, mb in enumerate(mailboxes):
        d.mailbox[g] = _lib.ptr(mb)
    return ws, d


def _mg_finalize(L, ws, W, h, y0, rounds, dev):
    import torch
    from . import _lib
    vr = torch.empty((h, W), dtype=torch.int64, device=dev)
    dist = torch.empty((h, W), dtype=torch.float32, device=dev)
    _lib.check(L.iwpp_edt_slab_finalize(_lib.ptr(ws), W, h, y0, rounds, _lib.ptr(vr), _lib.ptr(dist),
                                        _lib.stream_ptr()), "edt_slab_finalize")
    return vr, dist


def edt_slabs_local_device(mask, G: int, conn: int = 8, max_rounds: int | None = None,
                           timing: dict | None = None):
    """G horizontal slabs of one mask on ONE GPU through the device-resident
    multi-slab protocol: the slabs are CTA groups of one launch and their
    mailboxes live in this GPU's memory -- the same kernel, mailbox protocol
    and count exchange the multi-GPU run uses over NVLink (edt_slabs with
    engine="device").  Returns (vr, dist, rounds)."""
    import torch
    from . import _lib
    L = _lib.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    m = torch.as_tensor(mask)
    H, W = m.shape
    if not 1 <= G <= 16 or G > H:
        raise ValueError("1 <= G <= min(16, H) slabs")
    mbb = L.iwpp_edt_mg_mailbox_bytes(W)
    mailboxes = [torch.zeros(mbb, dtype=torch.uint8, device=dev) for _ in range(G)]
    keep, descs = [], (_lib.MgSlab * G)()
    md = m.to(dev)
    for r in range(G):
        y0, y1 = slab_bounds(H, G, r)
        ext = torch.zeros((y1 - y0 + 2, W), dtype=torch.uint8, device=dev)
        ext[1:-1] = md[y0:y1]
        if y0 > 0:
            ext[0] = md[y0 - 1]
        if y1 < H:
            ext[-1] = md[y1]
        ws, d = _mg_setup(L, ext, W, y1 - y0, y0, H, conn, r, G, mailboxes, dev)
        keep.append((ext, ws))
        descs[r] = d
    rounds = _lib.ctypes.c_int64(0)
    if timing is not None:  # diagnostics: CUDA events around the rounds kernel alone
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
    _lib.check(L.iwpp_edt_mg_run(descs, G, conn, -1 if max_rounds is None else max_rounds,
                                 _lib.ctypes.byref(rounds), _lib.stream_ptr()), "edt_mg_run")
    if timing is not None:
        ev[1].record()
        ev[1].synchronize()
        timing["rounds_ms"] = ev[0].elapsed_time(ev[1])
    parts = [_mg_finalize(L, keep[r][1], W, descs[r].h, descs[r].y0, rounds.value, dev) for r in range(G)]
    vr = torch.cat([p[0] for p in parts])
    dist = torch.cat([p[1] for p in parts])
    if isinstance(mask, np.ndarray):
        return vr.cpu().numpy(), dist.cpu().numpy(), rounds.value
    return vr, dist, rounds.value


def symmetric_mailboxes(nbytes: int, group=None):
    """Every rank's mailbox as a tensor valid on this GPU: this rank's own
    buffer plus the peers' buffers mapped over NVLink (torch symmetric
    memory, the CUDA IPC rendezvous).  Zeroed, and every rank has zeroed its
    own before this returns."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm

    world = dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device())
    buf = symm.empty(nbytes, dtype=torch.uint8, device=dev)
    buf.zero_()
    torch.cuda.synchronize()
    hdl = symm.rendezvous(buf, group if group is not None else dist.group.WORLD)
    peers = [buf if g == dist.get_rank(group) else hdl.get_buffer(g, (nbytes,), torch.uint8)
             for g in range(world)]
    dist.barrier(group=group)
    return peers, hdl


class DeviceSlabEDT:
    """One rank's slab of a multi-GPU EDT on the device-resident protocol
    (iwpp_edt_mg_*): ``run()`` zeroes this rank's mailbox, seeds the
    neighbours' mailboxes with the initial boundary items and runs every
    round in one kernel; ``finalize()`` returns this rank's (vr, dist) rows,
    with the ranks agreeing on errors.  ``mask_ext`` = the rank's rows plus
    one neighbour row above / below (device tensor, zeros past the edge)."""

    def __init__(self, mask_ext, y0: int, H: int, conn: int = 8, group=None, mailboxes=None):
        import torch
        import torch.distributed as dist
        from . import _lib
        self._lib, self.L = _lib, _lib.lib()
        self.group = group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.ext = mask_ext
        self.h, self.W = mask_ext.shape[0] - 2, mask_ext.shape[1]
        self.y0, self.H, self.conn = y0, H, conn
        self.device = mask_ext.device
        if mailboxes is None:
            mailboxes, self._hdl = symmetric_mailboxes(self.L.iwpp_edt_mg_mailbox_bytes(self.W), group)
        self.mailboxes = mailboxes
        self.rounds = 0
        self.ws = None

    def run(self, max_rounds: int | None = None) -> int:
        import torch
        import torch.distributed as dist
        _lib, L = self._lib, self.L
        dist.barrier(group=self.group)            # everyone is done with the previous run
        self.mailboxes[self.rank].zero_()
        torch.cuda.synchronize()
        dist.barrier(group=self.group)            # all mailboxes are clean
        self.ws, d = _mg_setup(L, self.ext, self.W, self.h, self.y0, self.H, self.conn, self.rank,
                               self.world, self.mailboxes, self.device)
        torch.cuda.synchronize()
        dist.barrier(group=self.group)            # every rank's initial items are in place
        descs = (_lib.MgSlab * 1)(d)
        rounds = _lib.ctypes.c_int64(0)
        _lib.check(L.iwpp_edt_mg_run(descs, 1, self.conn, -1 if max_rounds is None else max_rounds,
                                     _lib.ctypes.byref(rounds), _lib.stream_ptr()), "edt_mg_run")
        self.rounds = rounds.value
        return self.rounds

    def finalize(self):
        return _mg_finalize(self.L, self.ws, self.W, self.h, self.y0, self.rounds, self.device)


def run_edt_slab_device(mask, conn: int = 8, group=None, max_rounds: int | None = None):
    """One slab per rank, all rounds in one kernel per GPU (no host round
    trip per round): boundary items and frontier counts go straight into
    the neighbours' / everyone's mailboxes over NVLink.  Returns (vr rows,
    dist rows, rounds, (y0, y1)) of this rank."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    H, W = mask.shape
    y0, y1 = slab_bounds(H, world, rank)
    dev = torch.device("cuda", torch.cuda.current_device())
    slab = DeviceSlabEDT(mask_ext_rows(mask, y0, y1).to(dev), y0, H, conn, group)
    slab.run(max_rounds)
    vr, dist_ = finalize_agreed(slab, group)
    return vr, dist_, slab.rounds, (y0, y1)
