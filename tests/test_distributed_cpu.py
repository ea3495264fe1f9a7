"""Multi-GPU slab protocol checked on CPU: the wave loop,
border-row exchange and all-reduce termination of
``paper_1209_3314_b200.distributed`` with the CPU oracle as the per-slab
solver (test infrastructure), in-process and over a world-size-2 gloo
group.  Sharded result == single-image oracle, cell for cell (the
reference checks its tiling the same way, test_tiles.py)."""

import os
import socket

import numpy as np
import pytest

import oracle
from paper_1209_3314_b200.distributed import (SlabRecon, run_slab_dist, run_slabs_local,
                                              slab_bounds)


def cpu_solver(J, I, conn, rows):
    """Per-slab fixed point by the oracle (rows: ignored, full solve)."""
    Jn = J.numpy() if hasattr(J, "numpy") else J
    In = I.numpy() if hasattr(I, "numpy") else I
    Jn[...] = oracle.recon_fh(Jn, In, conn)


def zigzag():
    I = np.zeros((16, 16), np.uint8)
    I[1, 1:15] = 100
    I[1:14, 14] = 100
    I[13, 1:15] = 100
    I[4:14, 1] = 100
    J = np.zeros((16, 16), np.uint8)
    J[1, 1] = 100
    return J, I


def slabs_for(J, I, G, conn):
    H = J.shape[0]
    out = []
    for r in range(G):
        y0, y1 = slab_bounds(H, G, r)
        out.append(SlabRecon(J[y0:y1].copy(), I[y0:y1].copy(), r > 0, r + 1 < G, conn, cpu_solver))
    return out


def test_slab_bounds_cover():
    for H in (1, 7, 64, 1000):
        for G in (1, 2, 3, 8):
            if G > H:
                continue
            rows = [slab_bounds(H, G, r) for r in range(G)]
            assert rows[0][0] == 0 and rows[-1][1] == H
            assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
            assert max(b - a for a, b in rows) - min(b - a for a, b in rows) <= 1


@pytest.mark.parametrize("conn", [4, 8])
@pytest.mark.parametrize("G", [2, 3, 5])
def test_virtual_slabs_random(conn, G):
    J, I = oracle.gray_pair((200, 150), 31 + G, h=50)
    want = oracle.recon_fh(J, I, conn)
    slabs = slabs_for(J, I, G, conn)
    st = run_slabs_local(slabs)
    got = np.concatenate([s.result() for s in slabs])
    assert np.array_equal(got, want)
    assert st.waves >= 1


@pytest.mark.parametrize("conn", [4, 8])
def test_virtual_slabs_imfill_many_waves(conn):
    bw = oracle.gen_synthetic_mask(256, 256, 50, 7)
    J, I = oracle.imfill_pair(bw)
    want = oracle.recon_fh(J, I, conn)
    slabs = slabs_for(J, I, 8, conn)
    st = run_slabs_local(slabs)
    assert np.array_equal(np.concatenate([s.result() for s in slabs]), want)


def test_virtual_slabs_zigzag_needs_several_waves():
    """A corridor that crosses the slab cut three times needs >= 3 waves
    (the reference's wave-structure criterion, test_tiles.py:262-288)."""
    J, I = zigzag()
    want = oracle.recon_fh(J, I, 8)
    slabs = slabs_for(J, I, 2, 8)
    st = run_slabs_local(slabs)
    assert np.array_equal(np.concatenate([s.result() for s in slabs]), want)
    assert st.waves >= 3


def test_wave_cap():
    from paper_1209_3314_b200 import ContractViolation
    J, I = zigzag()
    with pytest.raises(ContractViolation):
        run_slabs_local(slabs_for(J, I, 2, 8), max_waves=1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, conn, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bw = oracle.gen_synthetic_mask(192, 160, 50, 3)
        J, I = oracle.imfill_pair(bw)
        H = J.shape[0]
        y0, y1 = slab_bounds(H, world, rank)
        slab = SlabRecon(torch.from_numpy(J[y0:y1].copy()), torch.from_numpy(I[y0:y1].copy()),
                         rank > 0, rank + 1 < world, conn, cpu_solver)
        st = run_slab_dist(slab)
        q.put((rank, y0, y1, slab.result().numpy().copy(), st.waves))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("conn", [4, 8])
def test_gloo_world2_slabs_match_oracle(conn):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, conn, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    bw = oracle.gen_synthetic_mask(192, 160, 50, 3)
    J, I = oracle.imfill_pair(bw)
    want = oracle.recon_fh(J, I, conn)
    got = np.empty_like(want)
    for rank, y0, y1, part, waves in res:
        got[y0:y1] = part
    assert np.array_equal(got, want)
    assert res[0][4] == res[1][4]  # both ranks ran the same number of waves


def test_slab_reset_reruns_identically():
    """SlabRecon.reset (the bench's per-step marker restore) starts the
    protocol over: a second run from the same marker gives the same rows."""
    J, I = oracle.gray_pair((120, 90), 9, h=40)
    want = oracle.recon_fh(J, I, 8)
    slabs = slabs_for(J, I, 3, 8)
    run_slabs_local(slabs)
    first = np.concatenate([s.result().copy() for s in slabs])
    for r, s in enumerate(slabs):
        y0, y1 = slab_bounds(J.shape[0], 3, r)
        s.reset(J[y0:y1])
    run_slabs_local(slabs)
    assert np.array_equal(first, want)
    assert np.array_equal(np.concatenate([s.result() for s in slabs]), want)
