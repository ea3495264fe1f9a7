"""Multi-rank EDT slab protocol on CPU: the round loop,
boundary-row exchange and all-reduce termination of
``distributed.run_edt_slab_dist`` with the CPU slab-round restatement
(tests/edt_slab_oracle.py) as each rank's solver, in-process and over a
world-size-2 gloo group.  The sharded result must equal the single-image
oracle cell for cell, with the same number of rounds (the reference checks
its tiled EDT the same way: pkg/tests/test_tiles.py:250-259, C5 in
test_acceptance.py:135-170)."""

import os
import socket

import numpy as np
import pytest

import oracle
from edt_slab_oracle import CpuSlabEDT
from paper_1209_3314_b200.distributed import (mask_ext_rows, run_edt_slabs_local,
                                              slab_bounds)


def _slabs(m, G, conn):
    H = m.shape[0]
    out = []
    for r in range(G):
        y0, y1 = slab_bounds(H, G, r)
        out.append(CpuSlabEDT(mask_ext_rows(m, y0, y1), y0, H, r > 0, r + 1 < G, conn))
    return out


def _gather(slabs):
    parts = [s.finalize() for s in slabs]
    return (np.concatenate([p[0].numpy() for p in parts]),
            np.concatenate([p[1].numpy() for p in parts]))


def _masks():
    rng = np.random.default_rng(5)
    yield oracle.gen_synthetic_mask(96, 80, 50, 7)
    yield (rng.random((61, 47)) < 0.93).astype(np.uint8) * 255      # sparse background
    m = np.full((40, 33), 255, np.uint8)
    m[3, 30] = 0                                                     # one source: deep rounds
    yield m


@pytest.mark.parametrize("conn", [4, 8])
@pytest.mark.parametrize("G", [1, 2, 3, 5])
def test_cpu_slab_rounds_match_oracle(conn, G):
    for m in _masks():
        vr_ref, d_ref = oracle.edt(m, conn)
        slabs = _slabs(m, G, conn)
        rounds = run_edt_slabs_local(slabs)
        vr, d = _gather(slabs)
        assert np.array_equal(vr, vr_ref)
        assert d.tobytes() == d_ref.tobytes()
        assert all(s.rounds == rounds for s in slabs)


def test_cpu_slabs_reference_golden_vectors():
    """Every EDT golden vector of the reference (tests/golden/edt_golden.npz,
    including the C6 adversarial 24x24 tie where d2[21,5] == 170 instead of
    the exact 169) through 2- and 3-way slab cuts: vr and dist identical."""
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "edt_golden.npz"))
    names = sorted({k.split("__")[0] for k in g.files if k.endswith("__mask")})
    assert any(n.startswith("adversarial24") for n in names)
    for name in names:
        m = g[name + "__mask"]
        if (m != 0).all():
            continue  # no background: covered by the gloo test's agreed error
        conn = 4 if name.endswith("c4") else 8
        for G in (2, 3):
            if G > m.shape[0]:
                continue
            slabs = _slabs(m, G, conn)
            run_edt_slabs_local(slabs)
            vr, d = _gather(slabs)
            assert np.array_equal(vr, g[name + "__vr"]), (name, G)
            assert d.tobytes() == g[name + "__dist"].tobytes(), (name, G)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, conn, q):
    import torch.distributed as dist

    import edt_slab_oracle
    from paper_1209_3314_b200.distributed import finalize_agreed, run_edt_slab_dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = oracle.gen_synthetic_mask(96, 80, 50, 3)
        H = m.shape[0]
        y0, y1 = slab_bounds(H, world, rank)
        slab = edt_slab_oracle.CpuSlabEDT(mask_ext_rows(m, y0, y1), y0, H, rank > 0,
                                          rank + 1 < world, conn)
        rounds = run_edt_slab_dist(slab)
        vr, d = finalize_agreed(slab)
        q.put((rank, y0, y1, vr.numpy().copy(), d.numpy().copy(), rounds))
        # a mask with no background: every rank must raise together
        full = np.full((H, 80), 255, np.uint8)
        slab2 = edt_slab_oracle.CpuSlabEDT(mask_ext_rows(full, y0, y1), y0, H, rank > 0,
                                           rank + 1 < world, conn)
        run_edt_slab_dist(slab2)
        try:
            finalize_agreed(slab2)
            q.put((rank, "no-raise"))
        except Exception as e:  # noqa: BLE001
            q.put((rank, type(e).__name__))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("conn", [4, 8])
def test_gloo_world2_edt_slabs_match_oracle(conn):
    import sys

    import torch.multiprocessing as mp

    here = os.path.dirname(os.path.abspath(__file__))
    if here not in sys.path:
        sys.path.insert(0, here)
    os.environ["PYTHONPATH"] = here + os.pathsep + os.environ.get("PYTHONPATH", "")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, conn, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(4)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m = oracle.gen_synthetic_mask(96, 80, 50, 3)
    vr_ref, d_ref = oracle.edt(m, conn)
    vr = np.empty_like(vr_ref)
    d = np.empty_like(d_ref)
    rounds = set()
    errs = {}
    for item in res:
        if len(item) == 2:
            errs[item[0]] = item[1]
            continue
        rank, y0, y1, a, b, r = item
        vr[y0:y1], d[y0:y1] = a, b
        rounds.add(r)
    assert np.array_equal(vr, vr_ref)
    assert d.tobytes() == d_ref.tobytes()
    assert len(rounds) == 1  # both ranks stop after the same round
    assert errs == {0: "NoBackgroundError", 1: "NoBackgroundError"}
