"""Slab (multi-GPU) reconstruction path with the CUDA engine as the slab
solver.  Only one GPU is available to the tests, so G slabs run as virtual
ranks on it (the same SlabRecon / wave protocol the NCCL driver runs), plus
the real torch.distributed driver on a one-rank NCCL group.  Results must
equal the single-image oracle bit for bit."""

import os
import socket

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _slabs(J, I, G, conn):
    import torch
    from paper_1209_3314_b200.distributed import SlabRecon, device_solver, slab_bounds
    out = []
    for r in range(G):
        y0, y1 = slab_bounds(J.shape[0], G, r)
        out.append(SlabRecon(torch.from_numpy(J[y0:y1].copy()).cuda(),
                             torch.from_numpy(I[y0:y1].copy()).cuda(), r > 0, r + 1 < G, conn,
                             device_solver))
    return out


@pytest.mark.parametrize("conn", [4, 8])
@pytest.mark.parametrize("G", [2, 4, 8])
def test_virtual_slabs_random_u8(conn, G):
    from paper_1209_3314_b200.distributed import run_slabs_local
    J, I = oracle.gray_pair((1000, 777), 17 + G, h=40)
    want = oracle.recon_fh(J, I, conn)
    slabs = _slabs(J, I, G, conn)
    run_slabs_local(slabs)
    got = np.concatenate([s.result().cpu().numpy() for s in slabs])
    assert np.array_equal(got, want)


@pytest.mark.parametrize("conn", [4, 8])
def test_virtual_slabs_imfill(conn):
    from paper_1209_3314_b200.distributed import run_slabs_local
    bw = oracle.gen_synthetic_mask(1024, 1024, 50, 7)
    J, I = oracle.imfill_pair(bw)
    want = oracle.recon_fh(J, I, conn)
    slabs = _slabs(J, I, 8, conn)
    st = run_slabs_local(slabs)
    assert np.array_equal(np.concatenate([s.result().cpu().numpy() for s in slabs]), want)
    assert st.waves >= 2


def test_virtual_slabs_int32():
    from paper_1209_3314_b200.distributed import run_slabs_local
    J, I = oracle.gray_pair((300, 257), 5, h=1 << 27, dtype=np.int32)
    want = oracle.recon_fh(J, I, 8)
    slabs = _slabs(J, I, 3, 8)
    run_slabs_local(slabs)
    assert np.array_equal(np.concatenate([s.result().cpu().numpy() for s in slabs]), want)


def test_recon_slabs_nccl_single_rank():
    import torch
    import torch.distributed as dist
    from paper_1209_3314_b200.distributed import recon_slabs

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        J, I = oracle.gray_pair((256, 300), 3, h=40)
        got, st = recon_slabs(J, I, 8)
        assert np.array_equal(got, oracle.recon_fh(J, I, 8))
    finally:
        dist.destroy_process_group()


def _edt_slabs(m, G, conn):
    import torch
    from paper_1209_3314_b200.distributed import SlabEDT, mask_ext_rows, slab_bounds
    H = m.shape[0]
    out = []
    for r in range(G):
        y0, y1 = slab_bounds(H, G, r)
        out.append(SlabEDT(mask_ext_rows(m, y0, y1).cuda(), y0, H, r > 0, r + 1 < G, conn))
    return out


@pytest.mark.parametrize("conn", [4, 8])
@pytest.mark.parametrize("G", [2, 3, 8])
def test_edt_virtual_slabs_blob(conn, G):
    """Round-synchronous slab EDT (one boundary exchange per round) ==
    single-image oracle: source map and f32 distance bytes."""
    from paper_1209_3314_b200.distributed import run_edt_slabs_local
    m = oracle.gen_synthetic_mask(300, 256, 50, 7)
    vr_ref, d_ref, (rounds, _) = oracle.edt(m, conn, stats=True)
    slabs = _edt_slabs(m, G, conn)
    r = run_edt_slabs_local(slabs)
    parts = [s.finalize() for s in slabs]
    vr = np.concatenate([p[0].cpu().numpy() for p in parts])
    dist = np.concatenate([p[1].cpu().numpy() for p in parts])
    assert np.array_equal(vr, vr_ref)
    assert dist.tobytes() == d_ref.tobytes()
    assert r in (rounds, rounds + 1)


def test_edt_virtual_slabs_random_and_thin():
    from paper_1209_3314_b200.distributed import run_edt_slabs_local
    rng = np.random.default_rng(3)
    for shape, G in [((97, 131), 4), ((8, 200), 8), ((64, 64), 2)]:
        m = (rng.random(shape) < 0.9).astype(np.uint8) * 255
        m.flat[0] = 0
        vr_ref, d_ref = oracle.edt(m, 8)
        slabs = _edt_slabs(m, G, 8)
        run_edt_slabs_local(slabs)
        parts = [s.finalize() for s in slabs]
        assert np.array_equal(np.concatenate([p[0].cpu().numpy() for p in parts]), vr_ref)


# ---------------------------------------------------------------------------
# device-resident multi-slab EDT (iwpp_edt_mg_*): all rounds in one kernel,
# boundary items and frontier counts through the ranks' mailboxes

@pytest.mark.parametrize("conn", [4, 8])
@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_edt_mg_local_device_matches_oracle(conn, G):
    from paper_1209_3314_b200.distributed import edt_slabs_local_device
    rng = np.random.default_rng(11 + G)
    masks = [oracle.gen_synthetic_mask(300, 256, 50, 7),                  # blob: ~100 rounds
             (rng.random((97, 131)) < 0.9).astype(np.uint8) * 255,        # sparse background
             oracle.gen_nuclei_mask(512, 512, 30.0, 3)]
    for m in masks:
        vr_ref, d_ref, (rounds, _) = oracle.edt(m, conn, stats=True)
        vr, d, r = edt_slabs_local_device(m, G, conn)
        assert np.array_equal(vr, vr_ref)
        assert d.tobytes() == d_ref.tobytes()
        assert r == rounds  # the reference's round count, whatever the cut


def test_edt_mg_local_device_4k_blob_rounds():
    """The bench's 4K blob mask (314 rounds, raster and queue rounds both)
    over 4 slabs: bit-exact, same rounds."""
    from paper_1209_3314_b200.distributed import edt_slabs_local_device
    m = oracle.gen_synthetic_mask(4096, 4096, 50, 7)
    vr_ref, d_ref, (rounds, _) = oracle.edt(m, 8, stats=True)
    vr, d, r = edt_slabs_local_device(m, 4, 8)
    assert r == rounds
    assert np.array_equal(vr, vr_ref)
    assert d.tobytes() == d_ref.tobytes()


def test_edt_mg_local_device_errors():
    from paper_1209_3314_b200 import EngineError, NoBackgroundError
    from paper_1209_3314_b200.distributed import edt_slabs_local_device
    m = oracle.gen_synthetic_mask(200, 160, 50, 7)
    with pytest.raises(EngineError):
        edt_slabs_local_device(m, 3, 8, max_rounds=2)
    with pytest.raises(NoBackgroundError):
        edt_slabs_local_device(np.full((64, 48), 255, np.uint8), 2, 8)
    vr, d, r = edt_slabs_local_device(np.zeros((33, 17), np.uint8), 3, 8)  # all background
    assert r == 0 and np.array_equal(vr, np.arange(33 * 17).reshape(33, 17))


def test_edt_mg_nccl_single_rank_device_protocol():
    """The multi-GPU driver (symmetric-memory mailboxes, one kernel per GPU)
    on a one-rank NCCL group."""
    import torch
    import torch.distributed as dist
    from paper_1209_3314_b200.distributed import edt_slabs

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        m = oracle.gen_synthetic_mask(256, 300, 50, 7)
        vr_ref, d_ref = oracle.edt(m, 8)
        for engine in ("device", "host"):
            vr, d = edt_slabs(m, 8, engine=engine)
            assert np.array_equal(vr, vr_ref), engine
            assert d.tobytes() == d_ref.tobytes(), engine
    finally:
        dist.destroy_process_group()
