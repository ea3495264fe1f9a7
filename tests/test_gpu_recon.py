"""Reconstruction parity on the B200: the CUDA engine through the public
(drop-in) API and the C ABI, against the reference's golden vectors and
the CPU oracle.  Bit-exact everywhere (integer work, zero tolerance).

Mirrors the reference's own recon tests (pkg/tests/test_recon.py,
test_acceptance.py C1-C4, C7)."""

import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gw():
    import torch
    import paper_1209_3314_b200 as gw
    torch.cuda.set_device(0)
    return gw


def _torch():
    import torch
    return torch


def _kind(a, name=""):
    if name.startswith(("bin", "imfill")):
        return "binary"
    return {np.uint8: "u8", np.uint16: "u16", np.int32: "i32", np.float32: "f32"}[a.dtype.type]


def _pair(gw, J, I, conn, kind, device):
    h, w = J.shape
    if device:
        t = _torch()
        J, I = t.from_numpy(J.copy()).cuda(), t.from_numpy(I.copy()).cuda()
    return gw.ReconInput(gw.Image2D(w, h, kind, J), gw.Image2D(w, h, kind, I),
                         gw.StructuringElement(conn))


def _np(a):
    return a.cpu().numpy() if hasattr(a, "cpu") else a


RZ = np.load(os.path.join(GOLD, "recon_golden.npz"))
RNAMES = sorted({k.split("__")[0] for k in RZ.files if k.endswith("__out")})


@pytest.mark.parametrize("device", [False, True])
@pytest.mark.parametrize("name", RNAMES)
def test_golden_vectors(gw, name, device):
    J, I, R = RZ[name + "__marker"], RZ[name + "__mask"], RZ[name + "__out"]
    conn = 8 if name.endswith("c8") else 4
    inp = _pair(gw, J, I, conn, _kind(J, name), device)
    out = gw.recon_fh(inp)
    assert out.elem_kind == inp.marker.elem_kind
    assert np.array_equal(_np(out.data), R)


@pytest.mark.parametrize("conn", [4, 8])
@pytest.mark.parametrize("dtype", [np.uint8, np.uint16, np.int32])
def test_random_sizes_vs_oracle(gw, conn, dtype):
    rng = np.random.default_rng(100 + conn)
    for shape in [(1, 1), (1, 300), (300, 1), (63, 65), (64, 64), (65, 129), (200, 333), (513, 257)]:
        seed = int(rng.integers(0, 1 << 30))
        h = {np.uint8: 40, np.uint16: 9000, np.int32: 1 << 27}[dtype]
        J, I = oracle.gray_pair(shape, seed, h=h, dtype=dtype)
        want = oracle.recon_fh(J, I, conn)
        got = gw.reconstruct(_torch().from_numpy(J).cuda(), _torch().from_numpy(I).cuda(), conn)
        assert np.array_equal(got.cpu().numpy(), want), (shape, seed)


@pytest.mark.parametrize("conn", [4, 8])
def test_4k_u8_vs_oracle(gw, conn):
    """BASELINE configs[1] at full size (4096^2 u8), seed 0."""
    J, I = oracle.gray_pair(4096, 0, h=40)
    want = oracle.recon_fh(J, I, conn)
    got = gw.reconstruct(_torch().from_numpy(J).cuda(), _torch().from_numpy(I).cuda(), conn)
    assert np.array_equal(got.cpu().numpy(), want)


@pytest.mark.parametrize("conn", [4, 8])
def test_2k_int32_seed3_vs_oracle(gw, conn):
    # 4096^2 int32 (configs[1]'s int32 variant) is in test_gpu_config_parity.py
    J, I = oracle.gray_pair(2048, 3, h=1 << 28, dtype=np.int32)
    want = oracle.recon_fh(J, I, conn)
    got = gw.reconstruct(_torch().from_numpy(J).cuda(), _torch().from_numpy(I).cuda(), conn)
    assert np.array_equal(got.cpu().numpy(), want)


@pytest.mark.parametrize("conn", [4, 8])
def test_imfill_vs_oracle(gw, conn):
    bw = oracle.gen_synthetic_mask(1024, 1024, 50, 7)
    marker, mask = oracle.imfill_pair(bw)
    want = oracle.recon_fh(marker, mask, conn)
    inp = _pair(gw, marker, mask, conn, "binary", True)
    assert np.array_equal(_np(gw.recon_fh(inp).data), want)


def test_all_entry_points_agree_and_inputs_untouched(gw):
    J, I = oracle.gray_pair(96, 7, h=50)
    want = oracle.recon_fh(J, I, 8)
    for device in (False, True):
        inp = _pair(gw, J, I, 8, "u8", device)
        J0, I0 = _np(inp.marker.data).copy(), _np(inp.mask.data).copy()
        outs = [gw.recon_sr(inp), gw.recon_qb(inp), gw.recon_fh(inp),
                gw.recon_parallel(inp, gw.EngineConfig(n_workers=4)),
                gw.recon_tiled(inp, (32, 32), gw.PipelineConfig(n_workers=2))]
        for o in outs:
            assert np.array_equal(_np(o.data), want)
        assert np.array_equal(_np(inp.marker.data), J0)
        assert np.array_equal(_np(inp.mask.data), I0)


def test_forced_overflow_recovers_exactly(gw):
    """C7 analog: a tiny block queue forces drop -> rescan -> re-execute."""
    J, I = oracle.gray_pair(256, 1007, h=40)
    want = oracle.recon_fh(J, I, 8)
    cfg = gw.EngineConfig(n_workers=2, queue=gw.QueueConfig(gbq_capacity=16))
    inp = _pair(gw, J, I, 8, "u8", True)
    got = gw.recon_parallel(inp, cfg)
    assert np.array_equal(_np(got.data), want)
    assert cfg.stats.overflow_count >= 2


def test_contract_violation_raises(gw):
    J = np.array([[5, 0]], np.uint8)
    I = np.array([[4, 9]], np.uint8)
    with pytest.raises(gw.ContractViolation):
        _pair(gw, J, I, 8, "u8", True)
    with pytest.raises(gw.ContractViolation):
        _pair(gw, J, I, 8, "u8", False)


def test_marker_equal_mask_identity_and_zero_marker(gw):
    rng = np.random.default_rng(1)
    I = rng.integers(0, 256, (77, 91)).astype(np.uint8)
    out = gw.recon_fh(_pair(gw, I.copy(), I, 8, "u8", True))
    assert np.array_equal(_np(out.data), I)
    Z = np.zeros_like(I)
    out = gw.recon_fh(_pair(gw, Z, np.maximum(I, 1), 4, "u8", True))
    assert not _np(out.data).any()


def test_fixed_point_equation_and_idempotence(gw):
    J, I = oracle.gray_pair(128, 23, h=40)
    out = _np(gw.recon_fh(_pair(gw, J, I, 8, "u8", True)).data)
    assert np.all(J <= out) and np.all(out <= I)
    P = np.pad(out, 1, mode="constant")
    neigh = np.stack([P[1 + dy:129 + dy, 1 + dx:129 + dx]
                      for dx, dy in [(a, b) for b in (-1, 0, 1) for a in (-1, 0, 1)]])
    assert np.array_equal(out, np.minimum(neigh.max(0), I))
    again = _np(gw.recon_fh(_pair(gw, out, I, 8, "u8", True)).data)
    assert np.array_equal(again, out)


def test_binary_components(gw):
    rng = np.random.default_rng(1004)
    for i in range(10):
        conn = 8 if i % 2 == 0 else 4
        mask = (rng.random((64, 64)) < 0.45).astype(np.uint8) * 255
        marker = np.where((rng.random((64, 64)) < 0.06) & (mask == 255), 255, 0).astype(np.uint8)
        want = oracle.recon_fh(marker, mask, conn)
        got = gw.recon_fh(_pair(gw, marker, mask, conn, "binary", True))
        assert np.array_equal(_np(got.data), want)


def test_row_sweep_stage_is_exact_row_recurrence(gw):
    """iwpp_recon_sweep_rows = K.115-139 forward then backward, exactly."""
    from paper_1209_3314_b200 import _lib
    t = _torch()
    L = _lib.lib()
    for dtype, W in [(np.uint8, 4096), (np.uint8, 1001), (np.int32, 777), (np.uint16, 64)]:
        J, I = oracle.gray_pair((37, W), 5, h=30 if dtype == np.uint8 else 1000, dtype=dtype)
        want = J.astype(np.int64).copy()
        Ii = I.astype(np.int64)
        for y in range(J.shape[0]):
            for x in range(1, W):
                want[y, x] = max(want[y, x], min(want[y, x - 1], Ii[y, x]))
            for x in range(W - 2, -1, -1):
                want[y, x] = max(want[y, x], min(want[y, x + 1], Ii[y, x]))
        dJ, dI = t.from_numpy(J).cuda(), t.from_numpy(I).cuda()
        code = {np.uint8: 0, np.uint16: 1, np.int32: 2}[dtype]
        _lib.check(L.iwpp_recon_sweep_rows(_lib.ptr(dJ), _lib.ptr(dI), W, J.shape[0], code,
                                           _lib.stream_ptr()))
        assert np.array_equal(dJ.cpu().numpy().astype(np.int64), want), (dtype, W)


def test_col_sweep_stage_is_exact_column_recurrence(gw):
    """iwpp_recon_sweep_cols = K.142-190 (vertical neighbour) forward then
    backward along full columns, exactly (segment composites + carry scan)."""
    from paper_1209_3314_b200 import _lib
    t = _torch()
    L = _lib.lib()
    for dtype, (H, W) in [(np.uint8, (1000, 37)), (np.uint8, (64, 128)), (np.int32, (333, 65)),
                          (np.uint16, (130, 7))]:
        J, I = oracle.gray_pair((H, W), 6, h=30 if dtype == np.uint8 else 1000, dtype=dtype)
        want = J.astype(np.int64).copy()
        Ii = I.astype(np.int64)
        for y in range(1, H):
            want[y] = np.maximum(want[y], np.minimum(want[y - 1], Ii[y]))
        for y in range(H - 2, -1, -1):
            want[y] = np.maximum(want[y], np.minimum(want[y + 1], Ii[y]))
        dJ, dI = t.from_numpy(J).cuda(), t.from_numpy(I).cuda()
        code = {np.uint8: 0, np.uint16: 1, np.int32: 2}[dtype]
        ws = _lib.workspace(L.iwpp_recon_workspace_bytes(W, H, code, 8))
        _lib.check(L.iwpp_recon_sweep_cols(_lib.ptr(dJ), _lib.ptr(dI), W, H, code, _lib.ptr(ws),
                                           _lib.stream_ptr()))
        assert np.array_equal(dJ.cpu().numpy().astype(np.int64), want), (dtype, H, W)


def test_seed_scan_matches_oracle(gw):
    J, I = oracle.gray_pair((130, 97), 9, h=60)
    for conn in (4, 8):
        want = oracle.recon_seed_scan(J, I, conn)
        got = gw.recon.seed_scan(J, I, conn)
        assert np.array_equal(got, want)


def test_sweeps_option_same_result(gw):
    """The full-image sweep pre-pass (any count) never changes the result."""
    J, I = oracle.gray_pair(300, 11, h=40)
    want = oracle.recon_fh(J, I, 8)
    for sweeps in (1, 2):
        got = gw.reconstruct(_torch().from_numpy(J).cuda(), _torch().from_numpy(I).cuda(), 8,
                             sweeps=sweeps)
        assert np.array_equal(got.cpu().numpy(), want)


# ---------------------------------------------------------------------------
# host path (iwpp_recon_host): slabs stream in and are reconstructed while
# later slabs are still in flight, then each cut is repaired; results must
# not depend on the slab height.

@pytest.mark.parametrize("conn", [4, 8])
@pytest.mark.parametrize("rows", [-1, 32, 64, 96, 256])
def test_host_pipeline_any_slab_height(gw, conn, rows):
    for shape, seed in [((1000, 300), 1), ((513, 700), 2), ((64, 33), 3)]:
        J, I = oracle.gray_pair(shape, seed, h=40)
        want = oracle.recon_fh(J, I, conn)
        st = {}
        got = gw.reconstruct(J, I, conn, pipeline_rows=rows, stats=st)
        assert np.array_equal(got, want), (shape, rows)
        assert st["contract_violations"] == 0


@pytest.mark.parametrize("conn", [4, 8])
def test_host_pipeline_long_range_imfill(gw, conn):
    """imfill: raises cross many cuts (the fill enters from the image border
    and runs through every slab), so later repairs rewrite earlier slabs."""
    bw = oracle.gen_synthetic_mask(512, 2048, 50, 7)
    marker, mask = oracle.imfill_pair(bw)
    want = oracle.recon_fh(marker, mask, conn)
    for rows in (0, 32, 128):
        got = gw.reconstruct(marker, mask, conn, pipeline_rows=rows)
        assert np.array_equal(got, want), rows
    # a marker seeded only in the last row: everything propagates upwards
    # through every cut after the earlier slabs were already copied back
    I = np.full((1024, 256), 200, np.uint8)
    I[::3, 1:] = 0  # a serpentine corridor
    M = np.zeros_like(I)
    M[-1, 0] = 200
    want = oracle.recon_fh(M, I, conn)
    for rows in (32, 64):
        assert np.array_equal(gw.reconstruct(M, I, conn, pipeline_rows=rows), want)


def test_host_pipeline_4k_auto(gw):
    """The auto slab height at BASELINE configs[1] (4096^2 u8)."""
    J, I = oracle.gray_pair(4096, 0, h=40)
    want = oracle.recon_fh(J, I, 8)
    assert np.array_equal(gw.reconstruct(J, I, 8), want)


@pytest.mark.parametrize("conn", [8, 4])
def test_host_pipeline_repeated_runs_agree(gw, conn):
    """Race guard: the pipelined host path runs the engine once per slab
    over growing heights, with tiles re-popped across runs; 24 calls on
    the same input must all give the oracle's image (a lost update between
    a tile's finish and its next owner showed up here as 1-3 wrong pixels
    in ~15% of calls before it was fixed)."""
    J, I = oracle.gray_pair(4096, 0, h=40)
    want = oracle.recon_fh(J, I, conn)
    bad = sum(not np.array_equal(gw.reconstruct(J, I, conn), want) for _ in range(24))
    assert bad == 0


@pytest.mark.parametrize("kind", ["i32", "u16"])
def test_device_repeated_runs_agree_wide(gw, kind):
    """The same guard for the 32-bit register engine (device-resident)."""
    import torch
    dt = np.int32 if kind == "i32" else np.uint16
    J, I = oracle.gray_pair(2048, 5, h=(1 << 27) if kind == "i32" else 5000, dtype=dt)
    want = oracle.recon_fh(J, I, 8)
    dJ, dI = torch.from_numpy(J).cuda(), torch.from_numpy(I).cuda()
    bad = sum(not np.array_equal(gw.reconstruct(dJ, dI, 8).cpu().numpy(), want) for _ in range(16))
    assert bad == 0


@pytest.mark.parametrize("row", [0, 63, 64, 300, 590])
def test_host_pipeline_contract_in_any_slab(gw, row):
    # the violation counter must survive every later engine run (the first
    # slab's count used to be wiped by the next run's counter reset)
    J, I = oracle.gray_pair((600, 128), 4, h=40)
    J[row, 100] = 255
    I[row, 100] = 3
    with pytest.raises(gw.ContractViolation):
        gw.reconstruct(J, I, 8, pipeline_rows=64)
    # default slab heights (~4 MB per slab): violation in the first slab
    J, I = oracle.gray_pair((4096, 2048), 5, h=40)
    J[0, 7] = 9
    I[0, 7] = 8
    with pytest.raises(gw.ContractViolation):
        gw.reconstruct(J, I, 8)


# ---------------------------------------------------------------------------
# f32 (a reference Image2D kind): the int32 engine on order-preserving bits

@pytest.mark.parametrize("conn", [4, 8])
def test_f32_random_vs_oracle(gw, conn):
    rng = np.random.default_rng(300 + conn)
    for shape in [(1, 1), (37, 300), (257, 129), (1024, 768)]:
        I = (rng.standard_normal(shape) * 1e3).astype(np.float32)
        I[::7, ::5] = np.float32(-1e30)  # deep negatives
        J = (I - np.float32(250.0)).astype(np.float32)
        want = oracle.recon_fh(J, I, conn)
        got_d = gw.reconstruct(_torch().from_numpy(J).cuda(), _torch().from_numpy(I).cuda(), conn)
        assert got_d.cpu().numpy().tobytes() == want.tobytes(), shape
        got_h = gw.reconstruct(J, I, conn)  # host path (C ABI, H2D/D2H inside)
        assert got_h.tobytes() == want.tobytes(), shape


def test_f32_operator_api_and_nan_contract(gw):
    rng = np.random.default_rng(5)
    I = rng.random((64, 80)).astype(np.float32)
    J = (I * np.float32(0.5)).astype(np.float32)
    want = oracle.recon_fh(J, I, 8)
    for device in (False, True):
        out = gw.recon_fh(_pair(gw, J, I, 8, "f32", device))
        assert out.elem_kind == "f32"
        assert _np(out.data).tobytes() == want.tobytes()
    Jn = J.copy()
    Jn[3, 3] = np.nan  # NaN <= x is false: recon.py:60 rejects it
    for device in (False, True):
        with pytest.raises(gw.ContractViolation):
            _pair(gw, Jn, I, 8, "f32", device)


# ---------------------------------------------------------------------------
# the u8 tile engines (register Jacobi engine on the tile queue = auto;
# shared-memory queue engine; register engine in level-synchronous tile
# rounds, which needs 16-byte aligned rows) on the same inputs

@pytest.mark.parametrize("engine", [1, 2, 3])
@pytest.mark.parametrize("conn", [4, 8])
def test_u8_engines_vs_oracle(gw, engine, conn):
    t = _torch()
    rng = np.random.default_rng(700 + conn)
    cases = [oracle.gray_pair(s, int(rng.integers(1 << 30)), h=40)
             for s in [(1, 1), (31, 33), (64, 64), (97, 130), (513, 257), (1000, 999),
                       (96, 176), (1040, 2048)]]
    bw = oracle.gen_synthetic_mask(700, 530, 50, 7)
    cases.append(oracle.imfill_pair(bw))
    I = np.full((300, 260), 200, np.uint8)
    I[::3, 1:] = 0  # long corridor
    M = np.zeros_like(I)
    M[-1, 0] = 200
    cases.append((M, I))
    I = np.full((320, 256), 200, np.uint8)  # the corridor with aligned rows
    I[::3, 1:] = 0
    M = np.zeros_like(I)
    M[-1, 0] = 200
    cases.append((M, I))
    for J, I in cases:
        want = oracle.recon_fh(J, I, conn)
        got = gw.reconstruct(t.from_numpy(J).cuda(), t.from_numpy(I).cuda(), conn, engine=engine)
        assert np.array_equal(got.cpu().numpy(), want), (J.shape, engine, conn)
        got = gw.reconstruct(J, I, conn, engine=engine, pipeline_rows=64)
        assert np.array_equal(got, want), (J.shape, engine, conn, "host")


# ---------------------------------------------------------------------------
# the binary kind (0 / 255): one-bit-per-pixel engine vs the grey engines

@pytest.mark.parametrize("conn", [4, 8])
def test_binary_engine_vs_oracle(gw, conn):
    t = _torch()
    rng = np.random.default_rng(900 + conn)
    cases = []
    for shape, cov in [((1, 1), 0.5), ((33, 65), 0.6), ((257, 300), 0.55), ((1000, 999), 0.5)]:
        mask = (rng.random(shape) < cov).astype(np.uint8) * 255
        marker = np.where((rng.random(shape) < 0.02) & (mask == 255), 255, 0).astype(np.uint8)
        cases.append((marker, mask))
    for n, cov in [(700, 50), (1024, 30)]:
        cases.append(oracle.imfill_pair(oracle.gen_synthetic_mask(n, n + 37, cov, 7)))
    for marker, mask in cases:
        want = oracle.recon_fh(marker, mask, conn)
        got = gw.reconstruct(t.from_numpy(marker).cuda(), t.from_numpy(mask).cuda(), conn,
                             kind="binary")
        assert np.array_equal(got.cpu().numpy(), want), marker.shape
        got = gw.reconstruct(marker, mask, conn, kind="binary", pipeline_rows=64)
        assert np.array_equal(got, want), (marker.shape, "host")
        out = gw.recon_fh(_pair(gw, marker, mask, conn, "binary", True))
        assert np.array_equal(_np(out.data), want)


def _serpentine(H, W, pitch=3):
    """A one-pixel-wide corridor snaking down the image (rows every `pitch`,
    joined alternately at the right and left ends) and its far-end marker:
    the fill must cross every 128 x 128 bit tile many times."""
    mask = np.zeros((H, W), np.uint8)
    rows = list(range(1, H - 1, pitch))
    for k, y in enumerate(rows):
        mask[y, 1:W - 1] = 255
        if k + 1 < len(rows):
            x = W - 2 if k % 2 == 0 else 1
            mask[y:rows[k + 1] + 1, x] = 255
    marker = np.zeros_like(mask)
    marker[rows[0], 1] = 255
    return marker, mask


@pytest.mark.parametrize("conn", [4, 8])
def test_binary_engine_long_paths(gw, conn):
    """The 128 x 128 bit-tile engine on inputs whose propagation crosses
    tiles, words and 32-row quarters many times: a serpentine corridor on a
    TMA-staged width (W % 128 == 0) and on a per-lane width, a diagonal
    staircase (8-conn corner hops), and near-percolation random masks in
    wide and tall shapes -- all against the oracle."""
    t = _torch()
    rng = np.random.default_rng(77 + conn)
    cases = [_serpentine(389, 640), _serpentine(389, 600, pitch=4)]
    st = np.zeros((700, 768), np.uint8)  # a staircase: diagonal steps of 1 px
    for i in range(0, 690):
        st[i, i % 768] = 255
        st[i, (i + 1) % 768] = 255
    m0 = np.zeros_like(st)
    m0[0, 0] = 255
    cases.append((m0, st))
    for shape in [(130, 2048), (2048, 130), (384, 640)]:
        mask = (rng.random(shape) < 0.6).astype(np.uint8) * 255
        marker = np.where((rng.random(shape) < 0.001) & (mask == 255), 255, 0).astype(np.uint8)
        cases.append((marker, mask))
    for marker, mask in cases:
        want = oracle.recon_fh(marker, mask, conn)
        got = gw.reconstruct(t.from_numpy(marker).cuda(), t.from_numpy(mask).cuda(), conn,
                             kind="binary")
        assert np.array_equal(got.cpu().numpy(), want), marker.shape
        got = gw.reconstruct(marker, mask, conn, kind="binary", pipeline_rows=128)
        assert np.array_equal(got, want), (marker.shape, "host")


def test_reconstruct_validates_raw_inputs(gw):
    """reconstruct() on raw arrays checks shape, dtype and residency before
    any kernel reads the buffers (an int32 marker with a u8 mask, or a
    smaller mask, would otherwise be read out of bounds)."""
    t = _torch()
    J, I = oracle.gray_pair(64, 2, h=40)
    dJ, dI = t.from_numpy(J).cuda(), t.from_numpy(I).cuda()
    with pytest.raises(gw.ContractViolation):
        gw.reconstruct(dJ.int(), dI, 8)
    with pytest.raises(gw.ContractViolation):
        gw.reconstruct(dJ, dI[:32], 8)
    with pytest.raises(gw.ContractViolation):
        gw.reconstruct(dJ, I, 8)  # device marker, host mask
    with pytest.raises(gw.ContractViolation):
        gw.reconstruct(t.from_numpy(J), t.from_numpy(I), 8)  # CPU tensors
    with pytest.raises(gw.ContractViolation):
        gw.reconstruct(J, I.astype(np.uint16), 8)
    with pytest.raises(gw.ContractViolation):
        gw.reconstruct(dJ, dI, 6)
    assert np.array_equal(gw.reconstruct(dJ, dI, 8).cpu().numpy(), oracle.recon_fh(J, I, 8))


# ---------------------------------------------------------------------------
# iwpp_recon_opts.marker: J is output only (its old contents never matter),
# the marker is not modified; the fused u8 engine copies it in its prologue,
# every other path copies it first.  Unaligned views take the byte path.

@pytest.mark.parametrize("conn", [4, 8])
def test_marker_option_every_path(gw, conn):
    t = _torch()
    from paper_1209_3314_b200 import _lib
    L = _lib.lib()
    rng = np.random.default_rng(1300 + conn)
    cases = []
    for shape, dt, h, code, eng in [((64, 64), np.uint8, 40, 0, 0),        # few tiles: init kernel
                                    ((1040, 2048), np.uint8, 40, 0, 0),    # fused prologue copy
                                    ((1000, 999), np.uint8, 40, 0, 0),     # unaligned rows
                                    ((1040, 2048), np.uint8, 40, 0, 3),    # rounds engine
                                    ((520, 512), np.uint8, 40, 0, 1),      # shared-memory engine
                                    ((300, 256), np.uint16, 9000, 1, 0),
                                    ((300, 256), np.int32, 1 << 27, 2, 0)]:
        J, I = oracle.gray_pair(shape, int(rng.integers(1 << 30)), h=h, dtype=dt)
        cases.append((J, I, code, eng, 0))
        cases.append((J, I, code, eng, 1))  # views one element off the allocation start
    bw = oracle.gen_synthetic_mask(700, 530, 50, 7)
    Jb, Ib = oracle.imfill_pair(bw)
    cases.append((Jb, Ib, 4, 0, 0))
    If = rng.standard_normal((200, 256)).astype(np.float32)
    cases.append(((If - 0.7).astype(np.float32), If, 3, 0, 0))
    for J, I, code, eng, off in cases:
        H, W = J.shape
        want = oracle.recon_fh(J, I, conn)
        dt = t.from_numpy(J).dtype
        bufs = [t.empty(W * H + off, dtype=dt, device="cuda") for _ in range(3)]
        dM, dI, dO = (b[off:].view(H, W) for b in bufs)
        dM.copy_(t.from_numpy(J))
        dI.copy_(t.from_numpy(I))
        dO.fill_(0x5A if code != 3 else 1e30)  # garbage: J is output only
        ws = _lib.workspace(L.iwpp_recon_workspace_bytes(W, H, code, conn))
        o = gw.recon._opts(None, engine=eng)
        o.marker = _lib.ptr(dM)
        _lib.check(L.iwpp_recon(_lib.ptr(dO), _lib.ptr(dI), W, H, code, conn, _lib.ptr(ws), ws.numel(),
                                _lib.ctypes.byref(o), None, _lib.stream_ptr()), "recon")
        assert np.array_equal(dO.cpu().numpy(), want), (J.shape, J.dtype, code, eng, off)
        assert np.array_equal(dM.cpu().numpy(), J), "marker modified"
        # marker == J: in place, as without the option
        o.marker = _lib.ptr(dM)
        _lib.check(L.iwpp_recon(_lib.ptr(dM), _lib.ptr(dI), W, H, code, conn, _lib.ptr(ws), ws.numel(),
                                _lib.ctypes.byref(o), None, _lib.stream_ptr()), "recon")
        assert np.array_equal(dM.cpu().numpy(), want), (J.shape, code, eng, off, "in place")


# ---------------------------------------------------------------------------
# iwpp_recon_host into a page-locked output: the last transfer (the last slab
# and every re-written tile row) is written by the SMs into mapped host
# memory instead of copies after a host read of the dirty flags.

def _recon_host_pinned(M, I, conn, rows, code=0):
    import torch
    from paper_1209_3314_b200 import _lib
    L = _lib.lib()
    H, W = M.shape
    pm, pi = torch.from_numpy(M.copy()).pin_memory(), torch.from_numpy(I.copy()).pin_memory()
    po = torch.from_numpy(np.full_like(M, 0x5A)).pin_memory()
    ws = _lib.workspace(L.iwpp_recon_host_workspace_bytes(W, H, code, conn))
    o = gw_opts(rows)
    st = _lib.Stats()
    _lib.check(L.iwpp_recon_host(_lib.ptr(po.numpy()), _lib.ptr(pm.numpy()), _lib.ptr(pi.numpy()), W, H, code,
                                 conn, _lib.ptr(ws), ws.numel(), _lib.ctypes.byref(o), _lib.ctypes.byref(st),
                                 _lib.stream_ptr()), "recon_host")
    return po.numpy().copy(), st.as_dict()


def gw_opts(rows):
    from paper_1209_3314_b200.recon import _opts
    return _opts(None, pipeline_rows=rows)


@pytest.mark.parametrize("conn", [4, 8])
def test_host_pipeline_pinned_output(gw, conn):
    cases = [oracle.gray_pair((1000, 300), 11, h=40), oracle.gray_pair((513, 704), 12, h=40),
             oracle.gray_pair(4096, 0, h=40)]
    cases.append(oracle.imfill_pair(oracle.gen_synthetic_mask(512, 2048, 50, 7)))
    I = np.full((1024, 256), 200, np.uint8)
    I[::3, 1:] = 0  # serpentine corridor: every cut re-written after its slab went back
    M = np.zeros_like(I)
    M[-1, 0] = 200
    cases.append((M, I))
    for M, I in cases:
        want = oracle.recon_fh(M, I, conn)
        for rows in (0, 64, 128):
            got, st = _recon_host_pinned(M, I, conn, rows)
            assert np.array_equal(got, want), (M.shape, rows)
            assert st["contract_violations"] == 0
    # the contract check still raises (violation in the first and in the last slab)
    M, I = oracle.gray_pair((1024, 256), 13, h=40)
    for row in (0, 1023):
        bad = M.copy()
        bad[row, 7] = 255
        I2 = I.copy()
        I2[row, 7] = 0
        with pytest.raises(Exception):
            _recon_host_pinned(bad, I2, conn, 64)


@pytest.mark.parametrize("dt,code,h", [(np.uint16, 1, 9000), (np.int32, 2, 1 << 27)])
def test_host_pipeline_pinned_output_wide(gw, dt, code, h):
    """The mapped last transfer for the 16/32-bit kinds (row bytes 2 / 4 x W)."""
    for shape, rows in [((1000, 300), 64), ((1024, 512), 0), ((777, 130), 128)]:
        M, I = oracle.gray_pair(shape, 21, h=h, dtype=dt)
        want = oracle.recon_fh(M, I, 8)
        got, st = _recon_host_pinned(M, I, 8, rows, code=code)
        assert np.array_equal(got, want), (shape, rows, dt)
