"""The rest of the reference's operator surface on the B200: the single
scan passes (raster / anti-raster with seeds / one-band parallel sweeps)
cell for cell against the reference's golden vectors and the oracle, the
wave pipeline (run_pipeline with both rules, recon_tiled / edt_tiled on
it), and EngineConfig.max_rounds for reconstruction."""

import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
KIND = {np.uint8: "u8", np.uint16: "u16", np.int32: "i32", np.float32: "f32"}


@pytest.fixture(scope="module")
def gw():
    import torch
    import paper_1209_3314_b200 as gw
    torch.cuda.set_device(0)
    return gw


def _img(gw, a, device):
    import torch
    data = torch.from_numpy(a.copy()).cuda() if device else a.copy()
    return gw.Image2D(a.shape[1], a.shape[0], KIND[a.dtype.type], data)


def _np(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


@pytest.mark.parametrize("device", [False, True])
def test_passes_match_reference_golden(gw, device):
    from paper_1209_3314_b200 import recon
    g = np.load(os.path.join(GOLD, "pass_golden.npz"))
    for c in range(24):
        p = f"c{c:03d}_"
        J, I, conn = g[p + "J"], g[p + "I"], int(g[p + "conn"])
        inp = gw.ReconInput(_img(gw, J, device), _img(gw, I, device), gw.StructuringElement(conn))
        assert recon.raster_pass(inp) == bool(g[p + "raster_changed"])
        assert np.array_equal(_np(inp.marker.data), g[p + "raster"]), c
        ch, seeds = recon._antiraster_packed(inp, True)
        assert ch == bool(g[p + "anti_changed"])
        assert np.array_equal(_np(inp.marker.data), g[p + "anti"]), c
        assert np.array_equal(_np(seeds), g[p + "anti_seeds"]), c
        Jw = _img(gw, J, device).data
        recon.parallel_sweeps(Jw, _img(gw, I, device).data, gw.StructuringElement(conn), 3)
        assert np.array_equal(_np(Jw), g[p + "sweeps"]), c


@pytest.mark.parametrize("conn", [4, 8])
@pytest.mark.parametrize("shape", [(37, 9000), (9000, 23), (300, 257)])
def test_passes_match_oracle_across_chunks(gw, conn, shape):
    """Rows / columns longer than one 8192-element chunk of the line scan."""
    import torch
    from paper_1209_3314_b200 import recon
    for dtype in (np.uint8, np.int32):
        J, I = oracle.gray_pair(shape, 5 + conn, h=40 if dtype == np.uint8 else 1 << 27,
                                dtype=dtype)
        for pas in range(6):
            want = J.copy()
            wch, wseeds = oracle.recon_pass(want, I, conn, pas)
            got = torch.from_numpy(J.copy()).cuda()
            ch, seeds = recon._run_pass(got, torch.from_numpy(I).cuda(), conn, pas, pas == 1)
            assert np.array_equal(got.cpu().numpy(), want), (pas, dtype)
            assert ch == wch
            if pas == 1:
                assert np.array_equal(seeds.cpu().numpy(), wseeds)


def test_antiraster_pass_coords_and_window_sweeps(gw):
    from paper_1209_3314_b200 import recon
    J, I = oracle.gray_pair((20, 30), 3, h=40)
    inp = gw.ReconInput(_img(gw, J, False), _img(gw, I, False), gw.SE8)
    ch, coords = recon.antiraster_pass(inp, collect_seeds=True)
    a = J.copy()
    _, s = oracle.recon_pass(a, I, 8, 1)
    assert coords == [gw.unpack(int(p), 30) for p in s]
    # bounds: the sweeps see only the window
    Jw = J.copy()
    recon.parallel_sweeps(Jw, I, gw.SE8, 1, bounds=(5, 2, 25, 17))
    sub = J[2:17, 5:25].copy()
    for pas in (2, 3, 4, 5):
        oracle.recon_pass(sub, np.ascontiguousarray(I[2:17, 5:25]), 8, pas)
    want = J.copy()
    want[2:17, 5:25] = sub
    assert np.array_equal(Jw, want)


def _zigzag():
    I = np.zeros((16, 16), np.uint8)
    I[1, 1:15] = 100
    I[1:14, 14] = 100
    I[13, 1:15] = 100
    I[4:14, 1] = 100
    J = np.zeros((16, 16), np.uint8)
    J[1, 1] = 100
    return J, I


@pytest.mark.parametrize("device", [False, True])
def test_run_pipeline_recon_rule_in_place(gw, device):
    """test_tiles.py:262-288 analogue: the rule's J is the reconstruction."""
    J, I = _zigzag()
    img = _img(gw, J, device)
    rule = gw.ReconRule(img.data, _img(gw, I, device).data, gw.SE8)
    cfg = gw.PipelineConfig(n_workers=2)
    out = gw.run_pipeline(img, rule, lambda: [1 * 16 + 1], (8, 8), cfg)
    assert out is img
    assert np.array_equal(_np(rule.J), oracle.recon_fh(J, I, 8))
    assert cfg.bp_waves >= 1 and {e.kind for e in cfg.events} == {"TP", "BP"}


def test_run_pipeline_distance_rule_matches_edt(gw):
    m = oracle.gen_synthetic_mask(200, 150, 50, 11)
    mask = gw.Image2D(200, 150, "binary", m)
    for se in (gw.SE4, gw.SE8):
        from paper_1209_3314_b200.edt import init_packed
        vmap, seeds = init_packed(mask, se)
        rule = gw.DistanceRule(vmap.vr, se)
        gw.run_pipeline(vmap, rule, lambda: seeds, (32, 32))
        vr_ref, _ = oracle.edt(m, se.connectivity)
        assert np.array_equal(_np(vmap.vr), vr_ref)


def test_tiled_operators_run_the_pipeline(gw):
    J, I = oracle.gray_pair((300, 200), 9, h=40)
    cfg = gw.PipelineConfig()
    out = gw.recon_tiled(gw.ReconInput(_img(gw, J, False), _img(gw, I, False), gw.SE8), (16, 16), cfg)
    assert np.array_equal(out.data, oracle.recon_fh(J, I, 8)) and cfg.bp_waves == 1
    with pytest.raises(gw.ContractViolation):
        gw.recon_tiled(gw.ReconInput(_img(gw, J, False), _img(gw, I, False), gw.SE8), (16, 16),
                       gw.PipelineConfig(max_waves=0))
    m = oracle.gen_synthetic_mask(120, 90, 50, 5)
    vm, d = gw.edt_tiled(gw.Image2D(120, 90, "binary", m), gw.SE8, (16, 16))
    vr_ref, d_ref = oracle.edt(m, 8)
    assert np.array_equal(_np(vm.vr), vr_ref) and _np(d.data).tobytes() == d_ref.tobytes()


def test_recon_max_rounds_engine_error(gw):
    """engine.py:311-317: EngineError when the fixed point needs more rounds
    than EngineConfig.max_rounds (the tile-rounds engine counts them)."""
    import torch
    I = np.full((64, 4096), 200, np.uint8)  # a corridor across many tiles
    I[::3, 1:] = 0
    J = np.zeros_like(I)
    J[-1, 0] = 200
    inp = gw.ReconInput(_img(gw, J, True), _img(gw, I, True), gw.SE8)
    with pytest.raises(gw.EngineError):
        gw.recon_parallel(inp, gw.EngineConfig(max_rounds=2))
    cfg = gw.EngineConfig(max_rounds=10 ** 6)
    out = gw.recon_parallel(inp, cfg)
    assert np.array_equal(_np(out.data), oracle.recon_fh(J, I, 8))
    assert cfg.stats.rounds >= 3
