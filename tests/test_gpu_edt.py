"""EDT parity on the B200 through the public API and the C ABI.

Source maps (int64), squared distances and float32 distance bytes must be
bit-identical to the reference's canonical round schedule (golden vectors
from gridwave + the CPU oracle).  Mirrors pkg/tests/test_edt.py and
test_acceptance.py C5/C6."""

import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
EZ = np.load(os.path.join(GOLD, "edt_golden.npz"))
ENAMES = sorted({k.split("__")[0] for k in EZ.files if k.endswith("__vr")})


@pytest.fixture(scope="module")
def gw():
    import torch
    import paper_1209_3314_b200 as gw
    torch.cuda.set_device(0)
    return gw


def _t():
    import torch
    return torch


def _np(a):
    return a.cpu().numpy() if hasattr(a, "cpu") else a


def _img(gw, m, device):
    d = _t().from_numpy(np.ascontiguousarray(m)).cuda() if device else np.ascontiguousarray(m)
    return gw.Image2D(m.shape[1], m.shape[0], "binary", d)


@pytest.mark.parametrize("device", [False, True])
@pytest.mark.parametrize("name", ENAMES)
def test_golden_vectors(gw, name, device):
    m, vr_ref, d_ref = EZ[name + "__mask"], EZ[name + "__vr"], EZ[name + "__dist"]
    se = gw.StructuringElement(8 if name.endswith("c8") else 4)
    img = _img(gw, m, device)
    if np.isnan(d_ref).all():
        with pytest.raises(gw.NoBackgroundError):
            gw.edt(img, se)
        vmap, seeds = gw.init_packed(img, se)
        gw.edt_propagate(vmap, seeds, se)
        assert np.array_equal(_np(vmap.vr), vr_ref)
        return
    for mode in ("sequential", "parallel"):
        vmap, dist = gw.edt(img, se, mode=mode)
        assert np.array_equal(_np(vmap.vr), vr_ref)
        assert _np(dist.data).tobytes() == d_ref.tobytes()


@pytest.mark.parametrize("conn", [4, 8])
def test_random_masks_vs_oracle(gw, conn):
    rng = np.random.default_rng(1005 + conn)
    for i in range(12):
        shape = [(64, 64), (97, 131), (256, 256), (1, 500), (500, 1), (300, 200)][i % 6]
        cov = [0.25, 0.5, 0.75, 0.95][i % 4]
        m = (rng.random(shape) < cov).astype(np.uint8) * 255
        if not (m == 0).any():
            m.flat[0] = 0
        vr_ref, d_ref = oracle.edt(m, conn)
        vmap, dist = gw.edt(_img(gw, m, True), gw.StructuringElement(conn))
        assert np.array_equal(_np(vmap.vr), vr_ref), (shape, cov)
        assert _np(dist.data).tobytes() == d_ref.tobytes()


@pytest.mark.parametrize("conn", [4, 8])
def test_blob_1k_vs_oracle(gw, conn):
    m = oracle.gen_synthetic_mask(1024, 1024, 50, 7)
    vr_ref, d_ref, (rounds, _) = oracle.edt(m, conn, stats=True)
    cfg = gw.EngineConfig()
    vmap, dist = gw.edt(_img(gw, m, True), gw.StructuringElement(conn), mode="parallel", cfg=cfg)
    assert np.array_equal(_np(vmap.vr), vr_ref)
    assert _np(dist.data).tobytes() == d_ref.tobytes()
    assert cfg.stats.rounds == rounds


@pytest.mark.slow
def test_nuclei_4k_vs_oracle(gw):
    """BASELINE configs[2] at full size: 4096^2 nuclei-like mask, SE8."""
    m = oracle.gen_nuclei_mask(4096, 4096, 30.0, 7)
    vr_ref, d_ref = oracle.edt(m, 8)
    vmap, dist = gw.edt(_img(gw, m, True), gw.SE8)
    assert np.array_equal(_np(vmap.vr), vr_ref)
    assert _np(dist.data).tobytes() == d_ref.tobytes()


def test_all_foreground_raises_and_all_background_is_identity(gw):
    with pytest.raises(gw.NoBackgroundError):
        gw.edt(_img(gw, np.full((4, 4), 255, np.uint8), True))
    vmap, dist = gw.edt(_img(gw, np.zeros((5, 7), np.uint8), True))
    assert np.array_equal(_np(vmap.vr), np.arange(35).reshape(5, 7))
    assert not _np(dist.data).any()


def test_edt_propagate_user_seeds_duplicates_and_coords(gw):
    m = oracle.gen_synthetic_mask(200, 160, 50, 3)
    vr_ref, _ = oracle.edt(m, 8)
    vmap, seeds = gw.init_packed(_img(gw, m, False), gw.SE8)
    seeds2 = np.concatenate([seeds, seeds[::-1]])
    gw.edt_propagate(vmap, seeds2, gw.SE8)
    assert np.array_equal(vmap.vr, vr_ref)
    vmap, coords = gw.edt_init(_img(gw, m, False), gw.SE8)
    gw.edt_propagate(vmap, coords, gw.SE8, mode="parallel")
    assert np.array_equal(vmap.vr, vr_ref)


def test_init_matches_reference_init(gw):
    m = EZ["blob256_c8__mask"]
    vr0, seeds_ref = oracle.edt_init(m, 8)
    vmap, seeds = gw.init_packed(_img(gw, m, True), gw.SE8)
    assert np.array_equal(_np(vmap.vr), vr0)
    assert np.array_equal(_np(seeds), seeds_ref)


def test_max_rounds_raises_engine_error(gw):
    m = oracle.gen_synthetic_mask(256, 256, 50, 7)
    with pytest.raises(gw.EngineError):
        gw.edt(_img(gw, m, True), gw.SE8, mode="parallel", cfg=gw.EngineConfig(max_rounds=3))
    _, _, (rounds, _) = oracle.edt(m, 8, stats=True)
    gw.edt(_img(gw, m, True), gw.SE8, mode="parallel", cfg=gw.EngineConfig(max_rounds=rounds))


def test_finalize_and_squared_distances(gw):
    vr = EZ["adversarial24_c4__vr"]
    vmap = gw.VoronoiMap(24, 24, vr.copy())
    d2 = vmap.squared_distances()
    assert d2[21, 5] == 170
    ex = EZ["adversarial24__exact_d2"]
    assert int((d2 > ex).sum()) == 1 and (d2 >= ex).all()
    dist = gw.finalize_distance_map(vmap)
    assert np.array_equal(dist.data, np.sqrt(d2).astype(np.float32))
    bad = gw.VoronoiMap(2, 2, np.array([[0, -1], [0, 0]], np.int64))
    with pytest.raises(gw.NoBackgroundError):
        gw.finalize_distance_map(bad)


def test_three_four_five_and_single_source_exact(gw):
    a = np.full((8, 8), 255, np.uint8)
    a[0, 0] = 0
    _, dist = gw.edt(_img(gw, a, True))
    assert _np(dist.data)[4, 3] == np.float32(5.0)
    rng = np.random.default_rng(53)
    for _ in range(5):
        a = np.full((33, 29), 255, np.uint8)
        a[rng.integers(0, 33), rng.integers(0, 29)] = 0
        _, dist = gw.edt(_img(gw, a, True))
        ex = gw.edt_exact_bruteforce(_img(gw, a, False))
        assert np.array_equal(_np(dist.data), ex.data)


def test_tie_cases_counted_against_exact(gw):
    """Order-dependent cases: the propagated map may exceed the exact EDT
    (SURVEY 8c); the excess is counted and bounded below by exact."""
    m = oracle.gen_synthetic_mask(256, 256, 50, 7)
    for conn in (4, 8):
        vmap, _ = gw.edt(_img(gw, m, True), gw.StructuringElement(conn))
        d2 = vmap.squared_distances().cpu().numpy()
        ex = oracle.bruteforce_sqdist(m)
        assert (d2 >= ex).all()
        if conn == 8:
            assert int((d2 > ex).sum()) == 0  # 8-conn refgen mask equals exact


# ---------------------------------------------------------------------------
# engine variants: the 32-bit-source CAS engine (used when a squared distance
# leaves the 32-bit key range) and the range-checked key engine must give the
# same canonical result as the default key engine.

@pytest.fixture
def engine_mode(gw):
    from paper_1209_3314_b200 import _lib
    L = _lib.lib()

    def set_mode(m):
        _lib.check(L.iwpp_edt_set_engine(m), "set_engine")
    yield set_mode
    set_mode(0)


@pytest.mark.parametrize("mode", [1, 2, 3, 4, 5, 6, 7])
@pytest.mark.parametrize("conn", [4, 8])
def test_engine_variants_vs_oracle(gw, engine_mode, mode, conn):
    engine_mode(mode)
    rng = np.random.default_rng(77 + conn)
    masks = [oracle.gen_synthetic_mask(300, 200, 50, 7),
             (rng.random((129, 257)) < 0.9).astype(np.uint8) * 255,
             oracle.gen_synthetic_mask(700, 517, 60, 3)]  # many passes, ragged regions
    for name in ENAMES[:6]:
        if name.endswith("c%d" % conn) and not np.isnan(EZ[name + "__dist"]).all():
            masks.append(EZ[name + "__mask"])
    for m in masks:
        if not (m == 0).any():
            continue
        vr_ref, d_ref = oracle.edt(m, conn)
        vmap, dist = gw.edt(_img(gw, m, True), gw.StructuringElement(conn))
        assert np.array_equal(_np(vmap.vr), vr_ref)
        assert _np(dist.data).tobytes() == d_ref.tobytes()
    # max_rounds through the variant: EngineError exactly when not converged
    m = masks[2]
    _, _, (rounds, _) = oracle.edt(m, conn, stats=True)
    cfg = gw.EngineConfig(max_rounds=rounds)
    gw.edt(_img(gw, m, True), gw.StructuringElement(conn), mode="parallel", cfg=cfg)
    with pytest.raises(gw.EngineError):
        gw.edt(_img(gw, m, True), gw.StructuringElement(conn), mode="parallel",
               cfg=gw.EngineConfig(max_rounds=rounds - 2))
    # edt_propagate through the variant
    m = masks[0]
    vr_ref, _ = oracle.edt(m, conn)
    vmap, seeds = gw.init_packed(_img(gw, m, True), gw.StructuringElement(conn))
    gw.edt_propagate(vmap, seeds, gw.StructuringElement(conn))
    assert np.array_equal(_np(vmap.vr), vr_ref)


def test_key_range_overflow_reruns_exactly(gw):
    """46342^2 with one background cell in a corner: the far corner's d^2 is
    2 * 46341^2 > 2^32, beyond the 64-bit key's d^2 field.  The range-checked
    key run flags it and the CAS engine re-runs; with a single source every
    cell's source is that cell, so the exact answer is known in closed form."""
    t = _t()
    n = 46342
    free = t.cuda.mem_get_info()[0]
    if free < 90 << 30:
        pytest.skip("needs ~90 GB of free device memory")
    m = t.full((n, n), 255, dtype=t.uint8, device="cuda")
    m[0, 0] = 0
    vmap, dist = gw.edt(gw.Image2D(n, n, "binary", m), gw.SE8)
    del m
    assert bool((vmap.vr == 0).all())
    corner = float(np.float32(np.sqrt(np.float64(2 * (n - 1) ** 2))))
    assert float(dist.data[n - 1, n - 1]) == corner
    ys = t.arange(0, n, 4097, device="cuda", dtype=t.float64)
    got = dist.data[::4097, ::4097].double()
    want = t.sqrt(ys[:, None] ** 2 + ys[None, :] ** 2).float().double()
    assert bool((got == want).all())
