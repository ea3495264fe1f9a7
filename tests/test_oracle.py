"""Pin the CPU oracle (oracle/iwpp_oracle.c) to the reference's own outputs.

The golden vectors in tests/golden/*.npz were produced by the reference
implementation (gridwave) by tests/golden/make_golden.py.  Every case must
match bit for bit; EDT cases compare the int64 source map and the float32
distance bytes.
"""

import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _cases(path, suffix):
    z = np.load(os.path.join(GOLD, path))
    names = sorted({k.split("__")[0] for k in z.files if k.endswith(suffix)})
    return z, names


RZ, RNAMES = _cases("recon_golden.npz", "__out")
EZ, ENAMES = _cases("edt_golden.npz", "__vr")


def _conn(name):
    return 8 if name.endswith("c8") else 4


@pytest.mark.parametrize("name", RNAMES)
def test_oracle_recon_fh_matches_reference(name):
    J, I, R = RZ[name + "__marker"], RZ[name + "__mask"], RZ[name + "__out"]
    got = oracle.recon_fh(J, I, _conn(name))
    assert got.dtype == R.dtype
    assert np.array_equal(got, R)


@pytest.mark.parametrize("name", [n for n in RNAMES if n.startswith(("u8_64", "bin", "zig"))])
def test_oracle_recon_sr_and_dilation_agree(name):
    J, I, R = RZ[name + "__marker"], RZ[name + "__mask"], RZ[name + "__out"]
    assert np.array_equal(oracle.recon_sr(J, I, _conn(name)), R)
    assert np.array_equal(oracle.recon_by_dilation(J, I, _conn(name)), R)


@pytest.mark.parametrize("name", ENAMES)
def test_oracle_edt_matches_reference(name):
    m, vr_ref, d_ref = EZ[name + "__mask"], EZ[name + "__vr"], EZ[name + "__dist"]
    vr, dist = oracle.edt(m, _conn(name))
    assert np.array_equal(vr, vr_ref)
    if np.isnan(d_ref).all():
        assert dist is None  # no background -> NoBackgroundError in the reference
    else:
        assert dist.tobytes() == d_ref.tobytes()


def test_oracle_adversarial_relay_gap():
    vr = EZ["adversarial24_c4__vr"]
    d2 = oracle.squared_distances(vr)
    ex = oracle.bruteforce_sqdist(EZ["adversarial24_c4__mask"])
    assert d2[21, 5] == 170 and ex[21, 5] == 169
    assert np.array_equal(ex, EZ["adversarial24__exact_d2"])
    assert int((d2 > ex).sum()) == 1


def test_oracle_edt_propagate_dedupe_invariant():
    """Deduplicating round items never changes the map."""
    m = EZ["blob256_c8__mask"]
    vr, seeds = oracle.edt_init(m, 8)
    seeds2 = np.concatenate([seeds, seeds[::-1]])
    oracle.edt_propagate(vr, seeds2, 8)
    assert np.array_equal(vr, EZ["blob256_c8__vr"])


def test_oracle_seed_scan_finds_leftover_work():
    J, I = oracle.gray_pair(32, 5, h=60)
    s = oracle.recon_seed_scan(J, I, 8)
    J2 = J.copy()
    oracle.recon_wavefront(J2, I, 8, s)
    assert np.array_equal(J2, oracle.recon_by_dilation(J, I, 8))


def test_single_passes_match_reference_golden():
    """oracle.recon_pass (K.38-190) against the reference's own raster_pass,
    _antiraster_packed (seeds in sweep order) and one-band parallel_sweeps
    (tests/golden/make_pass_golden.py)."""
    g = np.load(os.path.join(GOLD, "pass_golden.npz"))
    n = len({k[:4] for k in g.files})
    assert n == 24
    for c in range(n):
        p = f"c{c:03d}_"
        J, I, conn = g[p + "J"], g[p + "I"], int(g[p + "conn"])
        a = J.copy()
        ch, _ = oracle.recon_pass(a, I, conn, 0)
        assert np.array_equal(a, g[p + "raster"]) and ch == bool(g[p + "raster_changed"])
        ch, seeds = oracle.recon_pass(a, I, conn, 1)
        assert np.array_equal(a, g[p + "anti"]) and ch == bool(g[p + "anti_changed"])
        assert np.array_equal(seeds, g[p + "anti_seeds"])
        b = J.copy()
        for pas in (2, 3, 4, 5):
            oracle.recon_pass(b, I, conn, pas)
        assert np.array_equal(b, g[p + "sweeps"])
