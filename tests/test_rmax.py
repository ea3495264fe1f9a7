"""regional_maxima (host helper) against the reference's own outputs
(tests/golden/make_rmax_golden.py), plus a many-distinct-values case that
used to take one labelling pass per value."""
import os
import time

import numpy as np

from paper_1209_3314_b200 import Image2D, StructuringElement, regional_maxima

GOLD = os.path.join(os.path.dirname(__file__), "golden", "rmax_golden.npz")
KIND = {np.dtype(np.uint8): "u8", np.dtype(np.uint16): "u16", np.dtype(np.float32): "f32"}


def _packed(a, conn):
    got = regional_maxima(Image2D(a.shape[1], a.shape[0], KIND[a.dtype], a), StructuringElement(conn))
    return np.array([c.y * a.shape[1] + c.x for c in got], np.int64)


def test_regional_maxima_matches_reference_golden():
    g = np.load(GOLD)
    n = len([k for k in g.files if k.endswith("_img")])
    assert n >= 16
    for k in range(n):
        a, conn = g[f"c{k}_img"], int(g[f"c{k}_conn"])
        assert np.array_equal(_packed(a, conn), g[f"c{k}_max"]), f"case {k} conn {conn}"


def test_regional_maxima_many_values_is_linear():
    rng = np.random.default_rng(3)
    a = rng.integers(0, 1 << 16, (512, 512)).astype(np.uint16)  # ~60K distinct values
    t = time.perf_counter()
    got = _packed(a, 8)
    assert time.perf_counter() - t < 20.0
    # a strict maximum of its 3x3 window is a (single-cell) regional maximum
    P = np.pad(a.astype(np.int64), 1, constant_values=-1)
    win = np.stack([P[1 + dy:513 + dy, 1 + dx:513 + dx] for dy in (-1, 0, 1) for dx in (-1, 0, 1)
                    if dy or dx])
    strict = np.nonzero(((win < a).all(0)).ravel())[0]
    assert np.isin(strict, got).all()
