"""Generate golden vectors from the REFERENCE implementation (gridwave).

Run in the build container only (the reference is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Writes ``tests/golden/*.npz`` (committed).  Every case stores its inputs
and the reference outputs so the fixtures are self-contained.  Inputs are
generated with the reference's own generators / seeds where it has them
(test_acceptance.py:54-57, imgio.gen_synthetic_mask).
"""

from __future__ import annotations

import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

import gridwave  # noqa: E402
from gridwave import _kernels as K  # noqa: E402
from gridwave.edt import edt, edt_propagate, init_packed  # noqa: E402
from gridwave.grid import Image2D, StructuringElement  # noqa: E402
from gridwave.imgio import gen_synthetic_mask  # noqa: E402
from gridwave.oracles import bruteforce_sqdist  # noqa: E402
from gridwave.recon import ReconInput, recon_fh  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def gray_pair(rng, shape, h):
    I = rng.integers(0, 256, shape).astype(np.uint8)
    J = np.maximum(I.astype(np.int32) - h, 0).astype(np.uint8)
    return J, I


def recon_ref(J, I, conn, kind):
    se = StructuringElement(conn)
    h, w = J.shape
    inp = ReconInput(Image2D(w, h, kind, J.copy()), Image2D(w, h, kind, I.copy()), se)
    return recon_fh(inp).data.copy()


def recon_ref_kernels(J, I, conn):
    """int32 is not an Image2D kind; run the reference kernels directly
    (recon.py:174-182 with K.38-112 and K.220-270)."""
    J = J.copy()
    h, w = J.shape
    c8 = conn == 8
    K.recon_raster_pass(J, I, c8, 0, 0, w, h)
    buf = np.empty(h * w, np.int64)
    _, n = K.recon_antiraster_pass(J, I, c8, 0, 0, w, h, buf, True)
    K.recon_wavefront(J, I, c8, 0, 0, w, h, buf[:n], n)
    return J


def main():
    recon = {}
    # u8 random marker/mask pairs (the bench generator), conn 4/8
    for (n, seed) in [(1, 3), (7, 5), (64, 0), (64, 1001), (256, 0), (512, 0), (512, 1001)]:
        rng = np.random.default_rng(seed)
        J, I = gray_pair(rng, (n, n), 40)
        for conn in (4, 8):
            recon[f"u8_{n}_{seed}_c{conn}"] = (J, I, recon_ref(J, I, conn, "u8"))
    # ragged shapes
    for shape, seed in [((1, 97), 11), ((97, 1), 12), ((33, 130), 13), ((130, 33), 14), ((67, 203), 15)]:
        rng = np.random.default_rng(seed)
        J, I = gray_pair(rng, shape, 60)
        for conn in (4, 8):
            recon[f"u8_{shape[0]}x{shape[1]}_{seed}_c{conn}"] = (J, I, recon_ref(J, I, conn, "u8"))
    # u16
    rng = np.random.default_rng(21)
    I = rng.integers(0, 65536, (96, 80)).astype(np.uint16)
    J = np.maximum(I.astype(np.int64) - 9000, 0).astype(np.uint16)
    for conn in (4, 8):
        recon[f"u16_96x80_21_c{conn}"] = (J, I, recon_ref(J, I, conn, "u16"))
    # int32 (full range) through the reference kernels
    rng = np.random.default_rng(22)
    I = rng.integers(-2**31, 2**31 - 1, (128, 128), dtype=np.int32)
    J = np.maximum(I.astype(np.int64) - 2**28, -2**31).astype(np.int32)
    for conn in (4, 8):
        recon[f"i32_128_22_c{conn}"] = (J, I, recon_ref_kernels(J, I, conn))
    # f32 (a reference Image2D kind): signed values, ties, a flat plateau
    rng = np.random.default_rng(23)
    I = (rng.standard_normal((80, 96)) * 1000.0).astype(np.float32)
    I[10:20, 10:30] = np.float32(12.5)
    J = (I - np.float32(300.0)).astype(np.float32)
    for conn in (4, 8):
        recon[f"f32_80x96_23_c{conn}"] = (J, I, recon_ref(J, I, conn, "f32"))
    # binary: component selection + imfill
    rng = np.random.default_rng(1004)
    for i in range(4):
        mask = (rng.random((48, 48)) < 0.45).astype(np.uint8) * 255
        marker = np.where((rng.random((48, 48)) < 0.06) & (mask == 255), 255, 0).astype(np.uint8)
        for conn in (4, 8):
            recon[f"bin_48_{i}_c{conn}"] = (marker, mask, recon_ref(marker, mask, conn, "binary"))
    bw = gen_synthetic_mask(256, 256, 50, 7).data
    mask = np.where(bw == 0, 255, 0).astype(np.uint8)
    marker = np.zeros_like(mask)
    marker[0, :], marker[-1, :], marker[:, 0], marker[:, -1] = mask[0, :], mask[-1, :], mask[:, 0], mask[:, -1]
    for conn in (4, 8):
        recon[f"imfill_256_7_c{conn}"] = (marker, mask, recon_ref(marker, mask, conn, "binary"))
    # zig-zag corridor (test_tiles.py:262-288)
    I = np.zeros((8, 16), np.uint8)
    I[1, 1:15] = 100
    I[1:6, 14] = 100
    I[5, 1:15] = 100
    J = np.zeros((8, 16), np.uint8)
    J[1, 1] = 100
    recon["zigzag_c8"] = (J, I, recon_ref(J, I, 8, "u8"))

    arrs = {}
    for k, (J, I, R) in recon.items():
        arrs[k + "__marker"] = J
        arrs[k + "__mask"] = I
        arrs[k + "__out"] = R
    np.savez_compressed(os.path.join(OUT, "recon_golden.npz"), **arrs)
    print(f"recon: {len(recon)} cases")

    # ---------------------------------------------------------------- EDT
    cases = {}

    def add(name, mask, conn):
        img = Image2D(mask.shape[1], mask.shape[0], "binary", mask)
        se = StructuringElement(conn)
        if not (mask == 0).any():
            vmap, seeds = init_packed(img, se)
            edt_propagate(vmap, seeds, se)
            cases[name] = (mask, vmap.vr.copy(), np.full(mask.shape, np.nan, np.float32))
            return
        vmap, dist = edt(img, se, mode="sequential")
        cases[name] = (mask, vmap.vr.copy(), dist.data.copy())

    rng = np.random.default_rng(41)
    for i in range(6):
        cov = [0.3, 0.5, 0.7, 0.9, 0.97, 0.995][i]
        m = (rng.random((64, 64)) < cov).astype(np.uint8) * 255
        for conn in (4, 8):
            add(f"rand64_{i}_c{conn}", m, conn)
    for conn in (4, 8):
        add(f"blob256_c{conn}", gen_synthetic_mask(256, 256, 50, 7).data, conn)
        add(f"blob512_c{conn}", gen_synthetic_mask(512, 512, 50, 7).data, conn)
    # adversarial relay gap (test_edt.py:195-206)
    a = np.full((24, 24), 255, np.uint8)
    for x, y in ((1, 8), (17, 16), (18, 20)):
        a[y, x] = 0
    add("adversarial24_c4", a, 4)
    add("adversarial24_c8", a, 8)
    # 3-4-5 triangle / single source (test_edt.py:110-113, 144-148)
    a = np.full((8, 8), 255, np.uint8)
    a[0, 0] = 0
    add("single8_c8", a, 8)
    a = np.full((16, 16), 255, np.uint8)
    a[3, 2] = 0
    add("single16_c4", a, 4)
    add("allbg_c8", np.zeros((4, 4), np.uint8), 8)
    add("allfg_c8", np.full((5, 5), 255, np.uint8), 8)
    # ragged shapes
    for shape, seed in [((1, 77), 3), ((77, 1), 4), ((31, 95), 5), ((95, 31), 6)]:
        m = (np.random.default_rng(seed).random(shape) < 0.8).astype(np.uint8) * 255
        if not (m == 0).any():
            m.flat[0] = 0
        for conn in (4, 8):
            add(f"ragged{shape[0]}x{shape[1]}_c{conn}", m, conn)

    arrs = {}
    for k, (m, vr, dist) in cases.items():
        arrs[k + "__mask"] = m
        arrs[k + "__vr"] = vr
        arrs[k + "__dist"] = dist
    # brute-force exact reference for the adversarial instance
    arrs["adversarial24__exact_d2"] = bruteforce_sqdist(
        cases["adversarial24_c4"][0], 1 << 62)
    np.savez_compressed(os.path.join(OUT, "edt_golden.npz"), **arrs)
    print(f"edt: {len(cases)} cases; gridwave {gridwave.__version__}")


if __name__ == "__main__":
    main()
