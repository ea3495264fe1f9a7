"""Command-line front end on the B200 (reference: gridwave/cli.py; the
cases mirror pkg/tests/test_cli.py for recon / edt), plus a file-to-file
check of the device I/O path against the CPU oracle."""

import numpy as np
import pytest

import oracle
from paper_1209_3314_b200.cli import main
from paper_1209_3314_b200.grid import FG, Image2D
from paper_1209_3314_b200.imgio import read_f32_raw, read_pgm, write_pgm

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _dev():
    import torch
    torch.cuda.set_device(0)


def gray(path, arr):
    a = np.asarray(arr, dtype=np.uint8)
    write_pgm(Image2D(a.shape[1], a.shape[0], "u8", a), str(path))
    return str(path)


def binary(path, arr):
    a = np.asarray(arr, dtype=np.uint8) * FG
    write_pgm(Image2D(a.shape[1], a.shape[0], "binary", a), str(path))
    return str(path)


def test_recon_marker_equals_mask_reproduces_mask(tmp_path):
    rng = np.random.default_rng(1)
    mask = gray(tmp_path / "mask.pgm", rng.integers(0, 256, (16, 16)))
    out = tmp_path / "out.pgm"
    assert main(["recon", "--marker", mask, "--mask", mask, "--out", str(out)]) == 0
    assert out.read_bytes() == (tmp_path / "mask.pgm").read_bytes()


@pytest.mark.parametrize("algo", ["fh", "sr", "qb", "parallel", "tiled", "b200"])
def test_recon_algos_write_the_oracle_result(tmp_path, algo):
    rng = np.random.default_rng(2)
    I = rng.integers(0, 256, (48, 61)).astype(np.uint8)
    mask = gray(tmp_path / "mask.pgm", I)
    out = tmp_path / "o.pgm"
    args = ["recon", "--mask", mask, "--auto-marker", "40", "--out", str(out), "--algo", algo]
    if algo == "tiled":
        args += ["--tile", "16x16", "--workers", "2"]
    if algo == "parallel":
        args += ["--workers", "2", "--queue", "naive"]
    assert main(args) == 0
    J = np.maximum(I.astype(np.int32) - 40, 0).astype(np.uint8)
    want = oracle.recon_fh(J, I, 8)
    assert np.array_equal(read_pgm(str(out)).data, want)


def test_recon_marker_above_mask_exits_2(tmp_path, capsys):
    mask = gray(tmp_path / "mask.pgm", np.full((8, 8), 10))
    marker = gray(tmp_path / "marker.pgm", np.full((8, 8), 200))
    assert main(["recon", "--marker", marker, "--mask", mask,
                 "--out", str(tmp_path / "out.pgm")]) == 2
    assert "error:" in capsys.readouterr().err


def test_recon_missing_file_exits_2(tmp_path):
    assert main(["recon", "--mask", str(tmp_path / "nope.pgm"), "--auto-marker", "40",
                 "--out", str(tmp_path / "out.pgm")]) == 2


def test_recon_malformed_file_exits_2(tmp_path, capsys):
    p = tmp_path / "bad.pgm"
    p.write_bytes(b"P5 4 4 255\n" + bytes(3))
    assert main(["recon", "--mask", str(p), "--auto-marker", "4",
                 "--out", str(tmp_path / "o.pgm")]) == 2
    assert "raster truncated" in capsys.readouterr().err


def test_edt_all_background_writes_zero_map(tmp_path):
    mask = binary(tmp_path / "mask.pgm", np.zeros((12, 12), np.uint8))
    out = tmp_path / "d.f32"
    assert main(["edt", "--input", mask, "--out", str(out)]) == 0
    assert (read_f32_raw(str(out)).data == 0.0).all()


@pytest.mark.parametrize("mode", ["parallel", "tiled"])
def test_edt_modes_write_identical_f32(tmp_path, mode):
    rng = np.random.default_rng(4)
    mask = binary(tmp_path / "mask.pgm", rng.random((48, 48)) < 0.5)
    a, b = tmp_path / "a.f32", tmp_path / "b.f32"
    assert main(["edt", "--input", mask, "--out", str(a), "--mode", "seq"]) == 0
    assert main(["edt", "--input", mask, "--out", str(b), "--mode", mode, "--tile", "16x16"]) == 0
    assert a.read_bytes() == b.read_bytes()


def test_edt_matches_oracle_distances(tmp_path):
    m = oracle.gen_nuclei_mask(300, 257, 30.0, 7)
    mask = binary(tmp_path / "mask.pgm", m != 0)
    out = tmp_path / "d.f32"
    assert main(["edt", "--input", mask, "--out", str(out), "--conn", "4"]) == 0
    _, dist = oracle.edt(m, 4)
    assert np.array_equal(read_f32_raw(str(out)).data, dist)


def test_edt_all_foreground_exits_3(tmp_path, capsys):
    mask = binary(tmp_path / "mask.pgm", np.ones((8, 8), np.uint8))
    assert main(["edt", "--input", mask, "--out", str(tmp_path / "d.f32")]) == 3
    assert "error:" in capsys.readouterr().err


def test_edt_quantized_pgm_rounds_distances(tmp_path):
    a = np.ones((8, 8), np.uint8)
    a[0, 0] = 0
    mask = binary(tmp_path / "mask.pgm", a)
    out = tmp_path / "d.pgm"
    assert main(["edt", "--input", mask, "--out", str(out)]) == 0
    got = read_pgm(str(out))
    assert got.data[0, 0] == 0 and got.data[0, 1] == 1
    assert got.data[4, 3] == 5  # 3-4-5 triangle from the corner
    assert got.data[1, 1] == round(2 ** 0.5)


def test_edt_rejects_gray_input(tmp_path):
    mask = gray(tmp_path / "mask.pgm", np.arange(64).reshape(8, 8))
    assert main(["edt", "--input", mask, "--out", str(tmp_path / "d.f32")]) == 2


def test_bad_tile_flag_exits_2(tmp_path):
    rng = np.random.default_rng(5)
    mask = binary(tmp_path / "mask.pgm", rng.random((8, 8)) < 0.5)
    assert main(["edt", "--input", mask, "--out", str(tmp_path / "d.f32"),
                 "--mode", "tiled", "--tile", "16by16"]) == 2


def test_file_to_file_4k_u16_recon(tmp_path):
    """A 4096 x 2048 16-bit P5 file through the device decode, the u16
    register engine and the device encode, against the oracle."""
    rng = np.random.default_rng(6)
    I = rng.integers(0, 65536, (2048, 4096)).astype(np.uint16)
    mask = str(tmp_path / "m.pgm")
    write_pgm(Image2D(4096, 2048, "u16", I), mask)
    out = str(tmp_path / "o.pgm")
    assert main(["recon", "--mask", mask, "--auto-marker", "9000", "--out", out, "--conn", "4"]) == 0
    J = np.maximum(I.astype(np.int64) - 9000, 0).astype(np.uint16)
    got = read_pgm(out).data
    assert np.array_equal(got, oracle.recon_fh(J, I, 4))
