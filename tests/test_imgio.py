"""Image I/O (reference: gridwave/imgio.py; tests mirror pkg/tests/test_imgio.py).

CPU tests: the host reader against 331 golden outcomes recorded from the
reference reader (tests/golden/make_pgm_golden.py -- samples, or exception
type + message + byte offset), and the writers' byte formats.
GPU tests: the device path (pinned read -> HBM -> iwpp_pgm_decode /
iwpp_pgm_encode / iwpp_gen_marker / iwpp_quantize_u8) gives the same
images, errors and bytes as the host path."""

import json
import os

import numpy as np
import pytest

from paper_1209_3314_b200.errors import ContractViolation, PgmFormatError
from paper_1209_3314_b200.grid import BG, FG, Image2D
from paper_1209_3314_b200.imgio import (gen_marker, quantize_distance, read_f32_raw, read_pgm,
                                        write_f32_raw, write_pgm)

GOLD = os.path.join(os.path.dirname(__file__), "golden", "pgm_cases.json")
CASES = json.load(open(GOLD))


def _outcome(path, device=None):
    try:
        img = read_pgm(path, device=device)
        data = img.numpy()
        return {"ok": True, "kind": img.elem_kind, "w": img.width, "h": img.height,
                "samples": data.reshape(-1).tolist()}
    except PgmFormatError as e:
        return {"ok": False, "type": "PgmFormatError", "msg": str(e), "offset": e.offset}


def _check_cases(tmp_path, device):
    p = str(tmp_path / "c.pgm")
    bad = []
    for i, c in enumerate(CASES):
        with open(p, "wb") as f:
            f.write(bytes.fromhex(c["bytes"]))
        want = {k: v for k, v in c.items() if k != "bytes"}
        got = _outcome(p, device)
        if got != want:
            bad.append((i, want, got))
    assert not bad, bad[:3]


def test_host_reader_matches_reference_outcomes(tmp_path):
    _check_cases(tmp_path, None)


def test_read_p5_u8(tmp_path):
    p = tmp_path / "a.pgm"
    p.write_bytes(b"P5 4 4 255\n" + bytes(range(16)))
    img = read_pgm(str(p))
    assert (img.width, img.height, img.elem_kind) == (4, 4, "u8")
    assert np.array_equal(img.data.reshape(-1), np.arange(16))


def test_error_carries_byte_offset(tmp_path):
    p = tmp_path / "o.pgm"
    p.write_bytes(b"P2 2 2 255\n0 255 nope 0\n")
    with pytest.raises(PgmFormatError) as e:
        read_pgm(str(p))
    assert e.value.offset == 17


@pytest.mark.parametrize("kind,hi", [("u8", 256), ("u16", 65536)])
def test_round_trip_random(tmp_path, kind, hi):
    rng = np.random.default_rng(3)
    dt = np.uint8 if kind == "u8" else np.uint16
    img = Image2D(7, 5, kind, rng.integers(0, hi, (5, 7)).astype(dt))
    p = str(tmp_path / "r.pgm")
    write_pgm(img, p)
    back = read_pgm(p)
    assert back.elem_kind == kind and np.array_equal(back.data, img.data)
    hdr = b"P5\n7 5\n%d\n" % (255 if kind == "u8" else 65535)
    raw = open(p, "rb").read()
    assert raw.startswith(hdr) and len(raw) == len(hdr) + img.data.nbytes


def test_binary_written_with_maxval_255_reads_as_u8(tmp_path):
    rng = np.random.default_rng(5)
    data = (rng.random((6, 6)) < 0.5).astype(np.uint8) * FG
    p = str(tmp_path / "b.pgm")
    write_pgm(Image2D(6, 6, "binary", data), p)
    back = read_pgm(p)
    assert back.elem_kind == "u8" and np.array_equal(back.data, data)


def test_writers_reject_wrong_kinds():
    with pytest.raises(ContractViolation):
        write_pgm(Image2D(2, 2, "f32", np.zeros((2, 2), np.float32)), "/tmp/never.pgm")
    with pytest.raises(ContractViolation):
        write_f32_raw(Image2D(2, 2, "u8", np.zeros((2, 2), np.uint8)), "/tmp/never.f32")


def test_f32_payload_sidecar_and_round_trip(tmp_path):
    rng = np.random.default_rng(7)
    img = Image2D(9, 4, "f32", rng.random((4, 9)).astype(np.float32))
    p = str(tmp_path / "d.f32")
    write_f32_raw(img, p)
    assert os.path.getsize(p) == 9 * 4 * 4
    assert (tmp_path / "d.f32.hdr").read_text() == "9 4 f32le\n"
    assert np.array_equal(read_f32_raw(p).data, img.data)
    (tmp_path / "d.f32.hdr").write_text("3 2 f32le\n")
    with pytest.raises(ContractViolation):
        read_f32_raw(p)


def test_marker_formula_and_bounds():
    a = np.array([[0, 5, 40, 41, 255]], np.uint8)
    m = gen_marker(Image2D(5, 1, "u8", a), 40)
    assert m.data.tolist() == [[0, 0, 0, 1, 215]]
    with pytest.raises(ContractViolation):
        gen_marker(Image2D(5, 1, "binary", np.zeros((1, 5), np.uint8)), 3)
    with pytest.raises(ContractViolation):
        gen_marker(Image2D(5, 1, "u8", a), -1)


# ---------------------------------------------------------------------------
# device path

@pytest.fixture(scope="module")
def cuda():
    import torch
    torch.cuda.set_device(0)
    return torch


@pytest.mark.gpu
def test_device_reader_matches_reference_outcomes(tmp_path, cuda):
    _check_cases(tmp_path, "cuda")


@pytest.mark.gpu
@pytest.mark.parametrize("kind,shape", [("u8", (1000, 1333)), ("u16", (777, 1025)),
                                        ("binary", (513, 4099)), ("u16", (1, 1)), ("u8", (3, 5))])
def test_device_round_trip_and_bytes(tmp_path, cuda, kind, shape):
    rng = np.random.default_rng(11)
    h, w = shape
    if kind == "u16":
        a = rng.integers(0, 65536, shape).astype(np.uint16)
    elif kind == "binary":
        a = (rng.random(shape) < 0.4).astype(np.uint8) * FG
    else:
        a = rng.integers(0, 256, shape).astype(np.uint8)
    host = Image2D(w, h, kind, a)
    dev = Image2D(w, h, kind, cuda.from_numpy(a).cuda())
    ph, pd = str(tmp_path / "h.pgm"), str(tmp_path / "d.pgm")
    write_pgm(host, ph)
    write_pgm(dev, pd)
    assert open(ph, "rb").read() == open(pd, "rb").read()
    back = read_pgm(pd, device="cuda")
    assert back.on_device
    want = read_pgm(ph)
    assert back.elem_kind == want.elem_kind
    assert np.array_equal(back.numpy(), want.data)


@pytest.mark.gpu
def test_device_maxval_one_maps_to_fg(tmp_path, cuda):
    rng = np.random.default_rng(2)
    bits = (rng.random(70001) < 0.5).astype(np.uint8)
    p = tmp_path / "b.pgm"
    p.write_bytes(b"P5 70001 1 1\n" + bits.tobytes())
    img = read_pgm(str(p), device="cuda")
    assert img.elem_kind == "binary"
    assert np.array_equal(img.numpy()[0], np.where(bits != 0, FG, BG))
    bits[12345] = 7
    p.write_bytes(b"P5 70001 1 1\n" + bits.tobytes())
    with pytest.raises(PgmFormatError, match="sample exceeds maxval 1"):
        read_pgm(str(p), device="cuda")


@pytest.mark.gpu
def test_device_f32_raw_round_trip(tmp_path, cuda):
    rng = np.random.default_rng(8)
    a = rng.standard_normal((301, 257)).astype(np.float32)
    p = str(tmp_path / "x.f32")
    write_f32_raw(Image2D(257, 301, "f32", cuda.from_numpy(a).cuda()), p)
    assert open(p, "rb").read() == a.astype("<f4").tobytes()
    back = read_f32_raw(p, device="cuda")
    assert back.on_device and np.array_equal(back.numpy(), a)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["u8", "u16", "i32", "f32"])
def test_device_gen_marker_matches_host(cuda, kind):
    rng = np.random.default_rng(4)
    shape = (123, 457)
    if kind == "u8":
        a = rng.integers(0, 256, shape).astype(np.uint8)
    elif kind == "u16":
        a = rng.integers(0, 65536, shape).astype(np.uint16)
    elif kind == "i32":
        a = rng.integers(-2**31, 2**31 - 1, shape, dtype=np.int64).astype(np.int32)
    else:
        a = (rng.standard_normal(shape) * 100).astype(np.float32)
        a[0, :4] = [np.nan, -0.0, 40.0, np.inf]
    for h in (0, 1, 40, 300, 70000):
        want = gen_marker(Image2D(457, 123, kind, a), h).data
        got = gen_marker(Image2D(457, 123, kind, cuda.from_numpy(a).cuda()), h).numpy()
        assert got.dtype == want.dtype
        assert np.array_equal(got, want, equal_nan=(kind == "f32")), (kind, h)


@pytest.mark.gpu
def test_device_quantize_matches_host(cuda):
    rng = np.random.default_rng(9)
    d = (rng.random((97, 301)) * 400).astype(np.float32)
    d[0, :6] = [0.5, 1.5, 2.5, 254.5, 255.5, 0.0]
    want = quantize_distance(Image2D(301, 97, "f32", d)).data
    got = quantize_distance(Image2D(301, 97, "f32", cuda.from_numpy(d).cuda())).numpy()
    assert np.array_equal(got, want)
