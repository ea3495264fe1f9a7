"""Generate PGM-reader golden cases from the REFERENCE reader
(gridwave/imgio.py:62-110).  Build container only:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_pgm_golden.py

Writes tests/golden/pgm_cases.json: each case = the file bytes (hex) and the
reference's outcome -- (kind, samples) or (exception type, message, byte
offset).  Cases: the reference's own test_imgio.py inputs, header/body edge
cases, and seeded random P2 files with comments, mixed separators,
out-of-range samples, missing samples and malformed tokens.
"""

from __future__ import annotations

import json
import os
import random
import sys
import tempfile

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

from gridwave.imgio import read_pgm  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "pgm_cases.json")

FIXED = [
    b"P5 4 4 255\n" + bytes(range(16)),
    b"P2 2 2 255\n0 255 255 0\n",
    b"P5 3 1 1\n" + bytes([0, 1, 1]),
    b"P5 # magic\n2 # w\n1 # h\n255\n\x07\x09",
    b"P5 2 1 65535\n" + bytes([0x01, 0x00, 0x00, 0xFF]),
    b"P5 4 4 255\n" + bytes(10),
    b"P6 1 1 255\n\x00\x00\x00",
    b"P2 1 1 70000\n0\n",
    b"P2 2 2 255\n0 255 nope 0\n",
    b"P2 2 2 255\n0 2#c 5\n55 0\n",
    b"P2 2 2 255\n0 2#c 5\n55",
    b"P2 2 2 9\n0 2 10 1",
    b"P2 2 1 1\n0 1",
    b"P2 2 1 1\n0 2",
    b"P2 2 1 65535\n000000000000000000000001 65535 7",
    b"",
    b"P5",
    b"P5 0 1 255\n",
    b"P5 1 1 255",
    b"P5 1 1 255\n",
    b"P5 1 1 255x\x01",
    b"P2 3 1 255 #\n1 #2\n 2\r3 4",
    b"P5 2 1 200\n\x00\xff",
    b"P5 3 2 65535\n" + bytes(range(12)),
    b"P5 17 3 255\t" + bytes(range(51)),
    b"P5 9 2 1\n" + bytes([0, 1] * 9),
    b"P5 9 2 1\n" + bytes([0, 2] * 9),
    b"P5 5 1 1000\n" + bytes([0x03, 0xE8, 0x03, 0xE9, 0, 0, 0, 1, 0, 2]),
    b"P2 -1 1 255\n0",
    b"P2 1 1 0\n0",
    b"P2 1 1 255\n+5",
]


def random_cases(n=300, seed=1):
    rng = random.Random(seed)
    out = []
    seps = [" ", "\n", "\t", " # c\n", "#x\r", "  ", "\r\n", "\x0b", "\x0c"]
    for _ in range(n):
        w, h = rng.randint(1, 6), rng.randint(1, 4)
        mv = rng.choice([1, 9, 255, 300, 65535])
        k = w * h - (1 if rng.random() < 0.05 else 0)
        toks = [str(rng.randint(0, mv + (1 if rng.random() < 0.05 else 0))) for _ in range(k)]
        body = "".join(t + rng.choice(seps) for t in toks)
        if rng.random() < 0.05:
            body = body.replace("1", "a", 1)
        out.append(f"P2 {w} {h} {mv}\n".encode() + body.encode())
    return out


def outcome(data: bytes):
    with tempfile.NamedTemporaryFile(suffix=".pgm", delete=False) as f:
        f.write(data)
        path = f.name
    try:
        img = read_pgm(path)
        return {"ok": True, "kind": img.elem_kind, "w": img.width, "h": img.height,
                "samples": img.data.reshape(-1).tolist()}
    except Exception as e:  # noqa: BLE001 - recorded
        return {"ok": False, "type": type(e).__name__, "msg": str(e),
                "offset": getattr(e, "offset", None)}
    finally:
        os.unlink(path)


def main():
    cases = [{"bytes": c.hex(), **outcome(c)} for c in FIXED + random_cases()]
    with open(OUT, "w") as f:
        json.dump(cases, f, separators=(",", ":"))
    print(f"wrote {len(cases)} cases to {OUT}")


if __name__ == "__main__":
    main()
