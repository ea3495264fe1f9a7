"""Repeated runs of the device-resident multi-slab EDT (iwpp_edt_mg_*) on
one GPU against the oracle: random masks, connectivities and slab counts
(races in the mailbox / count-exchange protocol would show up as
mismatches or hangs).  python scripts/stress_mg.py [n_small] [n_big]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle
from paper_1209_3314_b200.distributed import edt_slabs_local_device

n_small = int(sys.argv[1]) if len(sys.argv) > 1 else 150
n_big = int(sys.argv[2]) if len(sys.argv) > 2 else 12
rng = np.random.default_rng(2026)
bad = 0
for i in range(n_small):
    H, W = int(rng.integers(16, 300)), int(rng.integers(16, 300))
    kind = i % 3
    if kind == 0:
        m = oracle.gen_synthetic_mask(W, H, int(rng.integers(20, 80)), int(rng.integers(0, 1000)))
    elif kind == 1:
        m = (rng.random((H, W)) < rng.uniform(0.5, 0.99)).astype(np.uint8) * 255
        m.flat[int(rng.integers(0, m.size))] = 0
    else:
        m = np.full((H, W), 255, np.uint8)
        m[int(rng.integers(0, H)), int(rng.integers(0, W))] = 0  # one source: deep rounds
    conn = 8 if i % 2 == 0 else 4
    G = int(rng.integers(1, min(16, H) + 1))
    vr_ref, d_ref, (rounds, _) = oracle.edt(m, conn, stats=True)
    vr, d, r = edt_slabs_local_device(m, G, conn)
    if not (np.array_equal(vr, vr_ref) and d.tobytes() == d_ref.tobytes() and r == rounds):
        bad += 1
        print(f"MISMATCH case {i}: {H}x{W} kind {kind} conn {conn} G {G}", flush=True)
m4 = oracle.gen_synthetic_mask(4096, 4096, 50, 7)
ref = {c: oracle.edt(m4, c, stats=True) for c in (4, 8)}
for i in range(n_big):
    conn = 8 if i % 2 == 0 else 4
    G = (2, 3, 4, 5, 6, 8)[i % 6]
    vr, d, r = edt_slabs_local_device(m4, G, conn)
    vr_ref, d_ref, (rounds, _) = ref[conn]
    if not (np.array_equal(vr, vr_ref) and d.tobytes() == d_ref.tobytes() and r == rounds):
        bad += 1
        print(f"MISMATCH 4K blob conn {conn} G {G}", flush=True)
print(f"multi-slab EDT stress: {n_small} random cases (G = 1..16) + {n_big} 4K blob runs, "
      f"mismatches: {bad}", flush=True)
sys.exit(1 if bad else 0)
