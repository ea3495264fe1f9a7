"""Queue / engine study on one B200 -- the analog of the paper's Table 1
(naive vs prefix-sum vs thread-queue wavefront queues).

EDT frontier-queue engine, next frontier appended three ways:
  block queue (default): warp reservations into a shared-memory queue, one
                         global atomic per block per round
  prefix-sum (PF)      : warp reservations straight into the global queue
  naive                : one global atomicAdd per pushed item
plus the temporally blocked EDT engine; and the reconstruction tile engines
(shared-memory BFS queue, register Jacobi, one-bit binary).

    python scripts/queue_study.py > profiles/r01_queue_study.txt
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_1209_3314_b200 as gw
from paper_1209_3314_b200 import _lib

L = _lib.lib()
torch.cuda.set_device(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    ts = []
    for i in range(reps):
        flush.fill_(i & 0xff)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


print("# B200 queue / engine study (median of 5, L2 flushed between calls)")
print("\n## EDT 4096^2, 8-connectivity")
print(f"{'mask':8s} {'engine':32s} {'ms':>8s} {'rounds':>7s} {'visits':>10s} {'us/round':>9s}")
masks = {"nuclei": oracle.gen_nuclei_mask(4096, 4096, 30.0, 7),
         "blob": oracle.gen_synthetic_mask(4096, 4096, 50, 7)}
engines = [(3, "frontier queue, block queue"), (5, "frontier queue, prefix-sum (PF)"),
           (6, "frontier queue, naive atomics"), (7, "raster frontier (default)"),
           (4, "temporally blocked (8 rounds/sync)")]
for name, m in masks.items():
    img = gw.Image2D(4096, 4096, "binary", torch.from_numpy(m).cuda())
    ref_vr = None
    for mode, label in engines:
        _lib.check(L.iwpp_edt_set_engine(mode), "set_engine")
        cfg = gw.EngineConfig()
        vm, _ = gw.edt(img, gw.SE8, mode="parallel", cfg=cfg)
        vr = vm.vr.cpu().numpy()
        same = True if ref_vr is None else bool(np.array_equal(vr, ref_vr))
        ref_vr = vr if ref_vr is None else ref_vr
        ms = timed(lambda: gw.edt(img, gw.SE8))
        r = cfg.stats.rounds
        print(f"{name:8s} {label:32s} {ms:8.3f} {r:7d} {cfg.stats.queued_total:10d} "
              f"{ms * 1e3 / max(r, 1):9.1f}{'' if same else '  MISMATCH'}", flush=True)
    _lib.check(L.iwpp_edt_set_engine(0), "set_engine")

print("\n## Reconstruction (device-resident), ms per call")
print(f"{'input':34s} {'conn':>4s} {'smem BFS queue':>15s} {'register Jacobi':>16s} {'binary 1-bit':>13s}")
J, I = oracle.gray_pair(4096, 0, h=40)
dJ, dI = torch.from_numpy(J).cuda(), torch.from_numpy(I).cuda()
bw = np.tile(oracle.gen_synthetic_mask(4096, 4096, 50, 7), (4, 4))
mk, ms_ = oracle.imfill_pair(bw)
dM, dK = torch.from_numpy(mk).cuda(), torch.from_numpy(ms_).cuda()
for label, (a, b), binary in [("random u8 4096^2 (h=40)", (dJ, dI), False),
                              ("imfill binary 16384^2", (dM, dK), True)]:
    for conn in (4, 8):
        t1 = timed(lambda: gw.reconstruct(a, b, conn, engine=1), reps=3, warm=1)
        t2 = timed(lambda: gw.reconstruct(a, b, conn, engine=2), reps=3, warm=1)
        t3 = timed(lambda: gw.reconstruct(a, b, conn, kind="binary"), reps=3, warm=1) if binary else float("nan")
        print(f"{label:34s} {conn:4d} {t1:15.3f} {t2:16.3f} {t3:13.3f}", flush=True)
