"""Device-resident multi-slab EDT (iwpp_edt_mg_*) on one GPU: time per call
and per round for G virtual slabs vs the single-image engine and vs the
host-driven per-round slab loop.  python scripts/probe_edt_mg.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_1209_3314_b200 as gw
from paper_1209_3314_b200.distributed import (SlabEDT, edt_slabs_local_device, mask_ext_rows,
                                              run_edt_slabs_local, slab_bounds)


def t_of(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return float(np.median(ts)), out


for name, m in (("nuclei4k", oracle.gen_nuclei_mask(4096, 4096, 30.0, 7)),
                ("blob4k", oracle.gen_synthetic_mask(4096, 4096, 50, 7))):
    dm = torch.from_numpy(m).cuda()
    img = gw.Image2D(4096, 4096, "binary", dm)
    ms1, _ = t_of(lambda: gw.edt(img, gw.SE8))
    print(f"{name}: single-image engine {ms1:.2f} ms (wall, incl. init/finalize)", flush=True)
    from paper_1209_3314_b200 import _lib
    L = _lib.lib()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(2):  # the rounds kernel alone (events around launch_rounds via edt's stats)
        ev[0].record()
        gw.edt(img, gw.SE8)
        ev[1].record()
        torch.cuda.synchronize()
    print(f"{name}: single-image edt() device time {ev[0].elapsed_time(ev[1]):.2f} ms", flush=True)
    for G in (1, 2, 4, 8):
        tm = {}
        edt_slabs_local_device(dm, G, 8)
        out = edt_slabs_local_device(dm, G, 8, timing=tm)
        ms = tm["rounds_ms"]
        print(f"{name}: device-resident {G} slabs: rounds kernel {ms:.2f} ms, rounds {out[2]}, "
              f"{ms * 1e3 / max(out[2], 1):.1f} us/round", flush=True)
    for G in (2, 8):
        def host_loop():
            H = 4096
            slabs = [SlabEDT(mask_ext_rows(m, *slab_bounds(H, G, r)).cuda(), slab_bounds(H, G, r)[0], H,
                             r > 0, r + 1 < G, 8) for r in range(G)]
            rr = run_edt_slabs_local(slabs)
            for s in slabs:
                s.finalize()
            return rr
        ms, rr = t_of(host_loop, reps=1)
        print(f"{name}: host-driven per-round loop {G} slabs {ms:.2f} ms, rounds {rr}, {ms * 1e3 / rr:.1f} us/round",
              flush=True)
