"""EDT engine A/B on the bench's 4K masks: python scripts/probe_edt.py [modes]
(modes: iwpp_edt_set_engine values, default 7,8).  Times the full edt()
call with CUDA events (median of 5) and checks every engine agrees."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_1209_3314_b200 as gw
from paper_1209_3314_b200 import _lib

modes = [int(m) for m in (sys.argv[1] if len(sys.argv) > 1 else "7,8").split(",")]
L = _lib.lib()
masks = {"nuclei": oracle.gen_nuclei_mask(4096, 4096, 30.0, 7),
         "blob": oracle.gen_synthetic_mask(4096, 4096, 50, 7)}
for name, m in masks.items():
    img = gw.Image2D(4096, 4096, "binary", torch.from_numpy(m).cuda())
    for conn in (8, 4):
        se = gw.StructuringElement(conn)
        ref = None
        for mode in modes:
            _lib.check(L.iwpp_edt_set_engine(mode), "set_engine")
            ts = []
            for r in range(7):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                vm, dist = gw.edt(img, se)
                b.record()
                torch.cuda.synchronize()
                if r >= 2:
                    ts.append(a.elapsed_time(b))
            got = (vm.vr.clone(), dist.data.clone())
            same = True if ref is None else bool(torch.equal(ref[0], got[0]) and torch.equal(ref[1], got[1]))
            ref = ref or got
            print(f"{name} c{conn} engine {mode}: {np.median(ts):.3f} ms (min {min(ts):.3f}) agree={same}", flush=True)
        _lib.check(L.iwpp_edt_set_engine(0), "set_engine")
