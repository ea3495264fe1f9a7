"""imfill 16K^2 timing (the bench's C4 rows) for A/B: python scripts/probe_imfill.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_1209_3314_b200 as gw

bw = np.tile(oracle.gen_synthetic_mask(4096, 4096, 50, 7), (4, 4))
J, I = (torch.from_numpy(a).cuda() for a in oracle.imfill_pair(bw))
for conn in (4, 8):
    ts = []
    for r in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        gw.reconstruct(J, I, conn, kind="binary")
        b.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(a.elapsed_time(b))
    print(f"imfill 16K c{conn}: {np.median(ts):.3f} ms (min {min(ts):.3f})", flush=True)
