"""64K^2 whole-slide EDT (the bench's mask: the 4K nuclei mask tiled 16x16)
timed with CUDA events, median of 3, plus a checksum of vr and dist so that
builds / IWPP_* variants can be compared: python scripts/probe_edt64k.py [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_1209_3314_b200 as gw

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
tile = oracle.gen_nuclei_mask(4096, 4096, 30.0, 7)
m = torch.from_numpy(tile).cuda().repeat(n // 4096, n // 4096)
img = gw.Image2D(n, n, "binary", m)
ts = []
for r in range(4):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    vm, dist = gw.edt(img, gw.SE8)
    b.record()
    torch.cuda.synchronize()
    if r:
        ts.append(a.elapsed_time(b))
    if r < 3:
        del vm, dist
ck_v, ck_d = 0, 0.0
for y in range(0, n, 2048):  # (in row blocks: a full f64 copy does not fit beside the workspace)
    ck_v += int(torch.sum(vm.vr[y:y + 2048:7, ::5]).item())
    ck_d += float(torch.sum(dist.data[y:y + 2048].to(torch.float64)).item())
print(f"edt {n}^2 nuclei c8: median {np.median(ts):.2f} ms (min {min(ts):.2f}); checksum vr {ck_v} dist {ck_d!r}",
      flush=True)
