"""Stress the device-resident engine: repeated reconstructions of one
instance, each compared with the CPU oracle.  Prints mismatching calls."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_1209_3314_b200 as gw

torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
h = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
conn = int(sys.argv[3]) if len(sys.argv) > 3 else 8
J, I = oracle.gray_pair((h, 4096), 0, h=40)
want = oracle.recon_fh(J, I, conn)
dJ, dI = torch.from_numpy(J).cuda(), torch.from_numpy(I).cuda()
bad = 0
for i in range(n):
    got = gw.reconstruct(dJ, dI, conn).cpu().numpy()
    if not np.array_equal(got, want):
        bad += 1
        if bad == 1:
            d = np.argwhere(got != want)
            print(f"  first mismatch call {i}: {len(d)} px at {d[:3].tolist()} got {got[tuple(d[0])]} want {want[tuple(d[0])]}")
print(f"{h}x4096 c{conn}: mismatching calls {bad}/{n}")
