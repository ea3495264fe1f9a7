"""Stress the pipelined host path: N iwpp_recon_host calls on one 4K^2 u8
instance (pageable buffers, as the API test uses), each compared with the
device-resident result.  Prints the number of mismatching calls."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_1209_3314_b200 as gw

torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
conn = int(sys.argv[2]) if len(sys.argv) > 2 else 8
J, I = oracle.gray_pair(4096, 0, h=40)
want = gw.reconstruct(torch.from_numpy(J).cuda(), torch.from_numpy(I).cuda(), conn).cpu().numpy()
bad = 0
for i in range(n):
    got = gw.reconstruct(J, I, conn)
    if not np.array_equal(got, want):
        bad += 1
        if bad <= 4:
            d = np.argwhere(got != want)
            y, x = d[0]
            from paper_1209_3314_b200 import _lib
            torch.cuda.synchronize()
            dev = _lib._ws[0][:4096 * 4096].view(4096, 4096).cpu().numpy()  # dJ = workspace head
            print(f"  call {i}: {len(d)} px, first ({y},{x}) got {got[y, x]} want {want[y, x]} "
                  f"device buffer {dev[y, x]} (device == want everywhere: {np.array_equal(dev, want)}); "
                  f"tile ({y // 32},{x // 32}) row-in-tile {y % 32} col {x % 32}")
print(f"mismatching calls: {bad}/{n}")
