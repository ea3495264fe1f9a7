"""Stress the binary (bit-plane) engine: repeated 4K imfill reconstructions
compared with the CPU oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_1209_3314_b200 as gw

torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
bw = oracle.gen_synthetic_mask(4096, 4096, 50, 7)
J, I = oracle.imfill_pair(bw)
for conn in (8, 4):
    want = oracle.recon_fh(J, I, conn)
    dJ, dI = torch.from_numpy(J).cuda(), torch.from_numpy(I).cuda()
    bad = sum(not np.array_equal(gw.reconstruct(dJ, dI, conn, kind="binary").cpu().numpy(), want)
              for _ in range(n))
    print(f"imfill 4K c{conn} binary engine: mismatching calls {bad}/{n}")
