"""One-off evidence (GPU box, >= 64 GB host RAM): the 64K x 64K whole-slide
reconstruction (bench.py slide_rows, u8, 8-conn) on the device against the
C oracle's recon_fh on the host, bit for bit.  ~45 GB of host RAM and a few
minutes of one core.  Usage: python scripts/slide_oracle_parity.py [N]"""

import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import oracle  # noqa: E402
import paper_1209_3314_b200 as gw  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
dev = torch.device("cuda:0")
M, I = bench.slide_rows(0, N, N, dev)
t0 = time.perf_counter()
J = gw.reconstruct(M, I, 8)
torch.cuda.synchronize()
t_dev = time.perf_counter() - t0
Jd = J.cpu().numpy()
del J, M, I
torch.cuda.empty_cache()
Mh, Ih = bench.slide_rows_np(0, N, N)
t0 = time.perf_counter()
want = oracle.recon_fh(Mh, Ih, 8)
t_cpu = time.perf_counter() - t0
eq = bool(np.array_equal(Jd, want))
diff = int((Jd != want).sum()) if not eq else 0
print(f"slide {N}x{N} u8 c8: device {t_dev*1e3:.1f} ms (incl. first-call setup), "
      f"oracle recon_fh 1 thread {t_cpu:.1f} s ({N*N/t_cpu/1e6:.1f} Mpx/s); "
      f"bit-exact={eq} differing_px={diff} raised_px={int((want != Mh).sum())}")
sys.exit(0 if eq else 1)
