"""Development probe: host-buffer (e2e) reconstruction through iwpp_recon_host,
pipelined (auto / given slab heights) vs unpipelined.  Pinned host buffers."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
from paper_1209_3314_b200 import _lib

L = _lib.lib()
torch.cuda.set_device(0)
sizes = [int(a) for a in sys.argv[1:]] or [4096, 16384]
for n in sizes:
    J, I = oracle.gray_pair(n, 0, h=40) if n <= 8192 else (None, None)
    if J is None:
        g = torch.Generator().manual_seed(0)
        It = torch.randint(0, 256, (n, n), dtype=torch.uint8, generator=g)
        Jt = torch.clamp(It.to(torch.int16) - 40, min=0).to(torch.uint8)
        J, I = Jt.numpy(), It.numpy()
    pJ = torch.from_numpy(J).pin_memory()
    pI = torch.from_numpy(I).pin_memory()
    pO = torch.empty_like(pJ).pin_memory()
    ws = _lib.workspace(L.iwpp_recon_host_workspace_bytes(n, n, 0, 8))
    stream = _lib.stream_ptr()
    ref = None
    for rows in [int(r) for r in os.environ.get("ROWS", "-1,0,512,1024").split(",")]:
        o = _lib.ReconOpts()
        o.sweeps, o.tile_sweeps, o.halo_sweep_threshold = -1, -1, -1
        o.pipeline_rows = rows

        def step():
            _lib.check(L.iwpp_recon_host(_lib.ptr(pO.numpy()), _lib.ptr(pJ.numpy()),
                                         _lib.ptr(pI.numpy()), n, n, 0, 8, _lib.ptr(ws),
                                         ws.numel(), _lib.ctypes.byref(o), None, stream),
                       "recon_host")
        for _ in range(3):
            step()
        ts = []
        for _ in range(10):
            t0 = time.perf_counter()
            step()
            ts.append(time.perf_counter() - t0)
        out = pO.numpy().copy()
        if ref is None:
            ref = out
        same = np.array_equal(out, ref)
        med = float(np.median(ts)) * 1e3
        print(f"e2e {n}^2 u8 c8 pipeline_rows={rows}: median {med:.3f} ms min {min(ts)*1e3:.3f} "
              f"-> {n*n/med/1e3:.0f} Mpx/s  same={same}", flush=True)
