"""Development probe: device-resident recon time for short, wide images
(the host pipeline's per-slab runs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
from paper_1209_3314_b200 import _lib

L = _lib.lib()
torch.cuda.set_device(0)
for (h, w) in [(32, 32), (256, 256), (512, 512), (32, 4096), (64, 4096), (256, 4096), (1024, 4096), (4096, 4096)]:
    J, I = oracle.gray_pair((h, w), 0, h=40)
    dJ, dI = torch.from_numpy(J).cuda(), torch.from_numpy(I).cuda()
    out = dJ.clone()
    ws = _lib.workspace(L.iwpp_recon_workspace_bytes(w, h, 0, 8))
    o = _lib.ReconOpts()
    o.sweeps, o.tile_sweeps, o.halo_sweep_threshold = -1, -1, -1
    st = _lib.Stats()
    ts = []
    for r in range(25):
        out.copy_(dJ)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.check(L.iwpp_recon(_lib.ptr(out), _lib.ptr(dI), w, h, 0, 8, _lib.ptr(ws), ws.numel(),
                                _lib.ctypes.byref(o), _lib.ctypes.byref(st) if r == 24 else None,
                                _lib.stream_ptr()))
        b.record()
        torch.cuda.synchronize()
        if r >= 5:
            ts.append(a.elapsed_time(b))
    print(f"{w}x{h}: median {np.median(ts) * 1e3:.1f} us  activations {st.tiles_processed} "
          f"tiles {(h // 32) * (w // 32)}", flush=True)
