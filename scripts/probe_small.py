"""Development probe: tile-engine latency vs image height (W=4096, u8 c8,
device-resident), to separate the per-launch fixed cost from throughput."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_1209_3314_b200 as gw
from paper_1209_3314_b200 import _lib

torch.cuda.set_device(0)
L = _lib.lib()
J0, I0 = oracle.gray_pair(4096, 0, h=40)
for h in (32, 64, 128, 256, 512, 1024, 2048, 4096):
    dJ = torch.from_numpy(J0[:h].copy()).cuda()
    dI = torch.from_numpy(I0[:h].copy()).cuda()
    W = 4096
    ws = _lib.workspace(L.iwpp_recon_workspace_bytes(W, h, 0, 8))
    J = dJ.clone()
    o = _lib.ReconOpts()
    o.sweeps, o.tile_sweeps, o.halo_sweep_threshold = -1, -1, -1
    def run():
        J.copy_(dJ)
        _lib.check(L.iwpp_recon(_lib.ptr(J), _lib.ptr(dI), W, h, 0, 8, _lib.ptr(ws), ws.numel(),
                                _lib.ctypes.byref(o), None, _lib.stream_ptr()))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); run(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    st = {}
    gw.reconstruct(dJ, dI, 8, stats=st)
    c = (_lib.ctypes.c_uint64 * 16)()
    L.iwpp_recon_engine_counters(_lib.ptr(ws), W, h, c, 16, _lib.stream_ptr())
    ph = [c[8 + i] for i in range(6)]
    tot = sum(ph) or 1
    print(f"h={h:5d} tiles={(h+31)//32*128:6d}: {np.median(ts):.3f} ms  tiles_proc={st['tiles_processed']} "
          f"reruns={st['tile_reruns']} phases(pop,load,sweep,detect,bfs,store)%="
          f"{[round(100*p/tot) for p in ph]} cyc/tile={tot/max(1,st['tiles_processed']):.0f}", flush=True)
