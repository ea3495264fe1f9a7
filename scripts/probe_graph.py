"""Does the headline step (marker restore + iwpp_recon, cooperative engine
launch) capture into a CUDA graph, and what does replay save?"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
from bench import gray_pair
from paper_1209_3314_b200 import _lib

L = _lib.lib()
J, I = gray_pair(4096, 0)
dJ, dI = torch.from_numpy(J).cuda(), torch.from_numpy(I).cuda()
out = torch.empty_like(dJ)
ws = _lib.workspace(L.iwpp_recon_workspace_bytes(4096, 4096, 0, 8))
o = _lib.ReconOpts()
o.sweeps, o.max_blocks, o.check_contract, o.queue_capacity = -1, 0, 0, 0
o.tile_sweeps, o.halo_sweep_threshold = -1, -1
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def step():
    out.copy_(dJ)
    _lib.check(L.iwpp_recon(_lib.ptr(out), _lib.ptr(dI), 4096, 4096, 0, 8, _lib.ptr(ws), ws.numel(),
                            _lib.ctypes.byref(o), None, _lib.stream_ptr()), "recon")


def timed(fn, n=20):
    ts = []
    for i in range(n):
        flush.fill_(i & 255)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


for _ in range(3):
    step()
torch.cuda.synchronize()
print(f"eager step: {timed(step):.4f} ms", flush=True)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        step()
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
try:
    with torch.cuda.graph(g):
        step()
    g.replay()
    torch.cuda.synchronize()
    ok = np.array_equal(out.cpu().numpy(), oracle.recon_fh(J, I, 8))
    print(f"graph step: {timed(g.replay):.4f} ms  exact={ok}", flush=True)
except Exception as e:
    print("capture failed:", type(e).__name__, str(e)[:300], flush=True)
