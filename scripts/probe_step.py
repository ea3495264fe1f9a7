"""Where the headline step's time goes beyond the engine kernel: events
before / inside / after one iwpp_recon call (4096^2 u8 c8, marker option),
L2 flushed between steps as in bench.py.  python scripts/probe_step.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from bench import gray_pair
from paper_1209_3314_b200 import _lib

L = _lib.lib()
n = int(os.environ.get("N", 4096))
Jh, Ih = gray_pair(n, 0)
dJ, dI = torch.from_numpy(Jh).cuda(), torch.from_numpy(Ih).cuda()
out = torch.empty_like(dJ)
ws = _lib.workspace(L.iwpp_recon_workspace_bytes(n, n, 0, 8))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
a0, e0, e1, a1 = (_lib.Event() for _ in range(4))
o = _lib.ReconOpts()
o.sweeps, o.max_blocks, o.check_contract, o.queue_capacity = -1, 0, 0, 0
o.tile_sweeps, o.halo_sweep_threshold = -1, -1
o.ev_begin, o.ev_end = e0.handle, e1.handle
st = _lib.stream_ptr()
for mode in ("marker", "copy"):
    o.marker = _lib.ptr(dJ) if mode == "marker" else None
    seg = []
    for i in range(30):
        flush.fill_(i & 255)
        a0.record()
        if mode == "copy":
            out.copy_(dJ)
        _lib.check(L.iwpp_recon(_lib.ptr(out), _lib.ptr(dI), n, n, 0, 8, _lib.ptr(ws), ws.numel(),
                                _lib.ctypes.byref(o), None, st))
        a1.record()
        torch.cuda.synchronize()
        if i >= 5:
            seg.append((a0.elapsed_ms(e0) * 1e3, e0.elapsed_ms(e1) * 1e3, e1.elapsed_ms(a1) * 1e3,
                        a0.elapsed_ms(a1) * 1e3))
    s = np.median(np.array(seg), axis=0)
    print(f"{mode}: before-kernel {s[0]:.1f} us, kernel {s[1]:.1f} us, after {s[2]:.1f} us, step {s[3]:.1f} us",
          flush=True)
# the same step without the inner events (what bench.py times): the step
# is then only the engine launch between the two outer events
o.marker = _lib.ptr(dJ)
o.ev_begin = o.ev_end = None
seg = []
for i in range(30):
    flush.fill_(i & 255)
    a0.record()
    _lib.check(L.iwpp_recon(_lib.ptr(out), _lib.ptr(dI), n, n, 0, 8, _lib.ptr(ws), ws.numel(),
                            _lib.ctypes.byref(o), None, st))
    a1.record()
    torch.cuda.synchronize()
    if i >= 5:
        seg.append(a0.elapsed_ms(a1) * 1e3)
print(f"marker, no inner events: step {np.median(seg):.1f} us", flush=True)
# back-to-back calls, no flush, no sync: the per-call spacing
o.marker = _lib.ptr(dJ)
o.ev_begin = o.ev_end = None
for reps in (1, 10):
    torch.cuda.synchronize()
    a0.record()
    for _ in range(reps):
        _lib.check(L.iwpp_recon(_lib.ptr(out), _lib.ptr(dI), n, n, 0, 8, _lib.ptr(ws), ws.numel(),
                                _lib.ctypes.byref(o), None, st))
    a1.record()
    torch.cuda.synchronize()
    print(f"{reps} back-to-back calls (L2 warm): {a0.elapsed_ms(a1) * 1e3 / reps:.1f} us per call", flush=True)
