"""Recon engine A/B at several sizes on device-generated inputs (the bench's
whole-slide counter hash): python scripts/probe_engines.py [sizes] [engines]
e.g. probe_engines.py 4096,16384,65536 2,3.  Prints the kernel time (events
around the engine), the engine counters, and whether all engines agree."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from bench import slide_rows
from paper_1209_3314_b200 import _lib

sizes = [int(s) for s in (sys.argv[1] if len(sys.argv) > 1 else "4096,16384,65536").split(",")]
engines = [int(s) for s in (sys.argv[2] if len(sys.argv) > 2 else "2,3").split(",")]
conn = int(os.environ.get("CONN", 8))
reps = int(os.environ.get("REPS", 5))
L = _lib.lib()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for n in sizes:
    M, I = slide_rows(0, n, n, "cuda")
    ws = _lib.workspace(L.iwpp_recon_workspace_bytes(n, n, 0, conn))
    out = torch.empty_like(M)
    ref = None
    for eng in engines:
        ev0, ev1 = _lib.Event(), _lib.Event()
        o = _lib.ReconOpts()
        o.sweeps, o.max_blocks, o.check_contract, o.queue_capacity = 0, int(os.environ.get("MB", "0")), 0, 0
        o.tile_sweeps, o.halo_sweep_threshold, o.engine = -1, -1, eng
        o.ev_begin, o.ev_end = ev0.handle, ev1.handle
        ts = []
        for r in range(reps + 2):
            out.copy_(M)
            flush.fill_(r & 255)
            _lib.check(L.iwpp_recon(_lib.ptr(out), _lib.ptr(I), n, n, 0, conn, _lib.ptr(ws), ws.numel(),
                                    _lib.ctypes.byref(o), None, _lib.stream_ptr()))
            torch.cuda.synchronize()
            if r >= 2:
                ts.append(ev0.elapsed_ms(ev1))
        cnt = (_lib.ctypes.c_uint64 * 16)()
        L.iwpp_recon_engine_counters(_lib.ptr(ws), n, n, cnt, 16, _lib.stream_ptr())
        if ref is None:
            ref = out.clone()
            same = True
        else:
            same = bool(torch.equal(ref, out))
        ntiles = ((n + 31) // 32) ** 2
        print(f"{n}^2 c{conn} engine={eng}: kernel median {np.median(ts):.4f} ms min {min(ts):.4f}; "
              f"activations {cnt[0]} ({cnt[0] / ntiles:.2f}/tile) reruns {cnt[1]} "
              f"steps/act {cnt[6] / max(cnt[0], 1):.2f} rounds {cnt[7]} diag {list(cnt)[8:12]}; agree={same}", flush=True)
    del M, I, ws, out, ref
    torch.cuda.empty_cache()
