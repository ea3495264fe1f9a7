"""The e2e call as bench.py times it (iwpp_recon_host, pinned host buffers,
4096^2 u8 c8): median of 20 calls.  IWPP_TRACE=1 adds the library's
timeline of the last call.  python scripts/probe_e2e.py [n]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from bench import gray_pair
from paper_1209_3314_b200 import _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
L = _lib.lib()
Jh, Ih = gray_pair(n, 0)
pin_J = torch.from_numpy(Jh).pin_memory()
pin_I = torch.from_numpy(Ih).pin_memory()
pin_O = torch.empty_like(pin_J).pin_memory()
ws = _lib.workspace(L.iwpp_recon_host_workspace_bytes(n, n, 0, 8))
o = _lib.ReconOpts()
o.sweeps, o.max_blocks, o.check_contract, o.queue_capacity = -1, 0, 0, 0
o.tile_sweeps, o.halo_sweep_threshold = -1, -1
o.pipeline_rows = int(os.environ.get("ROWS", "0"))
st = _lib.stream_ptr()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
trace = os.environ.pop("IWPP_TRACE", None)
ts = []
for i in range(22):
    flush.fill_(i & 255)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _lib.check(L.iwpp_recon_host(_lib.ptr(pin_O.numpy()), _lib.ptr(pin_J.numpy()), _lib.ptr(pin_I.numpy()),
                                 n, n, 0, 8, _lib.ptr(ws), ws.numel(), _lib.ctypes.byref(o), None, st))
    if i >= 2:
        ts.append(time.perf_counter() - t0)
ms = np.median(ts) * 1e3
print(f"e2e {n}^2 rows={o.pipeline_rows} slab_mb={os.environ.get('IWPP_SLAB_MB', 'auto')}: median {ms:.3f} ms "
      f"min {min(ts) * 1e3:.3f} -> {n * n / ms / 1e3:.0f} Mpx/s", flush=True)
if trace:
    os.environ["IWPP_TRACE"] = trace
    # (the library reads IWPP_TRACE per call)
    _lib.check(L.iwpp_recon_host(_lib.ptr(pin_O.numpy()), _lib.ptr(pin_J.numpy()), _lib.ptr(pin_I.numpy()),
                                 n, n, 0, 8, _lib.ptr(ws), ws.numel(), _lib.ctypes.byref(o), None, st))
