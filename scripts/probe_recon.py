"""Recon engine A/B probe: python scripts/probe_recon.py N CONN [case] [reps]
Times iwpp_recon on the device (events around the engine kernel), prints the
engine counters and checks the result against the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
from paper_1209_3314_b200 import _lib

n, conn = int(sys.argv[1]), int(sys.argv[2])
case = sys.argv[3] if len(sys.argv) > 3 else "rand"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
if case == "rand":
    J, I = oracle.gray_pair(n, 0, h=40)
elif case == "imfill":
    J, I = oracle.imfill_pair(np.tile(oracle.gen_synthetic_mask(4096, 4096, 50, 7), (n // 4096,) * 2))
elif case == "i32":
    J, I = oracle.gray_pair(n, 0, h=1 << 28, dtype=np.int32)
DT = {np.dtype(np.uint8): 0, np.dtype(np.int32): 2}[J.dtype]
L = _lib.lib()
H, W = J.shape
dJ, dI = torch.from_numpy(J).cuda(), torch.from_numpy(I).cuda()
ws = _lib.workspace(L.iwpp_recon_workspace_bytes(W, H, DT, conn))
out = dJ.clone()
ev0, ev1 = _lib.Event(), _lib.Event()
o = _lib.ReconOpts()
o.sweeps, o.max_blocks, o.check_contract, o.queue_capacity = 0, int(os.environ.get("MB", "0")), 0, 0
o.tile_sweeps, o.halo_sweep_threshold, o.engine = -1, -1, int(os.environ.get("ENGINE", "0"))
o.ev_begin, o.ev_end = ev0.handle, ev1.handle
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for r in range(reps + 3):
    out.copy_(dJ)
    flush.fill_(r & 255)
    _lib.check(L.iwpp_recon(_lib.ptr(out), _lib.ptr(dI), W, H, DT, conn, _lib.ptr(ws), ws.numel(),
                            _lib.ctypes.byref(o), None, _lib.stream_ptr()))
    torch.cuda.synchronize()
    if r >= 3:
        ts.append(ev0.elapsed_ms(ev1))
cnt = (_lib.ctypes.c_uint64 * 16)()
L.iwpp_recon_engine_counters(_lib.ptr(ws), W, H, cnt, 16, _lib.stream_ptr())
ok = np.array_equal(out.cpu().numpy(), oracle.recon_fh(J, I, conn)) if n <= 16384 else None
print(f"{case} {n}^2 c{conn} engine={o.engine} rounds_env={os.environ.get('IWPP_RECON_ROUNDS', '1')}: "
      f"kernel median {np.median(ts):.4f} ms min {min(ts):.4f}; activations {cnt[0]} reruns {cnt[1]} "
      f"steps/act {cnt[6] / max(cnt[0], 1):.2f} rounds {cnt[7]}; exact={ok}", flush=True)
