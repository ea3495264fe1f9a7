"""Recon engine experiments: python scripts/prof_recon.py N CONN TILE_SWEEPS MAX_BLOCKS [case] [reps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import paper_1209_3314_b200 as gw
from paper_1209_3314_b200 import _lib

n, conn, tsw, mb = (int(x) for x in sys.argv[1:5])
hth = int(os.environ.get("HTH", "-1"))
case = sys.argv[5] if len(sys.argv) > 5 else "rand"
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 5
if case == "rand":
    J, I = oracle.gray_pair(n, 0, h=40)
elif case == "same":
    J, I = oracle.gray_pair(n, 0, h=0)
elif case == "imfill":
    bw = oracle.gen_synthetic_mask(4096, 4096, 50, 7)
    J, I = oracle.imfill_pair(np.tile(bw, (n // 4096, n // 4096)))
DT = int(os.environ.get("DTYPE", "0"))
if DT == 1:
    J, I = J.astype(np.uint16) * 200, I.astype(np.uint16) * 200
elif DT == 2:
    J, I = J.astype(np.int32) * 1000 - 7, I.astype(np.int32) * 1000 - 7
elif DT == 3:
    J, I = J.astype(np.float32) * 0.5 - 3, I.astype(np.float32) * 0.5 - 3
dJ, dI = torch.from_numpy(J).cuda(), torch.from_numpy(I).cuda()
L = _lib.lib()
H, W = J.shape
ws = _lib.workspace(L.iwpp_recon_workspace_bytes(W, H, DT, conn))
out = dJ.clone()
o = _lib.ReconOpts(); o.engine = int(os.environ.get("ENGINE", "0")); o.sweeps = int(os.environ.get("GSW", "0")); o.max_blocks = mb; o.check_contract = 0; o.queue_capacity = 0; o.tile_sweeps = tsw; o.halo_sweep_threshold = hth
st = _lib.Stats()
ts = []
for r in range(reps + 2):
    out.copy_(dJ)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    _lib.check(L.iwpp_recon(_lib.ptr(out), _lib.ptr(dI), W, H, DT, conn, _lib.ptr(ws), ws.numel(), _lib.ctypes.byref(o), None, _lib.stream_ptr()))
    b.record(); torch.cuda.synchronize()
    if r >= 2: ts.append(a.elapsed_time(b))
out.copy_(dJ)
_lib.check(L.iwpp_recon(_lib.ptr(out), _lib.ptr(dI), W, H, DT, conn, _lib.ptr(ws), ws.numel(), _lib.ctypes.byref(o), _lib.ctypes.byref(st), _lib.stream_ptr()))
cnt = (_lib.ctypes.c_uint64 * 16)()
L.iwpp_recon_engine_counters(_lib.ptr(ws), W, H, cnt, 16, _lib.stream_ptr())
phs = list(cnt)[8:14]; tot = sum(phs) or 1
ph_str = " ".join(f"{n}={v/tot*100:.0f}%" for n, v in zip(["pop","load","sweep","detect","bfs","store"], phs))
print(f"  phases: {ph_str}; per-activation cycles {tot/max(cnt[0],1):.0f}; jacobi steps/activation {cnt[6]/max(cnt[0],1):.2f}")
print(f"{case} {n}^2 c{conn} tsw={tsw} mb={mb} hth={hth} gsw={o.sweeps}: median {np.median(ts):.3f} ms min {min(ts):.3f}  stats={st.as_dict()}", flush=True)
