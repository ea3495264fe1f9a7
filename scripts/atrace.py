"""Activation timeline of the u8 register tile engine (queue occupancy and
concurrency evidence).  Builds (or reuses) a -DIWPP_ATRACE variant of the
library, runs one recon of the bench's counter-hash slide, and summarises
the per-activation records: how many warps are inside an activation over
time, the ring depth seen at each pop, the phase split (pop / load / fixed
point / publish+finish) and the tail.

    python scripts/atrace.py [N] [CONN]      (N = 4096 default)

Run on the GPU box; prints a text summary (profiles/ keeps the output)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VAR = os.path.join(ROOT, "paper_1209_3314_b200", "libiwpp_b200_atrace.so")
if os.environ.get("IWPP_B200_LIB") != VAR:
    if not os.path.exists(VAR):
        from paper_1209_3314_b200 import build
        build.build(out=VAR, defines=("IWPP_ATRACE",))
    env = dict(os.environ, IWPP_B200_LIB=VAR)
    sys.exit(subprocess.call([sys.executable, *sys.argv], env=env))

import numpy as np
import torch

from bench import slide_rows
from paper_1209_3314_b200 import _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
conn = int(sys.argv[2]) if len(sys.argv) > 2 else 8
L = _lib.lib()
M, I = slide_rows(0, n, n, "cuda")
ws = _lib.workspace(L.iwpp_recon_workspace_bytes(n, n, 0, conn))
out = M.clone()
cap = int(((n + 31) // 32) ** 2 * 4)
buf = torch.zeros(cap * 8, dtype=torch.int32, device="cuda")
o = _lib.ReconOpts()
o.sweeps, o.max_blocks, o.check_contract, o.queue_capacity = 0, 0, 0, 0
o.tile_sweeps, o.halo_sweep_threshold, o.engine = -1, -1, 2
ev0, ev1 = _lib.Event(), _lib.Event()
o.ev_begin, o.ev_end = ev0.handle, ev1.handle
cnt = _lib.ctypes.c_uint32(0)
for rep in range(3):  # the last run is the traced one that counts
    out.copy_(M)
    torch.cuda.synchronize()
    assert L.iwpp_debug_atrace(_lib.ptr(buf), cap, None) == 32
    _lib.check(L.iwpp_recon(_lib.ptr(out), _lib.ptr(I), n, n, 0, conn, _lib.ptr(ws), ws.numel(),
                            _lib.ctypes.byref(o), None, _lib.stream_ptr()))
    torch.cuda.synchronize()
L.iwpp_debug_atrace(None, 0, _lib.ctypes.byref(cnt))
c = (_lib.ctypes.c_uint64 * 16)()
L.iwpp_recon_engine_counters(_lib.ptr(ws), n, n, c, 16, _lib.stream_ptr())
kms = ev0.elapsed_ms(ev1)
k = min(int(cnt.value), cap)
R = buf[: k * 8].view(k, 8).cpu().numpy().astype(np.int64) & 0xFFFFFFFF
t0 = R[:, 0].min()
rel = lambda a: (a - t0) & 0xFFFFFFFF  # noqa: E731
pop, take, load, fix, end = (rel(R[:, i]) for i in range(5))
cont = (R[:, 5] >> 31) & 1
sm = R[:, 6] >> 16
depth = R[:, 7]
span = end.max()
print(f"{n}^2 c{conn}: kernel {kms * 1000:.1f} us (traced build), {k} activation records "
      f"({c[0]} activations, {c[1]} re-runs, idle polls {c[15]})")
print(f"trace span {span / 1000:.1f} us; continuations {cont.mean() * 100:.1f}% of activations")
ph = np.stack([take - pop, load - take, fix - load, end - fix], 1)
names = ["pop(ticket+slot+take)", "load(TMA boxes)", "fixpoint", "publish+claims+finish(+reruns)"]
for i, nm in enumerate(names):
    a = ph[:, i]
    print(f"  {nm:32s} mean {a.mean() / 1000:7.2f} us  p50 {np.median(a) / 1000:7.2f}  p99 "
          f"{np.percentile(a, 99) / 1000:7.2f}")
tot = (end - pop)
print(f"  {'activation total':32s} mean {tot.mean() / 1000:7.2f} us")
noncont = cont == 0
print(f"  pop phase, ring pops only: mean {(take - pop)[noncont].mean() / 1000:.2f} us")
# concurrency over time: warps inside an activation (pop..end), 20 bins
bins = np.linspace(0, span, 21)
print("time bin (us)   activations-in-flight(avg)  started  ring depth at pop (median)")
for a, b in zip(bins[:-1], bins[1:]):
    ov = np.clip(np.minimum(end, b) - np.maximum(pop, a), 0, None).sum() / max(b - a, 1)
    st = (pop >= a) & (pop < b)
    d = np.median(depth[st]) if st.any() else 0
    print(f"{a / 1000:7.1f}-{b / 1000:7.1f}  {ov:10.0f}  {st.sum():8d}  {d:8.0f}")
last = np.sort(end)[-50:]
print(f"last 1% of activations end after {np.percentile(end, 99) / 1000:.1f} us; "
      f"SMs used {len(np.unique(sm))}")
