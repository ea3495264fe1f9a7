import sys, os, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import oracle
import paper_1209_3314_b200 as gw
from paper_1209_3314_b200 import _lib
L = _lib.lib()
N = 65536
m4 = oracle.gen_nuclei_mask(4096, 4096, 30.0, 7)
m = torch.from_numpy(m4).cuda().repeat(N // 4096, N // 4096)
img = gw.Image2D(N, N, "binary", m)
for mode in [int(x) for x in sys.argv[1:]]:
    L.iwpp_edt_set_engine(mode)
    cfg = gw.EngineConfig()
    vm, d = gw.edt(img, gw.SE8, mode="parallel", cfg=cfg)
    del vm, d
    torch.cuda.synchronize()
    ts = []
    for _ in range(2):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); vm, d = gw.edt(img, gw.SE8); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
        del vm, d
    print(f"mode {mode}: {np.median(ts):.2f} ms rounds={cfg.stats.rounds}", flush=True)
