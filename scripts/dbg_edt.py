import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import oracle
import paper_1209_3314_b200 as gw
from paper_1209_3314_b200 import _lib
L = _lib.lib()
for n in [int(x) for x in os.environ.get("NS", "1024,1536,2048,3072,4096").split(",")]:
    m = oracle.gen_synthetic_mask(n, n, 50, 7)
    img = gw.Image2D(n, n, "binary", torch.from_numpy(m).cuda())
    L.iwpp_edt_set_engine(3)
    vq, dq = gw.edt(img, gw.SE8)
    L.iwpp_edt_set_engine(0)
    try:
        vb, db = gw.edt(img, gw.SE8)
    except Exception as e:
        print(n, "block failed:", e)
        vm, seeds = gw.init_packed(img, gw.SE8)
        gw.edt_propagate(vm, seeds, gw.SE8)
        vb = vm
    a, b = vq.vr.cpu().numpy(), vb.vr.cpu().numpy()
    bad = np.argwhere(a != b)
    print(n, "mismatches", len(bad), "inf in block", int((b < 0).sum()), bad[:5].tolist(), flush=True)
    if len(bad):
        ys, xs = bad[:, 0], bad[:, 1]
        print("  region rows", np.unique(ys // 64)[:20], "cols", np.unique(xs // 64)[:20])
