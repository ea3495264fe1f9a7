"""Development probe: 16/32-bit reconstruction, shared-memory engine (engine=1)
vs the register engine (engine=0 auto), device-resident, L2 flushed."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_1209_3314_b200 as gw

torch.cuda.set_device(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=7, warm=2):
    for _ in range(warm):
        fn()
    ts = []
    for i in range(reps):
        flush.fill_(i & 0xff)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
J8, I8 = oracle.gray_pair(n, 0, h=40)
cases = {
    "i32": (torch.from_numpy(J8.astype(np.int32) * 1000 - 7), torch.from_numpy(I8.astype(np.int32) * 1000 - 7)),
    "u16": (torch.from_numpy(J8.astype(np.uint16) * 200), torch.from_numpy(I8.astype(np.uint16) * 200)),
    "f32": (torch.from_numpy(J8.astype(np.float32) * 0.5 - 3), torch.from_numpy(I8.astype(np.float32) * 0.5 - 3)),
}
for name, (J, I) in cases.items():
    dJ, dI = J.cuda(), I.cuda()
    kind = None
    for conn in (8, 4):
        outs = {}
        for eng in (1, 0):
            outs[eng] = gw.reconstruct(dJ, dI, conn, engine=eng, kind=kind)
            t = timed(lambda: gw.reconstruct(dJ, dI, conn, engine=eng, kind=kind))
            print(f"{name} {n}^2 c{conn} engine={eng}: {t:.3f} ms", flush=True)
        print(f"   same={torch.equal(outs[0], outs[1])}", flush=True)
