"""EDT engine timing: python scripts/prof_edt.py {blob,nuclei} N CONN [reps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
import paper_1209_3314_b200 as gw
kind, n, conn = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
m = oracle.gen_synthetic_mask(n, n, 50, 7) if kind == "blob" else oracle.gen_nuclei_mask(n, n, 30.0, 7)
if os.environ.get("EDT_ENGINE"):  # 3 = frontier queue, 4 = temporally blocked
    from paper_1209_3314_b200 import _lib
    _lib.lib().iwpp_edt_set_engine(int(os.environ["EDT_ENGINE"]))
img = gw.Image2D(n, n, "binary", torch.from_numpy(m).cuda())
cfg = gw.EngineConfig()
gw.edt(img, gw.StructuringElement(conn), mode="parallel", cfg=cfg)
ts = []
for r in range(reps + 2):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); gw.edt(img, gw.StructuringElement(conn)); b.record(); torch.cuda.synchronize()
    if r >= 2: ts.append(a.elapsed_time(b))
print(f"edt {kind} {n}^2 c{conn}: median {np.median(ts):.3f} ms  rounds={cfg.stats.rounds} visits={cfg.stats.queued_total} us/round={np.median(ts)*1e3/max(cfg.stats.rounds,1):.1f}")
