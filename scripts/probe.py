"""Quick device timings for development (not the bench contract)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import paper_1209_3314_b200 as gw

def timeit(fn, reps=10, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return np.median(ts), min(ts)

which = sys.argv[1:] or ["recon", "imfill", "edt"]
if "recon" in which:
  for n, conn in [(4096, 8), (4096, 4)]:
    J, I = oracle.gray_pair(n, 0, h=40)
    dJ, dI = torch.from_numpy(J).cuda(), torch.from_numpy(I).cuda()
    for sw, tsw in [(0, 0), (0, 1), (0, 2), (0, 3), (0, 4)]:
        st = {}
        gw.reconstruct(dJ, dI, conn, sweeps=sw, tile_sweeps=tsw, stats=st)
        med, mn = timeit(lambda: gw.reconstruct(dJ, dI, conn, sweeps=sw, tile_sweeps=tsw))
        print(f"recon u8 {n}^2 c{conn} sweeps={sw} tile_sweeps={tsw}: median {med:.3f} ms min {mn:.3f} ms  {n*n/med/1e3:.0f} Mpx/s  stats={st}", flush=True)
if "imfill" in which:
  bw = oracle.gen_synthetic_mask(4096, 4096, 50, 7)
  bw16 = np.tile(bw, (4, 4))
  mk, ms = oracle.imfill_pair(bw16)
  dJ, dI = torch.from_numpy(mk).cuda(), torch.from_numpy(ms).cuda()
  for conn in (4, 8):
    for sw, tsw in [(0, 1), (0, 2), (1, 1)]:
        st = {}
        gw.reconstruct(dJ, dI, conn, sweeps=sw, tile_sweeps=tsw, stats=st)
        med, mn = timeit(lambda: gw.reconstruct(dJ, dI, conn, sweeps=sw, tile_sweeps=tsw), reps=3, warm=1)
        n = 16384
        print(f"imfill 16K^2 c{conn} sweeps={sw} tile_sweeps={tsw}: median {med:.3f} ms  {n*n/med/1e3:.0f} Mpx/s stats={st}", flush=True)
if "edt" in which:
  bw = oracle.gen_synthetic_mask(4096, 4096, 50, 7)
  for name, m in [("nuclei4k", oracle.gen_nuclei_mask(4096, 4096, 30.0, 7)), ("blob4k", bw)]:
    dm = torch.from_numpy(m).cuda()
    img = gw.Image2D(4096, 4096, "binary", dm)
    cfg = gw.EngineConfig()
    gw.edt(img, gw.SE8, mode="parallel", cfg=cfg)
    med, mn = timeit(lambda: gw.edt(img, gw.SE8), reps=5, warm=2)
    print(f"edt {name} c8: median {med:.3f} ms  {4096*4096/med/1e3:.0f} Mpx/s rounds={cfg.stats.rounds} visits={cfg.stats.queued_total}", flush=True)
