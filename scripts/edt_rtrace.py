"""Per-round timeline of the raster EDT engine (IWPP_EDT_RTRACE=1): one run,
then a fit of round time against frontier size."""
import os
import re
import subprocess
import sys

import numpy as np

kind = sys.argv[1] if len(sys.argv) > 1 else "blob"
env = dict(os.environ, IWPP_EDT_RTRACE="1")
code = f"""
import sys; sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
import torch, oracle, paper_1209_3314_b200 as gw
n = 4096
m = oracle.gen_synthetic_mask(n, n, 50, 7) if {kind!r} == "blob" else oracle.gen_nuclei_mask(n, n, 30.0, 7)
img = gw.Image2D(n, n, "binary", torch.from_numpy(m).cuda())
gw.edt(img, gw.SE8)
"""
out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True).stderr
rows = [(int(a), int(b), float(c)) for a, b, c in
        re.findall(r"round (\d+) n (\d+) dt_us ([0-9.]+)", out)]
ph = np.array([(float(a), float(b), float(c)) for a, b, c in
               re.findall(r"work_us ([0-9.]+) bar_us ([0-9.]+) comp_us ([0-9.]+)", out)])
rows = rows[-(len(rows) // 2):] if len(rows) > 400 else rows  # last run only
n = np.array([r[1] for r in rows], float)
t = np.array([r[2] for r in rows])
print(f"{kind}: rounds {len(rows)} total {t.sum() / 1e3:.2f} ms, median {np.median(t):.1f} us/round")
for lo, hi in [(0, 1e3), (1e3, 1e4), (1e4, 5e4), (5e4, 1.5e5), (1.5e5, 2.62e5), (2.62e5, 1e9)]:
    sel = (n >= lo) & (n < hi)
    if sel.any():
        print(f"  n in [{lo:.0f},{hi:.0f}): {sel.sum():4d} rounds, mean n {n[sel].mean():9.0f}, "
              f"mean {t[sel].mean():6.1f} us, total {t[sel].sum() / 1e3:.2f} ms")
rs = ph[:, 0] > 0 if ph.ndim == 2 else np.zeros(0, bool)
if rs.any():
    w, b, c3 = ph[rs].mean(0)
    print(f"  raster rounds (block 0): work {w:.1f} us, phase-1 barrier wait {b:.1f} us, compaction {c3:.1f} us")
A = np.vstack([np.ones_like(n), n]).T
q = n < 262144
c = np.linalg.lstsq(A[q], t[q], rcond=None)[0]
print(f"  queue rounds fit: {c[0]:.1f} us + {c[1] * 1e3:.2f} us per 1000 items")
if (~q).any():
    c2 = np.linalg.lstsq(A[~q], t[~q], rcond=None)[0]
    print(f"  raster rounds fit: {c2[0]:.1f} us + {c2[1] * 1e3:.2f} us per 1000 items")
