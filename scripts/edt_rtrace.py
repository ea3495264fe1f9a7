"""Per-round trace of the raster EDT engine on a bench mask
(IWPP_EDT_RTRACE=1): python scripts/edt_rtrace.py blob|nuclei [conn]
Prints the library's per-round lines (frontier size, round time, and for
raster rounds the work / barrier / compaction split) on stderr, then a
summary by frontier-size bucket."""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if os.environ.get("_RT_CHILD"):
    sys.path.insert(0, ROOT)
    import torch
    import oracle
    import paper_1209_3314_b200 as gw
    name, conn = sys.argv[1], int(sys.argv[2])
    m = (oracle.gen_nuclei_mask(4096, 4096, 30.0, 7) if name == "nuclei"
         else oracle.gen_synthetic_mask(4096, 4096, 50, 7))
    img = gw.Image2D(4096, 4096, "binary", torch.from_numpy(m).cuda())
    for _ in range(3):
        gw.edt(img, gw.StructuringElement(conn))
    torch.cuda.synchronize()
    sys.exit(0)
name = sys.argv[1] if len(sys.argv) > 1 else "blob"
conn = sys.argv[2] if len(sys.argv) > 2 else "8"
env = dict(os.environ, _RT_CHILD="1", IWPP_EDT_RTRACE="1")
p = subprocess.run([sys.executable, __file__, name, conn], env=env, capture_output=True, text=True)
lines = [l for l in p.stderr.splitlines() if l.startswith("[edt rtrace]")]
# the last call's rounds
starts = [i for i, l in enumerate(lines) if " round 0 " in l]
last = lines[starts[-1]:] if starts else lines
rx = re.compile(r"round (\d+) n (\d+) dt_us ([\d.]+) work_us ([\d.]+) bar_us ([\d.]+) comp_us ([\d.]+)")
rows = [tuple(float(x) for x in rx.search(l).groups()) for l in last if rx.search(l)]
rows = [r for r in rows if r[1] > 0]  # (round 0 runs inside the init: no stamp)
buckets = [(0, 1024), (1024, 16384), (16384, 65536), (65536, 262144), (262144, 1 << 40)]
print(f"{name} c{conn}: {len(rows)} rounds traced, total {sum(r[2] for r in rows) / 1e3:.3f} ms")
for lo, hi in buckets:
    sel = [r for r in rows if lo <= r[1] < hi]
    if sel:
        t = sum(r[2] for r in sel)
        print(f"  frontier [{lo}, {hi}): {len(sel)} rounds, {t / 1e3:.3f} ms, {t / len(sel):.2f} us/round, "
              f"mean n {sum(r[1] for r in sel) / len(sel):.0f}, work {sum(r[3] for r in sel) / len(sel):.2f} "
              f"bar {sum(r[4] for r in sel) / len(sel):.2f} comp {sum(r[5] for r in sel) / len(sel):.2f}")
if os.environ.get("RT_ALL"):
    print("\n".join(last))
