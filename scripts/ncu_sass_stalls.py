"""Top stalled SASS instructions of an ncu report with their stall reasons:
python scripts/ncu_sass_stalls.py REPORT [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = rows[2:]
reasons = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
tot = sum(float(r[2] or 0) for r in data) or 1
agg = {}
for r in data:
    for i in reasons:
        agg[h[i]] = agg.get(h[i], 0) + float(r[i] or 0)
print("stall reasons (share of all samples):",
      ", ".join(f"{k[6:]} {v / tot * 100:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1]) if v))
top = sorted(range(len(data)), key=lambda i: -float(data[i][2] or 0))[:n]
for i in sorted(top):
    r = data[i]
    rs = sorted(((float(r[j] or 0), h[j][6:]) for j in reasons), reverse=True)[:2]
    why = ", ".join(f"{nm} {v / tot * 100:.1f}" for v, nm in rs if v)
    print(f"{float(r[2]) / tot * 100:5.1f}% [{i:4d}] {r[1].strip()[:64]:64s} ({why})")
