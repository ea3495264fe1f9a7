"""Aggregate ncu source-page 'Instructions Executed' (warp-level) by CUDA source line."""
import csv, collections, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None; agg = collections.Counter(); src = {}; tot = 0; col = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur = r[1].split('/')[-1]; continue
    if r[0] == "Line No":
        col = r.index("Instructions Executed"); continue
    if r[0] == "Function Name": continue
    try:
        ln = int(r[0]); v = float(r[col] or 0)
    except Exception:
        continue
    agg[(cur, ln)] += v; src[(cur, ln)] = r[1]; tot += v
print(f"total warp instructions: {tot:.3e}")
for k, v in agg.most_common(n):
    print(f"{v/tot*100:5.1f}% {k[0]}:{k[1]}  {src[k].strip()[:100]}")
