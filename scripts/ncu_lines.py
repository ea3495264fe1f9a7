"""Aggregate ncu source-page stall samples by CUDA source line."""
import csv, collections, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur = None; agg = collections.Counter(); src = {}; tot = 0
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur = r[1].split('/')[-1]; continue
    if r[0] in ("Function Name", "Line No"): continue
    try:
        ln = int(r[0]); s = float(r[4] or 0)
    except Exception:
        continue
    agg[(cur, ln)] += s; src[(cur, ln)] = r[1]; tot += s
for k, v in agg.most_common(n):
    print(f"{v/tot*100:5.1f}% {k[0]}:{k[1]}  {src[k].strip()[:100]}")
