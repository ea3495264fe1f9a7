"""Aggregate ncu source-page 'Instructions Executed' (and stall samples) by
CUDA source line: python scripts/ncu_inst_lines.py REPORT [N]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
cur = None
inst = collections.Counter()
samp = collections.Counter()
src = {}
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    try:
        inst[(cur, ln)] += float(r[7] or 0)
        samp[(cur, ln)] += float(r[4] or 0)
    except (ValueError, IndexError):
        continue
    src[(cur, ln)] = r[1]
ti = sum(inst.values()) or 1
ts = sum(samp.values()) or 1
print(f"total instructions {ti:.0f}")
for k, v in inst.most_common(n):
    print(f"{v / ti * 100:5.1f}% inst {samp[k] / ts * 100:5.1f}% stall  {k[0]}:{k[1]}  {src[k].strip()[:90]}")
