"""Summarise ncu outputs from gpurun_out/ into profiles/ (committed evidence).

  python scripts/summarize_ncu.py --round 1 --launches gpurun_out/launches.csv \
      --full gpurun_out/prof_tile.ncu-rep:recon_tile_engine_u8_c8 [...]

Writes profiles/r<NN>_launches.txt (per-kernel share of the launch list),
profiles/r<NN>_<key>.txt (key metrics of each full capture) and updates
profiles/ncu_summary.json (dram bytes per launch etc., read by bench.py).
"""

import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEY_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sectors.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
]


def read_csv_rows(path):
    txt = open(path).read().splitlines()
    start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
    return list(csv.DictReader(io.StringIO("\n".join(txt[start:]))))


def launches(path, out):
    rows = read_csv_rows(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"])
        if r["Metric Unit"] == "us":
            v *= 1e3
        elif r["Metric Unit"] == "ms":
            v *= 1e6
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values()) or 1.0
    lines = [f"# ncu launch list ({os.path.basename(path)}): gpu__time_duration.sum, "
             "--clock-control none (cold, serialised: compare shares, not absolutes)",
             f"{'kernel':70s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share':>7s}"]
    for k, (n, ns) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k[:70]:70s} {n:8d} {ns / 1e3:10.1f} {ns / n / 1e3:9.2f} {ns / tot:7.1%}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep, key, round_no):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    vals = rows[2]
    kname = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else key
    d = {"kernel": kname, "report": os.path.basename(rep)}
    lines = [f"# ncu --set full: {kname}", f"# report {os.path.basename(rep)}"]
    for m in KEY_METRICS:
        if m in hdr:
            i = hdr.index(m)
            d[m] = vals[i]
            lines.append(f"{m:65s} {vals[i]:>18s} {units[i]}")

    def num(m, unit_scale=None):
        if m not in hdr:
            return None
        i = hdr.index(m)
        v = float(vals[i].replace(",", ""))
        u = units[i]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
                 "ms": 1e-3, "usecond": 1e-6, "nsecond": 1e-9, "msecond": 1e-3}.get(u, 1)
        return v * scale

    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    if rd is not None and wr is not None:
        d["dram_bytes_per_launch"] = int(rd + wr)
        lines.append(f"{'dram bytes per launch (read+write)':65s} {int(rd + wr):>18d} byte")
    out = os.path.join(PROF, f"r{round_no:02d}_{key}.txt")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", type=int, required=True)
    ap.add_argument("--launches")
    ap.add_argument("--full", nargs="*", default=[])
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if a.launches:
        launches(a.launches, os.path.join(PROF, f"r{a.round:02d}_launches.txt"))
    sp = os.path.join(PROF, "ncu_summary.json")
    summ = json.load(open(sp)) if os.path.exists(sp) else {}
    for spec in a.full:
        rep, key = spec.split(":")
        summ[key] = full(rep, key, a.round)
    json.dump(summ, open(sp, "w"), indent=1)


if __name__ == "__main__":
    main()
