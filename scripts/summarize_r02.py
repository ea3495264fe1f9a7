"""Round-2 ncu evidence -> profiles/ (committed):

  python scripts/summarize_r02.py gpurun_out/r02

For every <case>.raw.csv (ncu --set full + L2 atomic counters, one row per
captured launch) writes the key metrics per kernel to profiles/r02_ncu.txt,
copies the per-line / per-SASS stall summaries, summarises the launch list
(launches.csv) and updates profiles/ncu_summary.json (the dram bytes per
launch bench.py reports as roofline.traffic)."""
import collections
import csv
import io
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
SRC = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "r02")
TAG = sys.argv[2] if len(sys.argv) > 2 else "r02"  # output prefix (r02b: the re-captures)

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 % peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("lts__t_requests_op_atom.sum", "L2 atom requests"),
    ("lts__t_requests_op_red.sum", "L2 red requests"),
    ("lts__t_sectors_op_atom.sum", "L2 atom sectors"),
    ("lts__t_sectors_op_red.sum", "L2 red sectors"),
    ("lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed", "L2 atomic unit busy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]
# case -> (ncu_summary key, kernel-name substring, algorithmic bytes per launch or None)
SUMMARY_KEYS = {
    "recon_u8_4k": [("recon_tile_engine_u8_c8", "tile_engine_reg_kernel", 3 * 4096 * 4096)],
    "recon_i32_4k": [("recon_tile_engine_reg32_i32_c8", "tile_engine_reg32_kernel", 12 * 4096 * 4096)],
    "recon_u8_64k": [("recon_tile_engine_u8_c8_64k", "tile_engine_reg_kernel", 3 * 65536 * 65536)],
    "imfill_16k": [("recon_tile_engine_bin_c8_16k", "tile_engine_bin_kernel", 3 * 16384 * 16384)],
    "edt_blob4k": [("edt_rounds_blob4k_c8", "edt_rounds_raster_kernel", None)],
    "edt_nuclei4k": [("edt_rounds_nuclei4k_c8", "edt_rounds_raster_kernel", None)],
    "edt_nuclei64k": [("edt_init_nuclei64k", "edt_init_key_rows", 17 * 65536 * 65536),
                      ("edt_finalize_nuclei64k", "edt_finalize_key_kernel", 20 * 65536 * 65536)],
    "edt_mg_blob4k": [("edt_mg_rounds_blob4k_4slabs", "mg_rounds_kernel", None)],
}


def unit_scale(unit):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
            "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
            "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}.get(unit, 1.0)


def read_raw(path):
    rows = list(csv.reader(open(path)))
    head, units, data = rows[0], rows[1], rows[2:]
    out = []
    for r in data:
        d = {"kernel": r[head.index("Kernel Name")]}
        for i, h in enumerate(head):
            name = h.split(".", 2)[-1] if h.count(".") >= 2 and h.split(".")[0].isupper() else h
            d[h] = (r[i], units[i])
            d.setdefault(name, (r[i], units[i]))
        out.append(d)
    return out


def val(d, key):
    if key not in d:
        return None
    v, u = d[key]
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    if u in ("byte", "Kbyte", "Mbyte", "Gbyte", "Tbyte"):
        return x * unit_scale(u)
    if u in ("nsecond", "usecond", "msecond", "second", "ns", "us", "ms", "s"):
        return x * unit_scale(u) * 1e3  # ms
    return x


def fmt(key, x):
    if x is None:
        return "-"
    if isinstance(x, str):
        return x
    if key.startswith("dram__bytes"):
        return f"{x / 1e6:.1f} MB"
    if key == "gpu__time_duration.sum":
        return f"{x:.4f} ms"
    return f"{x:,.1f}" if abs(x) < 1e6 else f"{x:,.0f}"


def main():
    os.makedirs(PROF, exist_ok=True)
    summary_path = os.path.join(PROF, "ncu_summary.json")
    summary = json.load(open(summary_path)) if os.path.exists(summary_path) else {}
    lines = [f"# Round-2 ncu captures ({TAG}; B200, --set full + L2 atomic counters, --clock-control none;",
             "# scripts/prof_r02.sh / prof_r02b.sh, workloads scripts/prof_r02.py). One block per captured launch.", ""]
    for f in sorted(os.listdir(SRC)):
        if not f.endswith(".raw.csv"):
            continue
        case = f[:-len(".raw.csv")]
        for d in read_raw(os.path.join(SRC, f)):
            lines.append(f"[{case}] {d['kernel'][:110]}")
            for key, label in KEYS:
                lines.append(f"    {label:24s} {fmt(key, val(d, key))}")
            t = val(d, "gpu__time_duration.sum")
            rb, wb = val(d, "dram__bytes_read.sum"), val(d, "dram__bytes_write.sum")
            if t and rb is not None:
                lines.append(f"    {'dram GB/s':24s} {(rb + wb) / (t / 1e3) / 1e9:,.1f}")
            for skey, sub, alg in SUMMARY_KEYS.get(case, []):
                if sub in d["kernel"]:
                    ent = {"kernel": d["kernel"][:120], "report": f"{TAG}/{case}",
                           "time_ms": t, "dram_bytes_per_launch": int((rb or 0) + (wb or 0)),
                           "l2_atom_requests": val(d, "lts__t_requests_op_atom.sum"),
                           "l2_red_requests": val(d, "lts__t_requests_op_red.sum"),
                           "l2_atomic_unit_busy_pct": val(
                               d, "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                           "issue_active_pct": val(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                           "dram_pct_peak": val(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")}
                    if alg:
                        ent["alg_bytes_per_launch"] = alg
                        ent["traffic_over_alg"] = round(ent["dram_bytes_per_launch"] / alg, 3)
                    summary[skey] = ent
            lines.append("")
        for ext in (".lines.txt", ".sass.txt"):
            p = os.path.join(SRC, case + ext)
            if os.path.exists(p) and os.path.getsize(p):
                shutil.copy(p, os.path.join(PROF, f"{TAG}_stalls_{case}{ext.replace('.txt', '')}.txt"))
    open(os.path.join(PROF, f"{TAG}_ncu.txt"), "w").write("\n".join(lines) + "\n")
    json.dump(summary, open(summary_path, "w"), indent=1, sort_keys=True)
    # launch list of the headline bench command
    lp = os.path.join(SRC, "launches.csv")
    if os.path.exists(lp):
        txt = open(lp).read().splitlines()
        start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
        agg = collections.defaultdict(lambda: [0, 0.0])
        for r in csv.DictReader(io.StringIO("\n".join(txt[start:]))):
            if r["Metric Name"] != "gpu__time_duration.sum":
                continue
            v = float(r["Metric Value"].replace(",", "")) * {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3,
                                                             "ms": 1e6, "msecond": 1e6}.get(r["Metric Unit"], 1)
            name = r["Kernel Name"].split("(")[0]
            agg[name][0] += 1
            agg[name][1] += v
        tot = sum(v[1] for v in agg.values()) or 1
        out = ["# ncu launch list of `python bench.py --steps 3 --warmup 3 --no-extras --no-cpu` (headline",
               "# steps + e2e host-pipeline calls), gpu__time_duration.sum, --clock-control none: cold and",
               "# serialised -- compare each kernel's share, not absolute times.",
               f"{'kernel':72s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share':>7s}"]
        for k, (n, ns) in sorted(agg.items(), key=lambda x: -x[1][1]):
            out.append(f"{k[:72]:72s} {n:8d} {ns / 1e3:10.1f} {ns / 1e3 / n:9.2f} {ns / tot * 100:6.1f}%")
        open(os.path.join(PROF, f"{TAG}_launches.txt"), "w").write("\n".join(out) + "\n")
    print("ok")


if __name__ == "__main__":
    main()
