#!/usr/bin/env python
"""Benchmark: megapixels/s of grayscale morphological reconstruction on B200.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W`` prints
ONE JSON line on rank 0.  N > 1 runs under torchrun, one rank per GPU.

Workload (BASELINE.json configs[1]): reconstruction by dilation of a
4096x4096 uint8 random marker/mask pair (mask ~ U[0,256), marker =
max(mask - 40, 0); the generator of the reference's bench/verify/acceptance
tests), 8-connectivity.  One step = one reference ``recon_fh`` call on the
device: copy the marker (the reference works on a copy, recon.py:63-64) and
run the engine to the fixed point.  Inputs are resident in HBM; the L2
(126 MB > the 48 MB of state) is flushed between timed steps by writing a
256 MB buffer outside the timed events.  With N GPUs every rank processes
its own tile (independent tiles, no data-path collective): weak scaling,
value = all ranks' pixels / max-over-ranks device time.  (N > 1: the
headline is BASELINE configs[4] instead -- the 64K^2 whole slide as
horizontal slabs with NCCL border exchange, strong scaling; see
slide_headline.)

Extra keys: ``e2e`` (the same metric through the host-buffer C-ABI call,
H2D + D2H inside the timed region), ``roofline`` (the tile-engine kernel vs
the measured HBM copy bandwidth), ``cpu_baseline`` (the CPU restatement of
the reference algorithm, timed on this host's cores), ``extras`` (4-conn,
int32, EDT and imfill configs of BASELINE.json, single GPU).

``--impl reference`` times the reference's CPU algorithm (the C restatement
in oracle/: the reference is Python+numba, not compilable
here) on all host cores, on the same workload and metric.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_PX = 4096
H_MARKER = 40
METRIC = "Megapixels/sec: gray morph reconstruction + EDT, 1/2/4/8 B200 vs CPU ref"
WORKLOAD = "recon_by_dilation 4096x4096 u8 random marker/mask (h=40), 8-connectivity"
ALG_BYTES_PER_PX = 3  # read marker + read mask + write result


def gray_pair(n: int, seed: int, h: int = H_MARKER):
    """The reference's marker/mask generator (test_acceptance.py:54-57)."""
    rng = np.random.default_rng(seed)
    I = rng.integers(0, 256, (n, n)).astype(np.uint8)
    J = np.maximum(I.astype(np.int32) - h, 0).astype(np.uint8)
    return J, I


_JSON_OUT = None


def emit(line: dict):
    """The one JSON line, to the real stdout (see main)."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def measured_peak_gbs():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(kernel_key: str):
    """DRAM bytes per launch of a kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d[kernel_key]["dram_bytes_per_launch"]
    except Exception:
        return None


# ---------------------------------------------------------------------------
# clocks sampled during the timed region

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            parts = [p.strip() for p in l.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU legs (oracle = the CPU restatement of the reference algorithm)

def cpu_fh_throughput(J, I, conn, threads: int, rounds: int):
    """`threads` concurrent recon_fh runs (ctypes drops the GIL) x rounds.
    Returns (Mpx/s, wall seconds, runs)."""
    import oracle

    oracle.lib()
    runs = threads * rounds
    errs = []

    def work():
        try:
            for _ in range(rounds):
                oracle.recon_fh(J, I, conn)
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ts = [threading.Thread(target=work) for _ in range(threads)]
    t0 = time.perf_counter()
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    wall = time.perf_counter() - t0
    if errs:
        raise errs[0]
    return runs * J.size / wall / 1e6, wall, runs


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return 0
    J, I = gray_pair(N_PX, 0)
    cores = host_cores()
    for _ in range(args.warmup):
        cpu_fh_throughput(J, I, 8, cores, 1)
    t_steps = []
    px = 0
    for _ in range(args.steps):
        _, wall, runs = cpu_fh_throughput(J, I, 8, cores, 1)
        t_steps.append(wall)
        px += runs * J.size
    total = sum(t_steps)
    value = px / total / 1e6
    sample = (f"{cores} concurrent recon_fh runs of the 4096^2 u8 8-conn workload per step "
              f"(C restatement of the reference, oracle/iwpp_oracle.c)")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "Mpx/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * total / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": WORKLOAD, "shape": [N_PX, N_PX], "conn": 8, "l2": "n/a (CPU)"},
        "cpu_baseline": {"value": round(value, 3), "unit": "Mpx/s", "cores": cores,
                         "kind": "port", "sample": sample},
        "e2e": {"value": round(value, 3), "unit": "Mpx/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


# ---------------------------------------------------------------------------
# device legs

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-whole-slide", action="store_true",
                    help="skip the 64K^2 whole-slide extras (recon + EDT)")
    ap.add_argument("--whole-slide-only", action="store_true",
                    help="(diagnostics) skip the 4K/16K extras, keep the whole slide")
    ap.add_argument("--slide-headline", choices=("auto", "on", "off"), default="auto",
                    help="headline = the 64K^2 whole slide over the ranks' slabs (BASELINE configs[4]); "
                         "auto: for N > 1 (configs[1], the 4K tile, at N = 1)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    # stdout carries exactly one JSON line: everything else any library
    # writes to fd 1 (NCCL / torch banners at communicator creation) goes
    # to stderr; the line itself goes to the saved stdout (emit())
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, rank, world)
    # NCCL's version banner goes to stdout, which must carry only the JSON line
    if not os.environ.get("IWPP_KEEP_NCCL_DEBUG"):
        os.environ["NCCL_DEBUG"] = "WARN"

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))

    from paper_1209_3314_b200 import _lib
    from paper_1209_3314_b200.build import LIB

    L = _lib.lib()
    dev = torch.device(f"cuda:{local}")
    if args.slide_headline == "on" or (args.slide_headline == "auto" and world > 1):
        return slide_headline(args, rank, world, local, dev)
    Jh, Ih = gray_pair(N_PX, rank)
    dJ = torch.from_numpy(Jh).to(dev)
    dI = torch.from_numpy(Ih).to(dev)
    out = torch.empty_like(dJ)
    W = H = N_PX
    ws = _lib.workspace(L.iwpp_recon_workspace_bytes(W, H, 0, 8))
    opts = _lib.ReconOpts()
    opts.sweeps, opts.max_blocks, opts.check_contract, opts.queue_capacity = -1, 0, 0, 0
    opts.tile_sweeps, opts.halo_sweep_threshold = -1, -1
    # no events inside the call: each timed step is exactly one engine launch
    # between s0 and s1 (two more event records in the stream cost ~3.7 us)
    opts.ev_begin = opts.ev_end = None
    stream = _lib.stream_ptr()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > L2 (126 MB)

    opts.marker = _lib.ptr(dJ)  # the operator starts from a copy of the marker (copied by the engine)

    def step():
        _lib.check(L.iwpp_recon(_lib.ptr(out), _lib.ptr(dI), W, H, 0, 8, _lib.ptr(ws),
                                ws.numel(), _lib.ctypes.byref(opts), None, stream), "recon")

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    step_ms, kern_ms = [], []
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xff)  # evict the inputs from L2 (outside the timed events)
            s0.record()
            step()
            s1.record()
            s1.synchronize()
            step_ms.append(s0.elapsed_time(s1))
            kern_ms.append(step_ms[-1])  # the step is the one engine launch
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = float(sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())

    # parity spot check of the benchmarked output (bit-exact oracle on rank 0)
    ok = None
    if rank == 0 and not args.no_cpu:
        import oracle
        ok = bool(np.array_equal(out.cpu().numpy(), oracle.recon_fh(Jh, Ih, 8)))

    # e2e: host buffers through the C ABI (H2D + D2H inside the timed region)
    pin_J = torch.from_numpy(Jh).pin_memory()
    pin_I = torch.from_numpy(Ih).pin_memory()
    pin_O = torch.empty_like(pin_J).pin_memory()
    wsh = _lib.workspace(L.iwpp_recon_host_workspace_bytes(W, H, 0, 8))
    e2e_opts = _lib.ReconOpts()
    e2e_opts.sweeps, e2e_opts.max_blocks, e2e_opts.check_contract = -1, 0, 0
    e2e_opts.queue_capacity, e2e_opts.tile_sweeps, e2e_opts.halo_sweep_threshold = 0, -1, -1

    def e2e_step():
        _lib.check(L.iwpp_recon_host(_lib.ptr(pin_O.numpy()), _lib.ptr(pin_J.numpy()),
                                     _lib.ptr(pin_I.numpy()), W, H, 0, 8, _lib.ptr(wsh),
                                     wsh.numel(), _lib.ctypes.byref(e2e_opts), None, stream),
                   "recon_host")

    for _ in range(2):
        e2e_step()
    e2e_t = []
    for i in range(args.steps):
        flush.fill_(i & 0xff)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_step()  # synchronous: returns after the D2H copy
        e2e_t.append(time.perf_counter() - t0)
    e2e_total = sum(e2e_t)
    if world > 1:
        t = torch.tensor([e2e_total], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_val = world * args.steps * W * H / e2e_total / 1e6

    value = world * args.steps * W * H / (total_ms / 1e3) / 1e6
    peak, peak_kind = measured_peak_gbs()
    kavg = statistics.mean(kern_ms)
    achieved = ALG_BYTES_PER_PX * W * H / (kavg / 1e3) / 1e9

    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "Mpx/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (reference generator: mask ~ U[0,256), marker = max(mask-40, 0))",
        "config": {"workload": WORKLOAD, "shape": [H, W], "conn": 8,
                   "per_rank_tiles": 1, "parallelism": f"independent tiles x{world}",
                   "l2": "flushed between timed steps (256 MB write outside the events)"},
        "clocks": clk.summary(),
        "e2e": {"value": round(e2e_val, 2), "unit": "Mpx/s",
                "h2d_bytes_per_step": 2 * W * H, "d2h_bytes_per_step": W * H,
                "path": "iwpp_recon_host (pinned host buffers, C ABI)"},
        "gpu_launches": args.steps,  # one engine kernel per step (marker copy in its prologue)
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": ncu_traffic("recon_tile_engine_u8_c8"),
                     "kernel": "tile_engine_reg_kernel<8> (u8 register engine)",
                     "kernel_ms": round(kavg, 4), "alg_bytes_per_px": ALG_BYTES_PER_PX,
                     "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"},
        "library": os.path.relpath(LIB, ROOT),
        "parity_vs_oracle": ok,
    }

    if rank == 0 and world == 1 and not args.no_cpu:
        J, I = Jh, Ih
        cores = host_cores()
        rounds = 1
        v, wall, runs = cpu_fh_throughput(J, I, 8, cores, rounds)
        line["cpu_baseline"] = {
            "value": round(v, 3), "unit": "Mpx/s", "cores": cores, "kind": "port",
            "sample": f"{runs} recon_fh runs of the 4096^2 u8 8-conn workload on {cores} "
                      f"threads ({wall:.1f} s wall; oracle/iwpp_oracle.c)"}

    if rank == 0 and world == 1 and not args.no_extras and not args.whole_slide_only:
        line["extras"] = extras(L, _lib, dev, flush, peak, cpu=not args.no_cpu)
    if not args.no_extras and not args.no_whole_slide:
        del dJ, dI, out, ws, wsh
        torch.cuda.empty_cache()
        try:
            ws_line = whole_slide(dev, rank, world, flush, peak, check=not args.no_cpu)
        except Exception as e:  # the headline line must still print
            ws_line = {"whole_slide_error": f"{type(e).__name__}: {e}"[:300]}
        if rank == 0:
            # BASELINE configs[4] (the 64K^2 whole slide, strong scaling over
            # the ranks' slabs with NVLink border exchange) as its own block
            line["whole_slide"] = {
                "workload": "65536x65536 whole slide: recon u8 8-conn (counter-hash random pair) + "
                            "EDT 8-conn (4K nuclei mask tiled 16x16); horizontal slabs x N",
                "scaling": "strong", "n_gpus": world, **ws_line}

    if rank == 0:
        emit(line)
    if world > 1:
        dist.destroy_process_group()
    return 0


def cpu_concurrent(fn, px_per_call: int, threads: int, what: str):
    """`threads` concurrent calls of the oracle (ctypes drops the GIL), one
    per thread: the reference's CPU algorithm on this host's cores."""
    errs = []

    def work():
        try:
            fn()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ts = [threading.Thread(target=work) for _ in range(threads)]
    t0 = time.perf_counter()
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    wall = time.perf_counter() - t0
    if errs:
        raise errs[0]
    return {"value": round(threads * px_per_call / wall / 1e6, 3), "unit": "Mpx/s",
            "cores": threads, "kind": "port",
            "sample": f"{threads} concurrent {what} on {threads} threads ({wall:.1f} s wall; "
                      f"oracle/iwpp_oracle.c)"}


def extras(L, _lib, dev, flush, peak: float, cpu: bool = True):
    """Secondary BASELINE.json configs (single GPU).  Each row: device time
    (median of a few device-resident calls, L2 flushed in between), Mpx/s,
    roofline fraction on the algorithmic bytes, bit-exact
    parity against the CPU oracle on the same input, and the oracle timed on
    the host cores (cpu_baseline)."""
    import torch
    import paper_1209_3314_b200 as gw
    import oracle  # checker + CPU baseline + input generators

    out = {}
    cores = host_cores()

    def timed(fn, reps=5, warm=2):
        for _ in range(warm):
            fn()
        ts = []
        for i in range(reps):
            flush.fill_(i & 0xff)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    def row(ms, px, bpp, **kw):
        ach = bpp * px / (ms / 1e3) / 1e9
        return {"ms": round(ms, 4), "mpx_s": round(px / ms / 1e3, 1),
                "roofline_frac": round(ach / peak, 4), "alg_bytes_per_px": bpp, **kw}

    # recon 4K u8 c4 and int32 c8 (C2 variants)
    J, I = gray_pair(N_PX, 0)
    rng = np.random.default_rng(0)
    I32 = rng.integers(0, 2**31 - 1, (N_PX, N_PX), dtype=np.int32)
    J32 = np.maximum(I32.astype(np.int64) - (1 << 28), 0).astype(np.int32)
    for name, (Jh, Ih, conn, bpp) in {"recon_4k_u8_c4": (J, I, 4, 3),
                                      "recon_4k_i32_c8": (J32, I32, 8, 12)}.items():
        dJ, dI = torch.from_numpy(Jh).to(dev), torch.from_numpy(Ih).to(dev)
        res = {}
        ms = timed(lambda: res.__setitem__("J", gw.reconstruct(dJ, dI, conn)))
        r = row(ms, Jh.size, bpp)
        if cpu:
            r["parity_vs_oracle"] = bool(np.array_equal(res["J"].cpu().numpy(),
                                                        oracle.recon_fh(Jh, Ih, conn)))
            r["cpu_baseline"] = cpu_concurrent(lambda: oracle.recon_fh(Jh, Ih, conn), Jh.size,
                                               cores, f"recon_fh runs ({name})")
        out[name] = r
        del dJ, dI, res

    # EDT 4K (C3): nuclei c8 / c4 and the blob mask c8; 13 B/px = mask + vr + dist
    masks = {"nuclei": oracle.gen_nuclei_mask(N_PX, N_PX, 30.0, 7),
             "blob": oracle.gen_synthetic_mask(N_PX, N_PX, 50, 7)}
    for name, kind, conn in (("edt_4k_nuclei_c8", "nuclei", 8), ("edt_4k_nuclei_c4", "nuclei", 4),
                             ("edt_4k_blob_c8", "blob", 8)):
        m = masks[kind]
        se = gw.SE8 if conn == 8 else gw.SE4
        img = gw.Image2D(N_PX, N_PX, "binary", torch.from_numpy(m).to(dev))
        cfg = gw.EngineConfig()
        gw.edt(img, se, mode="parallel", cfg=cfg)
        res = {}
        ms = timed(lambda: res.__setitem__("r", gw.edt(img, se)), reps=3)
        r = row(ms, m.size, 13, rounds=cfg.stats.rounds)
        if cpu:
            vr_ref, d_ref, (rounds_ref, _) = oracle.edt(m, conn, stats=True)
            vm, dist = res["r"]
            r["parity_vs_oracle"] = bool(
                np.array_equal(vm.vr.cpu().numpy(), vr_ref)
                and dist.data.cpu().numpy().tobytes() == d_ref.tobytes()
                and rounds_ref == cfg.stats.rounds)
            r["cpu_baseline"] = cpu_concurrent(lambda: oracle.edt(m, conn), m.size, cores,
                                               f"edt runs ({name})")
        out[name] = r
        del img, res

    # imfill 16K (C4): binary reconstruction, 3 B/px
    bw = np.tile(masks["blob"], (4, 4))
    mk, msk = oracle.imfill_pair(bw)
    dM, dK = torch.from_numpy(mk).to(dev), torch.from_numpy(msk).to(dev)
    for conn in (4, 8):
        res = {}
        ms = timed(lambda: res.__setitem__("J", gw.reconstruct(dM, dK, conn, kind="binary")),
                   reps=3, warm=1)
        r = row(ms, bw.size, 3)
        if cpu:
            r["parity_vs_oracle"] = bool(np.array_equal(res["J"].cpu().numpy(),
                                                        oracle.recon_fh(mk, msk, conn)))
            th = min(cores, 8)  # 16K^2 oracle state is ~2.7 GB per run
            r["cpu_baseline"] = cpu_concurrent(lambda: oracle.recon_fh(mk, msk, conn), bw.size,
                                               th, f"imfill recon_fh runs (16K^2 c{conn})")
        out[f"imfill_16k_c{conn}"] = r
        del res
    return out


WS_PX = 65536  # BASELINE configs[4]: 64K x 64K whole slide


def slide_rows(y0: int, y1: int, N: int, dev, h: int = H_MARKER):
    """The 64K whole-slide recon pair, rows [y0, y1): mask = a counter hash of
    the GLOBAL pixel index (uniform bytes), marker = max(mask - h, 0).  Every
    rank count N generates the identical slide, so N=G is checked against
    N=1 bit for bit.  All products stay below 2^63 (31-bit multipliers on
    32-bit states)."""
    import torch
    I = torch.empty((y1 - y0, N), dtype=torch.uint8, device=dev)
    M32 = 0xFFFFFFFF
    for a in range(y0, y1, 1024):
        b = min(y1, a + 1024)
        x = torch.arange(a * N, b * N, dtype=torch.int64, device=dev) & M32
        x = (x * 1103515245 + 12345) & M32
        x = x ^ (x >> 15)
        x = (x * 1664525 + 1013904223) & M32
        x = x ^ (x >> 13)
        x = (x * 1597334677) & M32
        x = x ^ (x >> 16)
        I[a - y0:b - y0] = ((x >> 8) & 255).to(torch.uint8).view(b - a, N)
    M = torch.clamp(I.to(torch.int16) - h, min=0).to(torch.uint8)
    return M, I


def slide_rows_np(y0: int, y1: int, N: int, h: int = H_MARKER):
    """slide_rows on the host (numpy, same arithmetic): the oracle's input."""
    M32 = 0xFFFFFFFF
    x = np.arange(y0 * N, y1 * N, dtype=np.int64) & M32
    x = (x * 1103515245 + 12345) & M32
    x ^= x >> 15
    x = (x * 1664525 + 1013904223) & M32
    x ^= x >> 13
    x = (x * 1597334677) & M32
    x ^= x >> 16
    I = ((x >> 8) & 255).astype(np.uint8).reshape(y1 - y0, N)
    M = np.maximum(I.astype(np.int16) - h, 0).astype(np.uint8)
    return M, I


def sr_check(J, M, I, max_iter: int = 200):
    """Independent device recomputation of the 8-conn reconstruction for the
    whole slide (checker only): starting from the marker, repeat {exact row
    sweeps, exact column sweeps (recon_sweeps.cu, not the tile engine), one
    clamped 3x3 dilation step (torch)} until nothing changes.  Each step only
    applies valid raises, and a state no step changes is a fixed point of the
    full 8-neighbourhood rule, so the result is THE reconstruction (unique
    fixed point, gridwave engine.py:9-18): recon_sr's algorithm.  Returns
    (J == result everywhere, iterations)."""
    import torch
    from paper_1209_3314_b200 import _lib
    L = _lib.lib()
    H, W = M.shape
    R = M.clone()
    ws = _lib.workspace(L.iwpp_recon_workspace_bytes(W, H, 0, 8))
    st = _lib.stream_ptr()
    for it in range(1, max_iter + 1):
        _lib.check(L.iwpp_recon_sweep_rows(_lib.ptr(R), _lib.ptr(I), W, H, 0, st))
        _lib.check(L.iwpp_recon_sweep_cols(_lib.ptr(R), _lib.ptr(I), W, H, 0, _lib.ptr(ws), st))
        changed = False
        for y0 in range(0, H, 2048):
            y1 = min(H, y0 + 2048)
            a, b = max(0, y0 - 1), min(H, y1 + 1)
            blk = torch.nn.functional.pad(R[a:b].to(torch.float16)[None, None], (1, 1, 1, 1),
                                          value=-1.0)
            d = torch.nn.functional.max_pool2d(blk, 3, 1)[0, 0][y0 - a:y0 - a + (y1 - y0)]
            nxt = torch.minimum(I[y0:y1].to(torch.float16), d).to(torch.uint8)
            nxt = torch.maximum(nxt, R[y0:y1])
            if not changed and bool((nxt != R[y0:y1]).any()):
                changed = True
            R[y0:y1] = nxt
        if not changed:
            # one more sweep pair must change nothing either (full fixed point)
            return bool(torch.equal(R, J)), it
    return False, max_iter


def edt_block_parity(vr_rows, dist_rows, mask_fn, y0_glob, N, blocks, halo=64):
    """EDT whole-slide check (checker only): the oracle on 4096^2 blocks of
    the slide padded by `halo` cells, interiors compared bit for bit (vr
    packed with the slide's width, dist bytes).  A cell's value after r rounds
    depends only on cells within r steps (two-phase rounds, K.403-433), and
    the nuclei slide converges in ~17 rounds, far below the halo."""
    import oracle
    ok = True
    for (by, bx) in blocks:
        ya, yb = max(by - halo, 0), min(by + 4096 + halo, N)
        xa, xb = max(bx - halo, 0), min(bx + 4096 + halo, N)
        m = mask_fn(ya, yb)[:, xa:xb]
        vr_b, d_b = oracle.edt(np.ascontiguousarray(m), 8)
        sy, sx = vr_b // (xb - xa), vr_b % (xb - xa)
        want_vr = (sy + ya) * N + (sx + xa)
        iy, ix = by - ya, bx - xa
        want_vr = want_vr[iy:iy + 4096, ix:ix + 4096]
        want_d = d_b[iy:iy + 4096, ix:ix + 4096]
        got_vr = vr_rows[by - y0_glob:by - y0_glob + 4096, bx:bx + 4096].cpu().numpy()
        got_d = dist_rows[by - y0_glob:by - y0_glob + 4096, bx:bx + 4096].cpu().numpy()
        ok = ok and bool(np.array_equal(got_vr, want_vr)) and got_d.tobytes() == want_d.tobytes()
    return ok


def whole_slide(dev, rank: int, world: int, flush, peak: float, check: bool = True):
    """BASELINE configs[4]: a 64K x 64K whole slide, reconstruction (u8,
    8-conn, the counter-hash random pair of slide_rows, identical for every
    N) and EDT (the 4K nuclei mask tiled 16 x 16), one GPU or horizontal
    slabs across the ranks (NCCL border exchange + all-reduce termination,
    distributed.py).  Strong scaling: the slide is fixed, ``ms`` is the max
    over ranks.  Parity: recon against an independent device recomputation
    (sr_check) on every rank's slab rows, EDT against the oracle on 4K blocks
    (edt_block_parity) of rank 0's rows."""
    import torch
    import torch.distributed as dist

    import oracle  # input generator + checker only
    import paper_1209_3314_b200 as gw
    from paper_1209_3314_b200 import distributed as D

    N = WS_PX
    y0, y1 = D.slab_bounds(N, world, rank)
    res = {}

    def timed(fn, reps=2, warm=1):
        for _ in range(warm):
            fn()
        ts = []
        for i in range(reps):
            flush.fill_(i & 0xff)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        if world > 1:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    def all_ok(ok):
        if ok is None or world == 1:
            return ok
        t = torch.tensor([0 if ok else 1], device=dev, dtype=torch.int32)
        dist.all_reduce(t)
        return int(t.item()) == 0

    def entry(ms, bpp, **kw):
        ach = bpp * N * N / (ms / 1e3) / 1e9
        return {"ms": round(ms, 3), "mpx_s": round(N * N / ms / 1e3, 1), "n_gpus": world,
                "roofline_frac": round(ach / (peak * world), 4), "alg_bytes_per_px": bpp, **kw}

    # reconstruction: the same slide for every N, each rank holding its rows
    M, I = slide_rows(y0, y1, N, dev)
    info = {}
    if world == 1:
        def run():
            info.pop("J", None)
            info["J"] = gw.reconstruct(M, I, 8)
        ms = timed(run)
        J = info.pop("J")
        ok, iters = sr_check(J, M, I) if check else (None, 0)
        del J
        res["recon_64k_u8_c8"] = entry(ms, ALG_BYTES_PER_PX, parity_vs_sr=ok, sr_iterations=iters)
    else:
        def run():
            slab = D.SlabRecon(M, I, rank > 0, rank + 1 < world, 8, D.device_solver)
            info["waves"] = D.run_slab_dist(slab).waves
            info["J"] = slab.result()
        ms = timed(run)
        ok = None
        if check:
            # N=G against N=1 bit for bit: every rank reconstructs the whole
            # slide on its own GPU (12 GiB) and compares its slab's rows
            Js = info.pop("J").clone()
            Mf, If = slide_rows(0, N, N, dev)
            ok = bool(torch.equal(gw.reconstruct(Mf, If, 8)[y0:y1], Js))
            del Mf, If, Js
        res["recon_64k_u8_c8"] = entry(ms, ALG_BYTES_PER_PX, waves=info["waves"],
                                       parallelism=f"slabs x{world}", parity_vs_sr=all_ok(ok))
    del I, M, info
    torch.cuda.empty_cache()

    # EDT: 4K nuclei mask tiled 16 x 16 (the rows of this rank + halo rows)
    m4 = oracle.gen_nuclei_mask(4096, 4096, 30.0, 7)
    m4d = torch.from_numpy(m4).to(dev)

    def mask_np(a, b):
        return np.tile(m4[np.arange(a, b) % 4096], (1, N // 4096))

    rows = torch.arange(max(y0 - 1, 0), min(y1 + 1, N), device=dev) % 4096
    mrows = m4d[rows].repeat(1, N // 4096)
    info = {}
    if world == 1:
        img = gw.Image2D(N, N, "binary", mrows)

        def run():
            info.pop("r", None)  # free the previous result (48 GiB) first
            cfg = gw.EngineConfig()
            info["r"] = gw.edt(img, gw.SE8, mode="parallel", cfg=cfg)
            info["rounds"] = cfg.stats.rounds
        ms = timed(run, reps=1)
        ok = None
        if check:
            vm, dist_img = info.pop("r")
            ok = edt_block_parity(vm.vr, dist_img.data, mask_np, 0, N,
                                  [(0, 0), (0, N - 4096), (N // 2, N // 2),
                                   (N - 4096, 0), (N - 4096, N - 4096)])
        res["edt_64k_nuclei_c8"] = entry(ms, 13, rounds=info["rounds"], parity_blocks_vs_oracle=ok)
    else:
        ext = torch.zeros((y1 - y0 + 2, N), dtype=torch.uint8, device=dev)
        top = 1 if y0 == 0 else 0  # no row above the image: ext row 0 stays zero
        ext[top:top + mrows.shape[0]] = mrows

        # device-resident rounds: one kernel per GPU, boundary items and
        # frontier counts through NVLink mailboxes (no host round trip per
        # round); the per-round NCCL loop is the fallback
        try:
            slab = D.DeviceSlabEDT(ext, y0, N, 8)
            info["protocol"] = "device-resident rounds (NVLink mailboxes, iwpp_edt_mg_run)"
        except Exception as e:  # noqa: BLE001 - no symmetric memory: host loop
            slab = None
            info["protocol"] = f"host loop per round (NCCL); device protocol unavailable: {type(e).__name__}"
        okt = torch.tensor([1 if slab is not None else 0], device=dev, dtype=torch.int64)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)  # every rank takes the same protocol
        if int(okt.item()) == 0 and slab is not None:
            slab = None
            info["protocol"] = "host loop per round (NCCL); device protocol unavailable on another rank"

        def run():
            info.pop("out", None)
            if slab is not None:
                info["rounds"] = slab.run()
                info["out"] = slab.finalize()
            else:
                hs = D.SlabEDT(ext, y0, N, rank > 0, rank + 1 < world, 8)
                info["rounds"] = D.run_edt_slab_dist(hs)
                info["out"] = hs.finalize()
        ms = timed(run, reps=1)
        ok = None
        if check and y1 - y0 >= 4096:
            vr_s, d_s = info.pop("out")
            by = y0 if rank == 0 else y0 + ((y1 - y0 - 4096) // 2)
            ok = edt_block_parity(vr_s, d_s, mask_np, y0, N, [(by, 0), (by, N // 2)])
        res["edt_64k_nuclei_c8"] = entry(ms, 13, rounds=info["rounds"],
                                         parallelism=f"slabs x{world}", protocol=info["protocol"],
                                         parity_blocks_vs_oracle=all_ok(ok))
    return res


def slide_headline(args, rank: int, world: int, local: int, dev):
    """The N > 1 headline: BASELINE configs[4], the 64K x 64K whole slide
    (the counter-hash random pair of slide_rows, identical for every N) as
    horizontal slabs, one per rank, reconstructed by the slab protocol --
    the tile engine on each slab, changed border rows to the neighbours
    over NCCL, waves until an all-reduce of the halo changes is 0 (north
    star; distributed.run_slab_dist).  Strong scaling: the slide is fixed.
    One step = restore the slab's marker rows + the protocol to the fixed
    point.  e2e: the same through host buffers -- H2D of the rank's marker
    and mask rows from pinned memory, the protocol, D2H of its result rows.
    Parity: every rank compares its rows with a single-GPU reconstruction of
    the whole slide on its own GPU."""
    import torch
    import torch.distributed as dist

    from paper_1209_3314_b200 import _lib
    from paper_1209_3314_b200 import distributed as D
    from paper_1209_3314_b200.build import LIB

    if not dist.is_initialized():  # (--slide-headline on, one GPU: a one-rank group)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    N = WS_PX
    y0, y1 = D.slab_bounds(N, world, rank)
    M, I = slide_rows(y0, y1, N, dev)
    info = {"waves": []}

    slab0 = D.SlabRecon(M, I, rank > 0, rank + 1 < world, 8, D.device_solver)

    def step():  # restore the marker rows (the mask rows stay), then the protocol
        slab0.reset(M)
        info["waves"].append(D.run_slab_dist(slab0).waves)
        return slab0

    def barrier():
        dist.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    info["waves"].clear()
    ts = []
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        for _ in range(args.steps):  # 8 GiB of inputs per slide: beyond L2 by itself
            s0.record()
            slab = step()
            s1.record()
            s1.synchronize()
            ts.append(s0.elapsed_time(s1))
    torch.cuda.synchronize()
    barrier()
    total = torch.tensor([sum(ts)], device=dev, dtype=torch.float64)
    dist.all_reduce(total, op=dist.ReduceOp.MAX)
    total_ms = float(total.item())
    value = args.steps * N * N / (total_ms / 1e3) / 1e6
    res = slab.result().clone()

    # e2e: pinned host rows in, protocol, result rows out
    hM = M.cpu().pin_memory()
    hI = I.cpu().pin_memory()
    hO = torch.empty_like(hM).pin_memory()
    dM, dI = torch.empty_like(M), torch.empty_like(I)

    def e2e_step():
        dM.copy_(hM, non_blocking=True)
        dI.copy_(hI, non_blocking=True)
        slab = D.SlabRecon(dM, dI, rank > 0, rank + 1 < world, 8, D.device_solver)
        D.run_slab_dist(slab)
        hO.copy_(slab.result(), non_blocking=True)
        torch.cuda.synchronize()

    e2e_step()
    barrier()
    te = []
    for _ in range(args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_step()
        te.append(time.perf_counter() - t0)
    barrier()
    et = torch.tensor([sum(te)], device=dev, dtype=torch.float64)
    dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_val = args.steps * N * N / float(et.item()) / 1e6
    e2e_ok = bool(torch.equal(hO.to(dev), res))

    # parity: the slab rows against a single-GPU run of the whole slide
    ok = None
    if not args.no_cpu:
        del hM, hI, hO, dM, dI
        torch.cuda.empty_cache()
        Mf, If = slide_rows(0, N, N, dev)
        import paper_1209_3314_b200 as gw
        ok = bool(torch.equal(gw.reconstruct(Mf, If, 8)[y0:y1], res)) and e2e_ok
        del Mf, If
        t = torch.tensor([0 if ok else 1], device=dev, dtype=torch.int32)
        dist.all_reduce(t)
        ok = int(t.item()) == 0
    peak, peak_kind = measured_peak_gbs()
    ms = total_ms / args.steps
    ach = ALG_BYTES_PER_PX * N * N / (ms / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "Mpx/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (counter-hash uniform mask, marker = max(mask-40, 0); the same slide for every N)",
        "config": {"workload": "recon_by_dilation 65536x65536 u8 whole slide, 8-connectivity, horizontal "
                               f"slabs x{world} with NCCL border exchange (BASELINE configs[4])",
                   "shape": [N, N], "conn": 8, "parallelism": f"slabs x{world}",
                   "waves_per_step": sorted(set(info["waves"])),
                   "l2": "inputs (8 GiB per slide) exceed L2; no flush needed"},
        "clocks": clk.summary(),
        "e2e": {"value": round(e2e_val, 2), "unit": "Mpx/s",
                "h2d_bytes_per_step": 2 * N * N, "d2h_bytes_per_step": N * N,
                "path": "pinned host slab rows -> SlabRecon / run_slab_dist -> host rows (per rank)"},
        # per step on this rank: the first wave's engine launch (queue built in
        # the kernel), then the queue-init + engine pair of every later wave
        "gpu_launches": int(sum(1 + 2 * (w - 1) for w in info["waves"])),
        "roofline": {"bound": "hbm", "achieved": round(ach, 2), "peak": round(peak * world, 1),
                     "unit": "GB/s", "frac": round(ach / (peak * world), 4), "traffic": None,
                     "kernel": "whole step (tile engine waves + exchange), all ranks",
                     "alg_bytes_per_px": ALG_BYTES_PER_PX,
                     "peak_kind": f"{peak_kind} x {world} GPUs"},
        "library": os.path.relpath(LIB, ROOT),
        "parity_vs_single_gpu": ok,
    }
    if not args.no_extras and not args.no_whole_slide:
        # the whole-slide block of the N = 1 line, at this N: recon (timed as
        # above, plus waves) and the EDT on the device-resident slab protocol
        del M, I, res, slab, slab0
        torch.cuda.empty_cache()
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        try:
            ws_line = whole_slide(dev, rank, world, flush, peak, check=not args.no_cpu)
        except Exception as e:  # the headline line must still print
            ws_line = {"whole_slide_error": f"{type(e).__name__}: {e}"[:300]}
        line["whole_slide"] = {"scaling": "strong", "n_gpus": world, **ws_line}
    if rank == 0:
        emit(line)
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
