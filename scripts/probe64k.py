"""Development probe: whole-slide (64K x 64K by default) recon / imfill / EDT
on one B200.  Inputs are generated on the device (recon) or tiled from the
4K generators (imfill, EDT).  Prints timings and size-independent property
checks (fixed-point equation for recon, local stability for EDT)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1209_3314_b200 as gw

N = int(os.environ.get("PROBE_N", 65536))
which = sys.argv[1:] or ["recon", "imfill", "edt"]


def timeit(fn, reps=3, warm=1):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)), float(min(ts))


def fixed_point_ok(J, I, M, conn):
    """J <= I, J >= marker, and J = min(I, max(J, dilate(J))) everywhere."""
    if not bool((J <= I).all()) or not bool((J >= M).all()):
        return False
    H, W = J.shape
    rows = 4096
    for y0 in range(0, H, rows):
        y1 = min(H, y0 + rows)
        a, b = max(0, y0 - 1), min(H, y1 + 1)
        blk = J[a:b].to(torch.int16)
        pad = torch.nn.functional.pad(blk[None, None].float(), (1, 1, 1, 1), value=-1.0)[0, 0]
        if conn == 8:
            d = torch.nn.functional.max_pool2d(pad[None, None], 3, 1)[0, 0]
        else:
            c = pad[1:-1, 1:-1]
            d = torch.maximum(torch.maximum(pad[:-2, 1:-1], pad[2:, 1:-1]),
                              torch.maximum(pad[1:-1, :-2], pad[1:-1, 2:]))
            d = torch.maximum(d, c)
        d = d[(y0 - a):(y0 - a) + (y1 - y0)]
        want = torch.minimum(I[y0:y1].float(), d)
        if not bool((want == J[y0:y1].float()).all()):
            return False
    return True


if "recon" in which:
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    I = torch.randint(0, 256, (N, N), dtype=torch.uint8, device="cuda", generator=g)
    M = torch.clamp(I.to(torch.int16) - 40, min=0).to(torch.uint8)
    for conn in (8, 4):
        st = {}
        J = gw.reconstruct(M, I, conn, stats=st)
        ok = fixed_point_ok(J, I, M, conn)
        del J
        med, mn = timeit(lambda: gw.reconstruct(M, I, conn))
        print(f"recon u8 {N}^2 c{conn}: median {med:.2f} ms min {mn:.2f}  {N*N/med/1e3:.0f} Mpx/s "
              f"alg {3*N*N/med/1e6:.0f} GB/s fixed_point={ok} stats={st}", flush=True)
    del I, M
    torch.cuda.empty_cache()

if "imfill" in which:
    import oracle
    bw = oracle.gen_synthetic_mask(4096, 4096, 50, 7)
    rep = N // 4096
    bwt = torch.from_numpy(bw).cuda().repeat(rep, rep)
    mask = torch.where(bwt == 0, 255, 0).to(torch.uint8)
    del bwt
    marker = torch.zeros_like(mask)
    marker[0, :] = mask[0, :]
    marker[-1, :] = mask[-1, :]
    marker[:, 0] = mask[:, 0]
    marker[:, -1] = mask[:, -1]
    for conn in (4, 8):
        st = {}
        J = gw.reconstruct(marker, mask, conn, stats=st)
        ok = fixed_point_ok(J, mask, marker, conn)
        del J
        med, mn = timeit(lambda: gw.reconstruct(marker, mask, conn))
        print(f"imfill {N}^2 c{conn}: median {med:.2f} ms  {N*N/med/1e3:.0f} Mpx/s fixed_point={ok} stats={st}",
              flush=True)
    del mask, marker
    torch.cuda.empty_cache()

if "edt" in which:
    import oracle
    t0 = time.time()
    m4 = oracle.gen_nuclei_mask(4096, 4096, 30.0, 7)
    rep = N // 4096
    m = torch.from_numpy(m4).cuda().repeat(rep, rep)
    img = gw.Image2D(N, N, "binary", m)
    cfg = gw.EngineConfig()
    vm, dist = gw.edt(img, gw.SE8, mode="parallel", cfg=cfg)
    del vm, dist
    torch.cuda.empty_cache()
    med, mn = timeit(lambda: gw.edt(img, gw.SE8), reps=3, warm=1)
    print(f"edt nuclei {N}^2 c8: median {med:.2f} ms  {N*N/med/1e3:.0f} Mpx/s "
          f"alg {13*N*N/med/1e6:.0f} GB/s rounds={cfg.stats.rounds} visits={cfg.stats.queued_total}",
          flush=True)
