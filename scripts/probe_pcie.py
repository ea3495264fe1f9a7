"""Development probe: host<->device copy rates from pinned memory (the floor
under the e2e number)."""
import time
import torch

torch.cuda.set_device(0)
for mb in (4, 16, 32, 64):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    def t(fn, reps=10):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
        return min(ts) * 1e3
    h2d = t(lambda: d.copy_(h, non_blocking=True))
    d2h = t(lambda: h.copy_(d, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    bi = t(both)
    print(f"{mb} MB: H2D {h2d:.3f} ms ({n/h2d/1e6:.1f} GB/s)  D2H {d2h:.3f} ms ({n/d2h/1e6:.1f} GB/s)  "
          f"both {bi:.3f} ms", flush=True)
