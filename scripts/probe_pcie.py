"""Host<->device copy bandwidth on this box (pinned buffers): H2D alone, D2H
alone, and both at once on two streams -- the floor under the e2e number.
python scripts/probe_pcie.py"""
import torch

MB = 1 << 20
h_in = torch.empty(32 * MB, dtype=torch.uint8).pin_memory()
h_out = torch.empty(16 * MB, dtype=torch.uint8).pin_memory()
d_in = torch.empty(32 * MB, dtype=torch.uint8, device="cuda")
d_out = torch.empty(16 * MB, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=20):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def h2d():
    d_in.copy_(h_in, non_blocking=True)


def d2h():
    h_out.copy_(d_out, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(f"H2D 32 MB: {t1:.3f} ms ({32 * MB / t1 / 1e6:.1f} GB/s)")
print(f"D2H 16 MB: {t2:.3f} ms ({16 * MB / t2 / 1e6:.1f} GB/s)")
print(f"both at once: {t3:.3f} ms ({48 * MB / t3 / 1e6:.1f} GB/s total)")
for sz in (1, 2, 4, 8):
    hv, dv = h_in[: sz * MB], d_in[: sz * MB]
    t = timed(lambda: dv.copy_(hv, non_blocking=True))
    print(f"H2D {sz} MB: {t * 1e3:.1f} us ({sz * MB / t / 1e6:.1f} GB/s)")
