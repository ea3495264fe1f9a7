"""Small workloads through every kernel family, for compute-sanitizer:

  compute-sanitizer --tool memcheck  python scripts/sanitize.py
  compute-sanitizer --tool racecheck python scripts/sanitize.py
  compute-sanitizer --tool synccheck python scripts/sanitize.py

Each case is also checked against the CPU oracle (test infrastructure), so a
run under a sanitizer is a parity run too.  Prints one line per case."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_1209_3314_b200 as gw
from paper_1209_3314_b200 import _lib

L = _lib.lib()
bad = []


def check(name, ok):
    print(f"{name}: {'ok' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        bad.append(name)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


rng = np.random.default_rng(5)
# reconstruction: u8 (register engine, non-fused and fused/cooperative), 4/8-conn
for shape in ((96, 160), (512, 512)):
    J, I = oracle.gray_pair(shape, 1, h=40)
    for conn in (4, 8):
        got = gw.reconstruct(dev(J), dev(I), conn).cpu().numpy()
        check(f"recon u8 {shape} c{conn}", np.array_equal(got, oracle.recon_fh(J, I, conn)))
# 16/32-bit register engine, f32 through the ordered-int path
for dt, h in ((np.uint16, 9000), (np.int32, 1 << 27)):
    J, I = oracle.gray_pair((200, 256), 2, h=h, dtype=dt)
    got = gw.reconstruct(dev(J), dev(I), 8).cpu().numpy()
    check(f"recon {np.dtype(dt).name} c8", np.array_equal(got, oracle.recon_fh(J, I, 8)))
If = rng.standard_normal((128, 192)).astype(np.float32)
Jf = (If - 0.7).astype(np.float32)
got = gw.reconstruct(dev(Jf), dev(If), 8).cpu().numpy()
check("recon f32 c8", np.array_equal(got, oracle.recon_fh(Jf, If, 8)))
# binary (bit-plane engine) and the shared-memory engine with a tiny queue (overflow path)
bw = oracle.gen_synthetic_mask(256, 256, 50, 7)
Jb, Ib = oracle.imfill_pair(bw)
got = gw.reconstruct(dev(Jb), dev(Ib), 8, kind="binary").cpu().numpy()
check("imfill binary c8", np.array_equal(got, oracle.recon_fh(Jb, Ib, 8)))
J, I = oracle.gray_pair((128, 128), 3, h=40)
got = gw.reconstruct(dev(J), dev(I), 8, cfg=gw.EngineConfig(n_workers=2, queue=gw.QueueConfig(gbq_capacity=16))
                     ).cpu().numpy()
check("recon smem engine, forced overflow", np.array_equal(got, oracle.recon_fh(J, I, 8)))
# host pipeline (slabs, copy streams, dirty-row recopy)
J, I = oracle.gray_pair((1024, 512), 4, h=40)
got = gw.reconstruct(J, I, 8, pipeline_rows=128)
check("recon host pipeline", np.array_equal(got, oracle.recon_fh(J, I, 8)))
# host pipeline into a page-locked output (the mapped last transfer)
J, I = oracle.gray_pair((1024, 512), 8, h=40)
pm, pi = torch.from_numpy(J).pin_memory(), torch.from_numpy(I).pin_memory()
po = torch.empty_like(pm).pin_memory()
wsh = _lib.workspace(L.iwpp_recon_host_workspace_bytes(512, 1024, 0, 8))
o = gw.recon._opts(None, pipeline_rows=128)
_lib.check(L.iwpp_recon_host(_lib.ptr(po.numpy()), _lib.ptr(pm.numpy()), _lib.ptr(pi.numpy()), 512, 1024, 0, 8,
                             _lib.ptr(wsh), wsh.numel(), _lib.ctypes.byref(o), None, _lib.stream_ptr()))
check("recon host pipeline, pinned output", np.array_equal(po.numpy(), oracle.recon_fh(J, I, 8)))
# stage kernels: sweeps, seed scan, passes
from paper_1209_3314_b200.recon import seed_scan  # noqa: E402
J, I = oracle.gray_pair((160, 200), 6, h=40)
Jd = dev(J)
ws = _lib.workspace(L.iwpp_recon_workspace_bytes(200, 160, 0, 8))
_lib.check(L.iwpp_recon_sweep_rows(_lib.ptr(Jd), _lib.ptr(dev(I)), 200, 160, 0, _lib.stream_ptr()))
seeds = seed_scan(Jd, dev(I), 8)
check("sweeps + seed scan run", seeds.numel() >= 0)
# EDT: raster (default), queue, blocked, CAS engines; propagate; multi-slab protocol
m = oracle.gen_synthetic_mask(200, 160, 50, 7)
vr_ref, d_ref = oracle.edt(m, 8)
img = gw.Image2D(m.shape[1], m.shape[0], "binary", dev(m))
for mode in (0, 3, 4, 1):
    _lib.check(L.iwpp_edt_set_engine(mode), "set_engine")
    vm, dist = gw.edt(img, gw.SE8)
    check(f"edt engine {mode}", np.array_equal(vm.vr.cpu().numpy(), vr_ref)
          and dist.data.cpu().numpy().tobytes() == d_ref.tobytes())
_lib.check(L.iwpp_edt_set_engine(0), "set_engine")
# the 4-cells-per-lane init (W % 128 == 0), both connectivities
m2 = oracle.gen_synthetic_mask(256, 96, 50, 7)
for conn in (4, 8):
    vr2, d2 = oracle.edt(m2, conn)
    vm, dist = gw.edt(gw.Image2D(m2.shape[1], m2.shape[0], "binary", dev(m2)), gw.StructuringElement(conn))
    check(f"edt init4 c{conn}", np.array_equal(vm.vr.cpu().numpy(), vr2) and dist.data.cpu().numpy().tobytes() == d2.tobytes())
from paper_1209_3314_b200.distributed import edt_slabs_local_device  # noqa: E402
vr, d, _ = edt_slabs_local_device(m, 3, 8)
check("edt multi-slab device protocol (3 slabs)", np.array_equal(vr, vr_ref) and d.tobytes() == d_ref.tobytes())
# image I/O decode / encode on the device
import tempfile  # noqa: E402
from paper_1209_3314_b200.imgio import read_pgm, write_pgm  # noqa: E402
with tempfile.TemporaryDirectory() as tdir:
    p = os.path.join(tdir, "a.pgm")
    write_pgm(gw.Image2D(64, 48, "u8", dev(rng.integers(0, 256, (48, 64)).astype(np.uint8))), p)
    back = read_pgm(p, device="cuda")
    check("pgm round trip", back.width == 64 and back.height == 48)
torch.cuda.synchronize()
print("BAD", bad)
sys.exit(1 if bad else 0)
