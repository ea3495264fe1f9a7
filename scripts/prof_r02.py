"""One workload per kernel family, run once after a warm-up, for ncu
captures (scripts/prof_r02.sh drives ncu over the cases):

  python scripts/prof_r02.py CASE

CASE: recon_u8_4k | recon_i32_4k | recon_u8_64k | imfill_16k | stages_16k |
      edt_blob4k | edt_nuclei4k | edt_mg_blob4k | edt_nuclei64k
Inputs are the bench's (reference generator / counter-hash slide / the 4K
nuclei and blob masks)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import oracle
import paper_1209_3314_b200 as gw
from bench import gray_pair, slide_rows
from paper_1209_3314_b200 import _lib

case = sys.argv[1]
L = _lib.lib()
dev = torch.device("cuda")


def twice(fn):
    fn()  # warm-up (ncu -s skips its launches)
    torch.cuda.synchronize()
    fn()
    torch.cuda.synchronize()


if case in ("recon_u8_4k", "recon_i32_4k", "recon_u8_64k"):
    if case == "recon_u8_4k":
        J, I = (torch.from_numpy(a).to(dev) for a in gray_pair(4096, 0))
    elif case == "recon_i32_4k":
        J, I = (torch.from_numpy(a).to(dev) for a in oracle.gray_pair(4096, 0, h=1 << 28, dtype=np.int32))
    else:
        J, I = slide_rows(0, 65536, 65536, dev)
    twice(lambda: gw.reconstruct(J, I, 8))
elif case == "imfill_16k":
    bw = np.tile(oracle.gen_synthetic_mask(4096, 4096, 50, 7), (4, 4))
    J, I = (torch.from_numpy(a).to(dev) for a in oracle.imfill_pair(bw))
    twice(lambda: gw.reconstruct(J, I, 8, kind="binary"))
elif case == "stages_16k":
    from paper_1209_3314_b200.recon import seed_scan
    J, I = (torch.from_numpy(a).to(dev) for a in gray_pair(16384, 0))
    ws = _lib.workspace(L.iwpp_recon_workspace_bytes(16384, 16384, 0, 8))

    def run():
        Jc = J.clone()
        _lib.check(L.iwpp_recon_sweep_rows(_lib.ptr(Jc), _lib.ptr(I), 16384, 16384, 0, _lib.stream_ptr()))
        _lib.check(L.iwpp_recon_sweep_cols(_lib.ptr(Jc), _lib.ptr(I), 16384, 16384, 0, _lib.ptr(ws),
                                           _lib.stream_ptr()))
        seed_scan(Jc, I, 8)
        n = _lib.ctypes.c_int64(0)
        _lib.check(L.iwpp_check_le(_lib.ptr(Jc), _lib.ptr(I), 16384 * 16384, 0, _lib.ptr(ws),
                                   _lib.ctypes.byref(n), _lib.stream_ptr()))
    twice(run)
elif case in ("edt_blob4k", "edt_nuclei4k"):
    m = oracle.gen_synthetic_mask(4096, 4096, 50, 7) if case == "edt_blob4k" \
        else oracle.gen_nuclei_mask(4096, 4096, 30.0, 7)
    img = gw.Image2D(4096, 4096, "binary", torch.from_numpy(m).to(dev))
    twice(lambda: gw.edt(img, gw.SE8))
elif case == "edt_mg_blob4k":
    from paper_1209_3314_b200.distributed import edt_slabs_local_device
    m = torch.from_numpy(oracle.gen_synthetic_mask(4096, 4096, 50, 7)).to(dev)
    twice(lambda: edt_slabs_local_device(m, 4, 8))
elif case == "edt_nuclei64k":
    m4 = torch.from_numpy(oracle.gen_nuclei_mask(4096, 4096, 30.0, 7)).to(dev)
    img = gw.Image2D(65536, 65536, "binary", m4.repeat(16, 16))
    twice(lambda: gw.edt(img, gw.SE8))
else:
    raise SystemExit(f"unknown case {case}")
print("done", case)
