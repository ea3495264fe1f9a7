"""One pipelined host-path reconstruction (4096^2 u8 c8) for an ncu launch list."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import oracle
from paper_1209_3314_b200 import _lib

L = _lib.lib()
torch.cuda.set_device(0)
n = 4096
J, I = oracle.gray_pair(n, 0, h=40)
pJ, pI = torch.from_numpy(J).pin_memory(), torch.from_numpy(I).pin_memory()
pO = torch.empty_like(pJ).pin_memory()
ws = _lib.workspace(L.iwpp_recon_host_workspace_bytes(n, n, 0, 8))
o = _lib.ReconOpts()
o.sweeps, o.tile_sweeps, o.halo_sweep_threshold = -1, -1, -1
for _ in range(int(os.environ.get("REPS", "2"))):
    _lib.check(L.iwpp_recon_host(_lib.ptr(pO.numpy()), _lib.ptr(pJ.numpy()), _lib.ptr(pI.numpy()),
                                 n, n, 0, 8, _lib.ptr(ws), ws.numel(), _lib.ctypes.byref(o), None,
                                 _lib.stream_ptr()), "recon_host")
torch.cuda.synchronize()
