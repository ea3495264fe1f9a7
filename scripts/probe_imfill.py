"""imfill 16K^2 timing (the bench's C4 rows) for A/B:
python scripts/probe_imfill.py.  Two forms of the same call through the C
ABI: the marker copied by torch into the output first ("copy"), and the
marker handed over in iwpp_recon_opts.marker ("marker", what reconstruct()
does).  IWPP_B200_LIB selects another build (an older build ignores
opts.marker, so only its "copy" line is meaningful)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
from paper_1209_3314_b200 import _lib
from paper_1209_3314_b200.recon import _opts

L = _lib.lib()
bw = np.tile(oracle.gen_synthetic_mask(4096, 4096, 50, 7), (4, 4))
J, I = (torch.from_numpy(a).cuda() for a in oracle.imfill_pair(bw))
H, W = J.shape
out = torch.empty_like(J)
for conn in (4, 8):
    ws = _lib.workspace(L.iwpp_recon_workspace_bytes(W, H, 4, conn))
    for form in ("copy", "marker"):
        o = _opts(None)
        ts = []
        for r in range(7):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            if form == "copy":
                out.copy_(J)
            else:
                o.marker = _lib.ptr(J)
            _lib.check(L.iwpp_recon(_lib.ptr(out), _lib.ptr(I), W, H, 4, conn, _lib.ptr(ws), ws.numel(),
                                    _lib.ctypes.byref(o), None, _lib.stream_ptr()), "recon")
            b.record()
            torch.cuda.synchronize()
            if r >= 2:
                ts.append(a.elapsed_time(b))
        cnt = (_lib.ctypes.c_uint64 * 16)()
        L.iwpp_recon_engine_counters(_lib.ptr(ws), W, H, cnt, 16, _lib.stream_ptr())
        ntiles = ((W + 127) // 128) * ((H + 127) // 128)  # the binary engine's 128 x 128 tiles
        print(f"imfill 16K c{conn} {form}: {np.median(ts):.3f} ms (min {min(ts):.3f}); activations {cnt[0]} "
              f"({cnt[0] / ntiles:.2f}/tile) reruns {cnt[1]} steps/act {cnt[6] / max(cnt[0], 1):.2f}", flush=True)
        if cnt[8] or cnt[13]:  # -DIWPP_PHASES build: cycles per activation (lane 0)
            na = max(cnt[0], 1)
            print("   phases (cycles/activation): pop %.0f load %.0f fix %.0f publish %.0f"
                  % (cnt[8] / na, cnt[9] / na, cnt[10] / na, cnt[13] / na), flush=True)
