"""CPU restatement of one rank's EDT slab round (test infrastructure only).

It follows the device slab engine's contract (csrc/edt_slab.cu) with
numpy arrays, so ``distributed.run_edt_slab_dist`` -- the round loop,
boundary-row exchange and all-reduce termination -- can run over a gloo
group on CPU.  The rules are the reference's synchronous two-phase round
(gridwave _kernels.py K.403-433, the wave-start snapshot of the tiled
variant K.493-522 / tiles.py:305-331):

  * keys are (d2 << 32) | (sy << 16 | sx) in GLOBAL coordinates, all-ones
    = no source; the plain unsigned order is the reference's closer_source
    order (K.320-336);
  * every frontier cell of the round -- the rank's own, plus the
    neighbours' boundary frontier items of the adjacent rows, which carry
    their round-start sources -- offers make_key(q, src) to each in-slab
    neighbour q; q keeps the minimum; the next frontier is the set of cells
    whose key dropped;
  * after the round, the changed cells of the first / last row are the
    boundary items sent up / down (source or all-ones per column).
"""

from __future__ import annotations

import numpy as np
import torch

KINF = np.uint64(0xFFFFFFFFFFFFFFFF)
OFFS = {4: [(0, -1), (-1, 0), (1, 0), (0, 1)],
        8: [(-1, -1), (0, -1), (1, -1), (-1, 0), (1, 0), (-1, 1), (0, 1), (1, 1)]}


def _keys_from(src: np.ndarray, gy: np.ndarray, gx: np.ndarray):
    """make_key(q, src) for arrays (src all-ones -> all-ones)."""
    valid = src != KINF
    s = np.where(valid, src, 0).astype(np.uint64)
    sy = (s >> np.uint64(16)) & np.uint64(0xFFFF)
    sx = s & np.uint64(0xFFFF)
    dy = gy.astype(np.int64) - sy.astype(np.int64)
    dx = gx.astype(np.int64) - sx.astype(np.int64)
    d2 = (dx * dx + dy * dy).astype(np.uint64)
    return np.where(valid, (d2 << np.uint64(32)) | s, KINF)


class CpuSlabEDT:
    """Same interface as distributed.SlabEDT, on the CPU."""

    device = torch.device("cpu")

    def __init__(self, mask_ext, y0: int, H: int, has_up: bool, has_down: bool, conn: int):
        m = np.asarray(mask_ext.numpy() if hasattr(mask_ext, "numpy") else mask_ext)
        self.h, self.W = m.shape[0] - 2, m.shape[1]
        self.y0, self.H, self.conn = y0, H, conn
        self.has_up, self.has_down = has_up, has_down
        self.rounds = 0
        h, W = self.h, self.W
        gy = (y0 + np.arange(h))[:, None] * np.ones((1, W), np.int64)
        gx = np.ones((h, 1), np.int64) * np.arange(W)[None, :]
        self.gy, self.gx = gy, gx
        bg = m[1:h + 1] == 0
        own = ((gy.astype(np.uint64) << np.uint64(16)) | gx.astype(np.uint64))
        self.keys = np.where(bg, own, KINF).astype(np.uint64)
        # contour seeds: background cells with a foreground neighbour on the
        # image (the neighbours' halo rows count only where they exist)
        fg_ext = m != 0
        if not has_up:
            fg_ext[0] = False
        if not has_down:
            fg_ext[-1] = False
        P = np.pad(fg_ext, ((0, 0), (1, 1)))
        near = np.zeros((h, W), bool)
        for dx, dy in OFFS[conn]:
            near |= P[1 + dy:1 + dy + h, 1 + dx:1 + dx + W]
        self.front = bg & near
        self._emit()

    def _emit(self):
        up = np.where(self.front[0], self.keys[0] & np.uint64(0xFFFFFFFF), KINF)
        dn = np.where(self.front[-1], self.keys[-1] & np.uint64(0xFFFFFFFF), KINF)
        self.out = (torch.from_numpy(up.view(np.int64).copy()), torch.from_numpy(dn.view(np.int64).copy()))

    def boundary_rows(self):
        return self.out

    def round(self, halo_up, halo_dn) -> int:
        h, W = self.h, self.W
        src = np.full((h + 2, W), KINF, np.uint64)
        src[1:h + 1] = np.where(self.front, self.keys & np.uint64(0xFFFFFFFF), KINF)
        if halo_up is not None:
            src[0] = halo_up.numpy().view(np.uint64)
        if halo_dn is not None:
            src[h + 1] = halo_dn.numpy().view(np.uint64)
        S = np.pad(src, ((0, 0), (1, 1)), constant_values=KINF)
        new = self.keys.copy()
        for dx, dy in OFFS[self.conn]:
            # the item at q - (dx, dy) offers to q
            sv = S[1 - dy:1 - dy + h, 1 - dx:1 - dx + W]
            new = np.minimum(new, _keys_from(sv, self.gy, self.gx))
        self.front = new < self.keys
        self.keys = new
        self.rounds += 1
        self._emit()
        return int(self.front.sum())

    def finalize(self):
        k = self.keys
        inf = k == KINF
        s = np.where(inf, 0, k & np.uint64(0xFFFFFFFF))
        vr = np.where(inf, -1, ((s >> np.uint64(16)).astype(np.int64) * self.W
                                + (s & np.uint64(0xFFFF)).astype(np.int64)))
        d2 = (k >> np.uint64(32)).astype(np.float64)
        dist = np.where(inf, 0.0, np.sqrt(d2)).astype(np.float32)
        if inf.any():
            from paper_1209_3314_b200.errors import NoBackgroundError
            raise NoBackgroundError("no background reachable: distance map undefined")
        return torch.from_numpy(vr), torch.from_numpy(dist)
