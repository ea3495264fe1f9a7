import sys; sys.path.insert(0, ".")
import torch, oracle, paper_1209_3314_b200 as gw
from paper_1209_3314_b200 import _lib
L = _lib.lib(); L.iwpp_edt_set_engine(4)
m = oracle.gen_synthetic_mask(4096, 4096, 50, 7)
img = gw.Image2D(4096, 4096, "binary", torch.from_numpy(m).cuda())
for _ in range(2):
    gw.edt(img, gw.SE8); torch.cuda.synchronize()
