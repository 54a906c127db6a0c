"""One forward + one inverse NTT of 10 polys x 22 limbs at P16 (for ncu captures)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_02574_b200 import _dev, _lib, ckks  # noqa: E402
from tools.microbench import rand_limbs  # noqa: E402

params = ckks.get_preset("p16")
n, k, polys = params.ring_degree, 22, 10
ring = params.ring.device()
x = rand_limbs(params, (polys, k, n), k)
sel = np.arange(k, dtype=np.int32)
for inv in (0, 1):
    _lib.call("hegpu_ntt", ring, inv, x.data_ptr(), k * n, x.data_ptr(), k * n, polys, k,
              sel.ctypes.data, _dev.stream())
torch.cuda.synchronize()
print("ok")
