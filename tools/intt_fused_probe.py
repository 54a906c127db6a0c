"""Inverse NTT of 10 polys x 22 limbs at N=2^16: output digest and CUDA-event
time.  Run once with HEGPU_INTT_FUSED=1 and once without (the switch is read
once per process): equal digests = bit-identical limbs."""
import hashlib
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_02574_b200 import _dev, _lib, ckks  # noqa: E402
from tools.microbench import rand_limbs  # noqa: E402

preset = os.environ.get("PROBE_PRESET", "p16")
params = ckks.get_preset(preset)
n = params.ring_degree
k = int(os.environ.get("PROBE_LIMBS", "22"))
polys = int(os.environ.get("PROBE_POLYS", "10"))
torch.manual_seed(5)
ring = params.ring.device()
x = rand_limbs(params, (polys, k, n), k)
y = torch.empty_like(x)
sel = np.arange(k, dtype=np.int32)


def run():
    _lib.call("hegpu_ntt", ring, 1, x.data_ptr(), k * n, y.data_ptr(), k * n, polys, k,
              sel.ctypes.data, _dev.stream())


run()
torch.cuda.synchronize()
digest = hashlib.sha256(y.cpu().numpy().tobytes()).hexdigest()[:16]
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 50
a.record()
for _ in range(reps):
    run()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
gbs = 2 * x.numel() * 8 / (ms * 1e-3) / 1e9
print(json.dumps({"fused": os.environ.get("HEGPU_INTT_FUSED", "0"), "preset": preset,
                  "digest": digest, "ms": round(ms, 4), "GB_s_rw": round(gbs, 1)}))
