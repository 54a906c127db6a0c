"""TEST INFRASTRUCTURE ONLY -- CPU baseline of bench.py from the oracle.

The reference runs the hot path one operation at a time on the host
(hebert: numba kernels per op, host numpy FFT per encode).  A full
N=2^16 training minibatch takes ~20 minutes on 8 cores, far
beyond the bench's time budget, so the baseline times a BOUNDED SAMPLE of the
same operations with the oracle (C/OpenMP kernels on all host cores):

  * key switch at a spread of levels (linearly interpolated in between),
  * encode (host FFT + NTT) at two levels,
  * rescale of one polynomial at two levels,
  * plaintext multiply (2 polys) at two levels,

and weights them by the op histogram of the workload (how many times the
reference algorithm runs each op at each level; recorded from an
instrumented run of the engine, see paper_2210_02574_b200/_stats.py).
The modelled time omits the reference's additions, permutations and Python
overhead, so it UNDER-estimates the reference's CPU time (conservative).
"""

import os
import time

import numpy as np

from . import scheme as S


class OracleCostModel:
    def __init__(self, preset_text, seed=7):
        self.p = S.Params.from_text(preset_text)
        t0 = time.perf_counter()
        self.keys = S.keygen(self.p, [], seed, conj=False)
        self.keygen_s = time.perf_counter() - t0
        self.t = {}

    def _rand(self, level, seed):
        rng = np.random.default_rng(seed)
        return np.stack([rng.integers(0, q, size=self.p.n, dtype=np.uint64)
                         for q in self.p.chain[: level + 1]])

    def _time(self, fn, reps=1):
        best = float("inf")
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            best = min(best, time.perf_counter() - t0)
        return best

    def sample(self, ks_levels, other_levels):
        p = self.p
        top = len(p.chain) - 1  # a histogram recorded on a deeper chain: clamp its levels
        ks_levels = [min(int(lvl), top) for lvl in ks_levels]
        other_levels = [min(int(lvl), top) for lvl in other_levels]
        for lvl in sorted(set(ks_levels)):
            d = self._rand(lvl, 100 + lvl)
            self.t[("ks", lvl)] = self._time(lambda: S.ks_apply(p, self.keys.relin, d, lvl))
        vals = np.random.default_rng(5).uniform(-1, 1, p.slots)
        for lvl in sorted(set(other_levels)):
            self.t[("encode", lvl)] = self._time(lambda: S.encode(p, vals, lvl, p.scale))
            a = self._rand(lvl, 200 + lvl)
            if lvl > 0:
                self.t[("rescale_poly", lvl)] = self._time(lambda: S._rescale_poly(p, a, lvl))
            primes = p.chain[: lvl + 1]
            self.t[("ptmul", lvl)] = self._time(
                lambda: (S.mul(p, a, a, primes), S.mul(p, a, a, primes)))
        return self.t

    def _interp(self, op, lvl):
        pts = sorted(l for (o, l) in self.t if o == op)
        if not pts:
            return 0.0
        if lvl in pts:
            return self.t[(op, lvl)]
        lo = max([l for l in pts if l < lvl], default=pts[0])
        hi = min([l for l in pts if l > lvl], default=pts[-1])
        if lo == hi:
            return self.t[(op, lo)] * (lvl + 1) / (lo + 1)
        f = (lvl - lo) / (hi - lo)
        return self.t[(op, lo)] * (1 - f) + self.t[(op, hi)] * f

    def seconds(self, histogram):
        """Modelled reference seconds for an op histogram {"op@level": count}."""
        total = 0.0
        top = len(self.p.chain) - 1
        for key, count in histogram.items():
            op, lvl = key.split("@")
            total += count * self._interp(op, min(int(lvl), top))
        return total


def histogram_levels(histogram):
    ks = sorted({int(k.split("@")[1]) for k in histogram if k.startswith("ks@")})
    other = sorted({int(k.split("@")[1]) for k in histogram if not k.startswith("ks@")})
    # a bounded spread: at most 6 KS levels, 2 levels for the cheap ops
    if len(ks) > 6:
        idx = np.linspace(0, len(ks) - 1, 6).round().astype(int)
        ks = sorted({ks[i] for i in idx})
    if len(other) > 2:
        other = [other[0], other[-1]]
    return ks, other


def load_histogram(name):
    import json

    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                        "profiles", f"op_histogram_{name}.json")
    with open(path) as fh:
        return json.load(fh)
