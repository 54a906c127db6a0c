"""Where the torch copies of one eager bench step (PROBE_CONFIG, default the
cfg4 train step) come from: wraps
Tensor.copy_, torch.stack / cat, Tensor.clone / contiguous during one
training minibatch (no graph) and counts the calls on CUDA tensors by the
innermost package frame (non-contiguous ones launch a copy kernel)."""
import collections
import os
import sys
import traceback

os.environ["BENCH_GRAPH"] = "0"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

wl = bench.WORKLOADS[os.environ.get("PROBE_CONFIG", "train")]()
wl.setup(0, 1)
for _ in range(2):
    wl.step()
torch.cuda.synchronize()
where = collections.Counter()
nbytes = collections.Counter()
active = [False]


def site(depth=3):
    out = []
    for fr in reversed(traceback.extract_stack()[:-2]):
        if "paper_2210_02574_b200" in fr.filename or fr.filename.endswith("bench.py"):
            out.append(f"{os.path.basename(fr.filename)}:{fr.lineno} {fr.name}")
            if len(out) == depth:
                break
    return " <- ".join(out) or "(outside)"


def wrap(owner, name, kind):
    orig = getattr(owner, name)

    def f(*a, **k):
        out = orig(*a, **k)
        if active[0]:
            t = out if isinstance(out, torch.Tensor) else None
            if t is not None and t.is_cuda:
                src = a[1] if name == "copy_" and len(a) > 1 else (a[0] if a else None)
                nc = ""
                if name == "copy_" and isinstance(src, torch.Tensor):
                    nc = "" if (src.is_contiguous() and a[0].is_contiguous()) else " noncontig"
                key = f"{kind}{nc} @ {site()}"
                where[key] += 1
                nbytes[key] += t.numel() * t.element_size()
        return out

    setattr(owner, name, f)


_orig_to = torch.Tensor.to


def _to(self, *a, **k):
    out = _orig_to(self, *a, **k)
    if active[0] and out.is_cuda and not self.is_cuda:
        key = f"h2d to @ {site()}"
        where[key] += 1
        nbytes[key] += out.numel() * out.element_size()
    return out


torch.Tensor.to = _to
wrap(torch.Tensor, "copy_", "copy_")
wrap(torch.Tensor, "clone", "clone")
wrap(torch.Tensor, "contiguous", "contiguous")
wrap(torch, "stack", "stack")
wrap(torch, "cat", "cat")
active[0] = True
wl.step()
torch.cuda.synchronize()
active[0] = False
for key, c in where.most_common(40):
    print(f"{c:4d} {nbytes[key] / 2**20:9.1f} MiB  {key}")
