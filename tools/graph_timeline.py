"""Device timeline of the captured cfg4 step (PROBE_CONFIG, default train):
sums kernel, memcpy and memset time inside graph replays with torch.profiler
(CUPTI) and compares it with the replay's wall time, i.e. how much of a step
is gaps between nodes."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

wl = bench.WORKLOADS[os.environ.get("PROBE_CONFIG", "train")]()
wl.setup(0, 1)
for _ in range(3):
    wl.step()
torch.cuda.synchronize()
reps = 3
acts = [torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]
with torch.profiler.profile(activities=acts) as prof:
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        wl.step()
    b.record()
    torch.cuda.synchronize()
wall = a.elapsed_time(b) / reps
kinds = collections.Counter()
counts = collections.Counter()
spans = []
for ev in prof.events():
    if ev.device_type != torch.autograd.DeviceType.CUDA:
        continue
    name = ev.name
    kind = ("memcpy" if "emcpy" in name else "memset" if "emset" in name else "kernel")
    dur = ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
    kinds[kind] += dur / 1000.0 / reps
    counts[kind] += 1
    if kind != "kernel":
        spans.append((dur, name))
print(f"step wall (events) {wall:.2f} ms; per step: " +
      ", ".join(f"{k} {v:.2f} ms ({counts[k] // reps} ops)" for k, v in kinds.items()))
for dur, name in sorted(spans, reverse=True)[:8]:
    print(f"  {dur / 1000:.3f} ms {name}")
