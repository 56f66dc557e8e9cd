"""Timeline of one pipelined mf_apply_host call (torch.profiler / CUPTI): copy and kernel
start / end times relative to the first copy."""
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_1910_13247_b200 import Operator  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
nc, k, geom, coeff, _ = CONFIGS[cfg]
op = Operator(nc, k, geometry=geom, coeff=coeff)
n = op.n_local
hs = torch.from_numpy(synth.vector(n, 0)).pin_memory()
hd = torch.empty_like(hs).pin_memory()
for _ in range(3):
    op.apply_host_ptr(hs.data_ptr(), hd.data_ptr())
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(2):
        op.apply_host_ptr(hs.data_ptr(), hd.data_ptr())
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev:
    print(f"{e.time_range.start - t0:9.1f} {e.time_range.end - t0:9.1f} {e.time_range.end - e.time_range.start:8.1f}  {e.name[:60]}")
