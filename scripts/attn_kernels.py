"""Per-kernel device times of one decode-attention layer-step (torch.profiler / CUPTI; dev aid)."""
import re
import os, runpy, sys
sys.argv = [sys.argv[0], "128", "3"]
ns = runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "prof_attn_gm.py"))
import torch
from torch.profiler import profile, ProfilerActivity
f = ns["f"]
for _ in range(3): f()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA], acc_events=True) as prof:
    for _ in range(5): f()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
from collections import defaultdict
tot = defaultdict(float); cnt = defaultdict(int)
for e in ev:
    pass
    m = re.search(r"(\w+_kernel)", e.name)
    k = m.group(1) if m else e.name[:40]
    tot[k] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
    cnt[k] += 1
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:42s} {cnt[k]:3d} x {v / cnt[k]:8.1f} us")
# the window of the LUT build + raw rows: first start to last end of those kernels per step
# timeline of the last call: start / end of each kernel relative to the first kernel of that call
evs = sorted([e for e in ev if "_kernel" in e.name or "Memcpy" in e.name], key=lambda e: e.time_range.start)
per_call = len(evs) // 5
last = evs[-per_call:]
t0 = last[0].time_range.start
for e in last:
    m = re.search(r"(\w+_kernel)", e.name)
    print(f"  {m.group(1) if m else e.name[:30]:32s} {e.time_range.start - t0:8.1f} -> {e.time_range.end - t0:8.1f} us")
