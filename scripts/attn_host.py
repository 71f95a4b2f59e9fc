"""Host issue time vs device time of the decode-attention call (dev aid)."""
import os, runpy, sys, time
sys.argv = [sys.argv[0], "128", "3"]
ns = runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "prof_attn_gm.py"))
import torch
f = ns["f"]
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
s.record()
for _ in range(20): f()
t1 = time.perf_counter()
e.record()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host issue {1e3*(t1-t0)/20:.3f} ms/call, device {s.elapsed_time(e)/20:.3f} ms/call, wall {1e3*(t2-t0)/20:.3f} ms/call")
