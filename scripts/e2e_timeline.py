"""Per-call spans of back-to-back host-buffer steps (dev aid): where the e2e step's time goes."""
import sys, torch
sys.path.insert(0, '.')
import bench
from paper_2603_16435_b200 import device as Dv
kst, vst = bench.make_stacks(0)
ns = 256
Kh, Vh = bench.gen_inputs(torch, ns, bench.PREFILL, 0)
mid = Kh.shape[1]
out = {n: (torch.empty((ns, st.device.payload_bytes(mid)), dtype=torch.uint8, pin_memory=True),
           torch.empty((ns, mid), dtype=torch.float32, pin_memory=True)) for n, st in (("K", kst), ("V", vst))}
def call(n):
    st, xh = (kst, Kh) if n == "K" else (vst, Vh)
    Dv.quantize_streams_host(st, xh, payload_host=out[n][0], norms_host=out[n][1], blocking=False)
for _ in range(4):
    call("K"); call("V")
torch.cuda.synchronize()
import time
ev, host = [], []
for _ in range(4):
    h0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True); e0.record(); call("K")
    e1 = torch.cuda.Event(enable_timing=True); e1.record(); call("V")
    e2 = torch.cuda.Event(enable_timing=True); e2.record()
    ev.append((e0, e1, e2))
    host.append(1e3 * (time.perf_counter() - h0))
torch.cuda.synchronize()
print("host enqueue ms per step:", " ".join(f"{h:.1f}" for h in host))
for i, (a, b, c) in enumerate(ev):
    print(f"step {i}: K span {a.elapsed_time(b):.1f} ms, V span {b.elapsed_time(c):.1f} ms, step {a.elapsed_time(c):.1f} ms")
