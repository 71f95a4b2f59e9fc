"""e2e steady state (dev aid): back-to-back host-buffer steps for K+V, K only, V only; device-only for reference."""
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
def timed(fn, n):
    for _ in range(n): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / n
for name, fn in (("K+V", lambda: (call("K"), call("V"))), ("K", lambda: call("K")), ("V", lambda: call("V"))):
    print(f"{name}: 1 step {timed(fn, 1):.1f} ms, 3 steps {timed(fn, 3):.1f} ms/step")
Kd, Vd = Kh.cuda(), Vh.cuda()
print(f"device K+V {timed(lambda: (Dv.quantize_streams(kst, Kd), Dv.quantize_streams(vst, Vd)), 3):.1f} ms/step")
