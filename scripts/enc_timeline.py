"""Timeline of one bench encode step (K then V, 256 streams x 31,740 rows): kernel intervals, idle gaps
and overlap between the two compute streams (dev aid; torch.profiler / CUPTI)."""
import re, sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2603_16435_b200 import codebook as P, device as Dv
from torch.profiler import profile, ProfilerActivity
rows, streams = 31740, int(sys.argv[1]) if len(sys.argv) > 1 else 256
stacks = []
for seed, n, S in ((1, 56, 1024), (2, 16, 512)):
    g = np.random.default_rng(seed)
    stacks.append(P.CodebookStack.from_arrays([g.standard_normal((S, 128), dtype=np.float32) for _ in range(n)],
                                              [(g.standard_normal((128, 128), dtype=np.float32) / np.sqrt(128)).astype(np.float32) for _ in range(n)]))
x = torch.randn(streams, rows, 128, device='cuda')
outs = [(torch.empty(streams, st.device.payload_bytes(rows), dtype=torch.uint8, device='cuda'),
         torch.empty(streams, rows, device='cuda')) for st in stacks]
def step():
    for st, (p, nrm) in zip(stacks, outs):
        Dv.quantize_streams(st, x, payload=p, norms=nrm)
for _ in range(2): step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and "_kernel" in e.name],
            key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
iv = [(e.time_range.start - t0, e.time_range.end - t0, re.search(r"(\w+_kernel)", e.name).group(1)) for e in ev]
end = max(b for _, b, _ in iv)
# busy = union of encode_tc intervals; overlap = time with 2+ encode kernels running
pts = sorted([(a, 1) for a, b, n in iv if "encode_tc" in n] + [(b, -1) for a, b, n in iv if "encode_tc" in n])
busy = over = 0.0
cur, last = 0, 0.0
for t, d in pts:
    if cur >= 1: busy += t - last
    if cur >= 2: over += t - last
    cur += d
    last = t
enc = [b - a for a, b, n in iv if "encode_tc" in n]
print(f"step {end/1e3:.2f} ms, encode_tc launches {len(enc)} (mean {np.mean(enc)/1e3:.3f} ms), union busy {busy/1e3:.2f} ms, "
      f"idle {(end-busy)/1e3:.2f} ms, two launches overlapping {over/1e3:.2f} ms")
others = {}
for a, b, n in iv:
    if "encode_tc" not in n: others[n] = others.get(n, 0.0) + (b - a)
print("other kernels (sum us):", {k: round(v, 1) for k, v in others.items()})
