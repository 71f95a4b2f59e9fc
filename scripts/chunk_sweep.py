"""Encode time at the bench shape (256 streams x 31,740 rows) vs VQKV_CHUNK_STREAMS (dev aid)."""
import os, sys, torch
sys.path.insert(0, '.')
import bench
from paper_2603_16435_b200 import device as Dv
kst, vst = bench.make_stacks(0)
Kh, Vh = bench.gen_inputs(torch, 256, bench.PREFILL, 0)
Kd, Vd = Kh.cuda(), Vh.cuda()
del Kh, Vh
for c in sys.argv[1:]:
    os.environ["VQKV_CHUNK_STREAMS"] = c
    for _ in range(2):
        Dv.quantize_streams(kst, Kd); Dv.quantize_streams(vst, Vd)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        s, m, e = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        s.record(); Dv.quantize_streams(kst, Kd); m.record(); Dv.quantize_streams(vst, Vd); e.record()
        torch.cuda.synchronize()
        ts.append((s.elapsed_time(m), m.elapsed_time(e)))
    k = sorted(t[0] for t in ts)[1]; v = sorted(t[1] for t in ts)[1]
    print(f"chunk={c:>4}: K {k:.1f} ms  V {v:.1f} ms  step {k+v:.1f} ms")
