"""Encode timing for A/B comparisons (dev aid): median / min of per-launch times."""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2603_16435_b200 import codebook as P, device as Dv
streams = int(sys.argv[1]) if len(sys.argv) > 1 else 32
rows = 31740
out = []
for name, seed, n, S in (("K", 1, 56, 1024), ("V", 2, 16, 512)):
    g = np.random.default_rng(seed)
    st = P.CodebookStack.from_arrays([g.standard_normal((S, 128), dtype=np.float32) for _ in range(n)],
                                     [(g.standard_normal((128, 128), dtype=np.float32) / np.sqrt(128)).astype(np.float32) for _ in range(n)])
    x = torch.randn(streams, rows, 128, device='cuda')
    Dv.quantize_streams(st, x); torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); Dv.quantize_streams(st, x); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    fl = 2 * 128 * n * S * streams * rows
    out.append(f"{name}: med {ts[3]:.2f} ms ({fl/ts[3]/1e9:.0f} TF/s) min {ts[0]:.2f} max {ts[-1]:.2f}")
print("  ".join(out))
