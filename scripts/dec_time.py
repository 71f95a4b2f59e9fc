"""Decode (K2) timing at the bench's configs[0] shape (dev aid)."""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2603_16435_b200 import codebook as P, device as Dv
out = []
for name, seed, n, S in (("K", 1, 56, 1024), ("V", 2, 16, 512)):
    g = np.random.default_rng(seed)
    st = P.CodebookStack.from_arrays([g.standard_normal((S, 128), dtype=np.float32) for _ in range(n)],
                                     [(g.standard_normal((128, 128), dtype=np.float32) / np.sqrt(128)).astype(np.float32) for _ in range(n)])
    x = torch.randn(256, 4096, 128, device='cuda')
    pay, _ = Dv.quantize_streams(st, x)
    for _ in range(3): Dv.reconstruct_streams(st, pay, 4096)
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); Dv.reconstruct_streams(st, pay, 4096); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    gb = 256 * 4096 * n * 512 / 1e9
    out.append(f"{name}: {ts[3]:.3f} ms ({gb/ts[3]:.1f} TB/s L2 gather)")
print("  ".join(out))
