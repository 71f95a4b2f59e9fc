"""Runs the K-stack tensor-core encode a few times (ncu target)."""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2603_16435_b200 import codebook as P, device as Dv
n, S = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (56, 1024)
streams = int(sys.argv[3]) if len(sys.argv) > 3 else 8
g = np.random.default_rng(1)
ent = [g.standard_normal((S, 128), dtype=np.float32) for _ in range(n)]
prj = [(g.standard_normal((128, 128), dtype=np.float32) / np.sqrt(128)).astype(np.float32) for _ in range(n)]
st = P.CodebookStack.from_arrays(ent, prj)
x = torch.randn(streams, 31740, 128, device='cuda')
for _ in range(3):
    Dv.quantize_streams(st, x)
torch.cuda.synchronize()
print("ok", Dv.encode_counters(st))
