"""Bare MMA pipeline timing (VQKV_DBG=32: epilogue only drains accumulators; codes are wrong)."""
import os, sys
os.environ["VQKV_DBG"] = os.environ.get("VQKV_DBG", "32")
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2603_16435_b200 import codebook as P, device as Dv
for n, S in ((56, 1024), (16, 512), (8, 2048)):
    g = np.random.default_rng(1)
    st = P.CodebookStack.from_arrays([g.standard_normal((S, 128), dtype=np.float32) for _ in range(n)],
                                     [(g.standard_normal((128, 128), dtype=np.float32) / np.sqrt(128)).astype(np.float32) for _ in range(n)])
    x = torch.randn(32, 31740, 128, device='cuda')
    Dv.quantize_streams(st, x); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3): Dv.quantize_streams(st, x)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 3
    print(f"N={n} S={S}: {ms:.2f} ms  {2*128*n*S*x.shape[0]*x.shape[1]/ms/1e9:.0f} TFLOP/s (dbg={os.environ['VQKV_DBG']})")
