"""configs[3] sweep: S in {256..4096} x N in {2,4,8} on 1,048,576 vectors, tensor-core encoder."""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2603_16435_b200 import codebook as P, device as Dv
rows = 1 << 20
x = torch.randn(32, rows // 32, 128, device='cuda')
print("S     N   ms       Mvec/s   TFLOP/s  ambiguous")
for S in (256, 512, 1024, 2048, 4096):
    for N in (2, 4, 8):
        g = np.random.default_rng(S * 10 + N)
        st = P.CodebookStack.from_arrays([g.standard_normal((S, 128), dtype=np.float32) for _ in range(N)],
                                         [(g.standard_normal((128, 128), dtype=np.float32) / np.sqrt(128)).astype(np.float32) for _ in range(N)])
        Dv.quantize_streams(st, x); torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); Dv.quantize_streams(st, x); e.record(); torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        ms = sorted(ts)[2]
        c = Dv.encode_counters(st)
        print(f"{S:5d} {N:2d} {ms:8.3f} {rows/ms/1e3:9.1f} {2*128*S*N*rows/ms/1e9:8.1f}  {c['ambiguous']/max(c['row_stages'],1):.3f}")
