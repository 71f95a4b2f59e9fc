"""reconstruct_block timing at the configs[0] shape: 256 streams x 4096 rows, random codes (dev aid)."""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2603_16435_b200 import codebook as P, device as Dv
streams, rows = 256, 4096
for name, n, S in (("K", 56, 1024), ("V", 16, 512)):
    g = np.random.default_rng(n)
    st = P.CodebookStack.from_arrays([g.standard_normal((S, 128), dtype=np.float32) for _ in range(n)],
                                     [(g.standard_normal((128, 128), dtype=np.float32) / np.sqrt(128)).astype(np.float32) for _ in range(n)])
    pb = st.device.payload_bytes(rows)
    pay = torch.randint(0, 256, (streams, pb), dtype=torch.uint8, device='cuda')  # 2^bits == S: every field valid
    out = Dv.reconstruct_streams(st, pay, rows)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        Dv.reconstruct_streams(st, pay, rows)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"decode {name}: {ms:.3f} ms  {streams*rows/ms/1e3:.1f} M rows/s  gather {streams*rows*n*512/ms/1e9:.2f} TB/s")
