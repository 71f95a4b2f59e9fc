"""Quick device-side timing of encode / decode at the LLaMA3.1-8B shape (dev aid)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2603_16435_b200 import codebook as P, device as Dv

def stack(seed, n, S, D=128):
    g = np.random.default_rng(seed)
    ent = [g.standard_normal((S, D), dtype=np.float32) for _ in range(n)]
    prj = [(g.standard_normal((D, D), dtype=np.float32) / np.sqrt(D)).astype(np.float32) for _ in range(n)]
    return P.CodebookStack.from_arrays(ent, prj)

def timeit(fn, iters=3):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters

streams = int(sys.argv[1]) if len(sys.argv) > 1 else 32
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 31740
for name, n, S in (("K", 56, 1024), ("V", 16, 512)):
    st = stack(1 if name == "K" else 2, n, S)
    x = torch.randn(streams, rows, 128, device='cuda')
    ms = timeit(lambda: Dv.quantize_streams(st, x))
    vec = streams * rows
    flop = 2 * 128 * n * S * vec
    print(f"encode {name}: {vec} vectors {ms:.2f} ms  {vec/ms/1e3:.1f} Mvec/s  {flop/ms/1e9:.1f} TFLOP/s  counters={Dv.encode_counters(st)}")
    pay, nrm = Dv.quantize_streams(st, x)
    msd = timeit(lambda: Dv.reconstruct_streams(st, pay, rows))
    byt = pay.numel() + vec * 512
    print(f"decode {name}: {msd:.2f} ms  {byt/msd/1e6:.1f} GB/s  gather {vec*n*512/msd/1e6:.1f} GB/s")
