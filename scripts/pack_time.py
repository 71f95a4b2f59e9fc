"""Times the code-packing kernel at the bench shape (dev aid)."""
import sys, ctypes
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2603_16435_b200 import codebook as P, device as Dv, _lib
streams = int(sys.argv[1]) if len(sys.argv) > 1 else 32
L = _lib.load()
for name, seed, n, S in (("K", 1, 56, 1024), ("V", 2, 16, 512)):
    g = np.random.default_rng(seed)
    st = P.CodebookStack.from_arrays([g.standard_normal((S, 128), dtype=np.float32) for _ in range(n)],
                                     [(g.standard_normal((128, 128), dtype=np.float32) / np.sqrt(128)).astype(np.float32) for _ in range(n)])
    x = torch.randn(streams, 31740, 128, device='cuda')
    Dv.quantize_streams(st, x); torch.cuda.synchronize()
    L.vqkv_profile_enable(1)
    for nm in (b"pack", b"encode_tc"): L.vqkv_profile_collect(nm, None, None)
    for _ in range(3): Dv.quantize_streams(st, x)
    torch.cuda.synchronize()
    out = []
    for nm in (b"encode_tc", b"pack"):
        t = ctypes.c_double(); c = ctypes.c_uint64()
        L.vqkv_profile_collect(nm, ctypes.byref(t), ctypes.byref(c))
        out.append(f"{nm.decode()} {t.value / max(c.value, 1):.3f} ms")
    L.vqkv_profile_enable(0)
    print(name, "  ".join(out))
