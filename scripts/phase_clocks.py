"""Per-phase epilogue clock breakdown of the tensor-core encoder (dev aid; VQKV_DBG=2)."""
import os, sys, ctypes
os.environ["VQKV_DBG"] = os.environ.get("VQKV_DBG", "2")
# the phase counters exist only in the diagnostics build (python -c "from paper_2603_16435_b200 import build; build.build_diag()")
os.environ.setdefault("VQKV_LIB", os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "build", "diag", "libvqkv_b200.so"))
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2603_16435_b200 import codebook as P, device as Dv, _lib
n, S = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (56, 1024)
streams = int(sys.argv[3]) if len(sys.argv) > 3 else 32
g = np.random.default_rng(1)
st = P.CodebookStack.from_arrays([g.standard_normal((S, 128), dtype=np.float32) for _ in range(n)],
                                 [(g.standard_normal((128, 128), dtype=np.float32) / np.sqrt(128)).astype(np.float32) for _ in range(n)])
x = torch.randn(streams, 31740, 128, device='cuda')
Dv.quantize_streams(st, x); torch.cuda.synchronize()
L = _lib.load()
base = (ctypes.c_uint64 * 18)()
L.vqkv_encode_phase_clocks(Dv._dev(st).h, base)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); Dv.quantize_streams(st, x); e.record(); torch.cuda.synchronize()
out = (ctypes.c_uint64 * 18)()
L.vqkv_encode_phase_clocks(Dv._dev(st).h, out)
d = [out[k] - base[k] for k in range(18)]
warps = 8 * 148
ms = s.elapsed_time(e)
print(f"n={n} S={S} streams={streams}: {ms:.2f} ms  (~{ms*1.9e6:.3g} clk per warp at 1.9 GHz)")
names = ["prologue", "acc wait", "chunk max", "candidates", "upd: st-wait+arrive", "rs setup", "rs load+dot", "rs min", "code store", "upd: issue+ld0", "upd: e_z wait", "upd: rest", "acc ld"]
tot = sum(d[:13])
for k in range(13):
    print(f"  {names[k]:13s} {d[k]/warps:12.4g} clk/warp  {100*d[k]/tot:5.1f}%")
print("  rescored pairs", d[13])
mma_threads = 2 * 148 if os.environ.get("VQKV_ENC_PAIR", "1") == "0" else 2 * 74  # leader MMA-issuer threads
print("  MMA issuer (clk per thread, leader threads only): acc-free wait %.4g, issue %.4g, chunk wait %.4g, A-tile wait %.4g"
      % tuple(d[14 + k] / mma_threads for k in range(4)))
