"""Per-phase clock64 breakdown of the decode-attention main kernel (diagnostics build:
python -c "from paper_2603_16435_b200 import build as b; b.build_variant('phases', ('VQKV_ATTN_PHASES',))"
then VQKV_LIB=build/var/phases.so python scripts/attn_phases.py)."""
import ctypes, os, runpy, sys
import numpy as np
sys.argv = [sys.argv[0], "128", "3"]
ns = runpy.run_path(os.path.join(os.path.dirname(__file__), "prof_attn_gm.py"))
from paper_2603_16435_b200 import _lib
L = _lib.load()
buf = (ctypes.c_ulonglong * (256 * 16))()
L.vqkv_attn_phase_read(buf)  # clear
ns["f"]()
import torch
torch.cuda.synchronize()
L.vqkv_attn_phase_read(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(256, 16)[:148].astype(np.float64)
names = ["keys(incl LUT wait)", "LUT wait", "softmax", "values", "fold", "contraction/seg", "chunks", "kernel",
         " val: zero+bar", " val: slab waits", " val: compact+flush (t0)", " val: slab barriers (t0)",
         " keys: pass 1", " keys: sums+stats", " keys: pass 2", " keys: final logits"]
mhz = 1.9e3
for i, n in enumerate(names):
    col = a[:, i]
    if n == "chunks":
        print(f"{n:22s} mean {col.mean():8.2f} min {col.min():6.0f} max {col.max():6.0f}")
    else:
        print(f"{n:22s} mean {col.mean()/mhz:8.1f} us  min {col.min()/mhz:8.1f}  max {col.max()/mhz:8.1f}")
