"""Per-CTA phase clocks of the attention main kernel: what the slowest CTAs do differently (dev aid;
VQKV_LIB=build/var/phases.so)."""
import ctypes, os, runpy, sys
import numpy as np
sys.argv = [sys.argv[0], "128", "3"]
ns = runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "prof_attn_gm.py"))
from paper_2603_16435_b200 import _lib
import torch
L = _lib.load()
buf = (ctypes.c_ulonglong * (256 * 16))()
L.vqkv_attn_phase_read(buf)
ns["f"]()
torch.cuda.synchronize()
L.vqkv_attn_phase_read(buf)
a = np.frombuffer(buf, dtype=np.uint64).reshape(256, 16)[:148].astype(np.float64) / 1.9e3
kern, keys, vals, con, chunks = a[:, 7], a[:, 0], a[:, 3], a[:, 5], a[:, 6] * 1.9e3
order = np.argsort(kern)
print("CTA  kernel  keys  lutwait values (zero slabw flush) contraction  chunks")
for i in list(order[:5]) + list(order[-8:]):
    print(f"{i:4d} {kern[i]:7.1f} {keys[i]:6.1f} {a[i,1]:5.1f} {vals[i]:6.1f} ({a[i,8]:4.1f} {a[i,9]:4.1f} {a[i,10]:6.1f}) {con[i]:8.1f} {chunks[i]:5.0f}")
vo = np.argsort(vals)
print("values extremes:", [(int(i), round(vals[i], 1), int(chunks[i])) for i in list(vo[:4]) + list(vo[-4:])])
print("corr(kernel, keys) %.2f  corr(kernel, values) %.2f  corr(kernel, contraction) %.2f" %
      (np.corrcoef(kern, keys)[0, 1], np.corrcoef(kern, vals)[0, 1], np.corrcoef(kern, con)[0, 1]))
# SM id parity / die halves, if the CTA -> SM mapping is the identity for a one-wave persistent grid
print("mean kernel by CTA half: %.1f / %.1f" % (kern[:74].mean(), kern[74:].mean()))
