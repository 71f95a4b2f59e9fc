"""Decode-attention timing at BASELINE config 3 shape (dev aid): B=16, 128K context, 8 KV heads, G=4."""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2603_16435_b200 import codebook as P, device as Dv
B, HKV, G, D = 16, 8, 4, 128
ctx = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 131072
gm_mode = "--gm" in sys.argv
import os
n_init, n_local = (0, 0) if os.environ.get("NO_RAW") else (4, 1024)
n_comp = ctx - n_init - n_local
pairs = B * HKV
def stack(seed, n, S):
    g = np.random.default_rng(seed)
    return P.CodebookStack.from_arrays([g.standard_normal((S, D), dtype=np.float32) for _ in range(n)],
        [(g.standard_normal((D, D), dtype=np.float32) / np.sqrt(D)).astype(np.float32) for _ in range(n)])
ks, vs = stack(1, 56, 1024), stack(2, 16, 512)
kb, vb = ks.device.payload_bytes(n_comp), vs.device.payload_bytes(n_comp)
kc = torch.randint(0, 256, (pairs, kb), dtype=torch.uint8, device='cuda')
vc = torch.randint(0, 256, (pairs, vb), dtype=torch.uint8, device='cuda')
rnd = lambda n: torch.randn(pairs, n, D, device='cuda') if n else None
ik, iv, lk, lv = rnd(n_init), rnd(n_init), rnd(n_local), rnd(n_local)
q = torch.randn(pairs, G, D, device='cuda')
if gm_mode:  # the cache's attention layout for the key codes (maintained at append time)
    cap = -(-n_comp // 16) * 16
    kg = Dv.keycodes_to_gm(ks, kc, n_comp, cap=cap)
    f = lambda: Dv.attend_decode(ks, vs, q, kg, vc, n_comp, ik, iv, lk, lv, kcodes_gm_cap=cap)
else:
    f = lambda: Dv.attend_decode(ks, vs, q, kc, vc, n_comp, ik, iv, lk, lv)
f(); torch.cuda.synchronize()
from paper_2603_16435_b200 import _lib
import ctypes
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3): f()
s.record()
for _ in range(10): f()
e.record(); torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
L = _lib.load(); L.vqkv_profile_enable(1)
for nm in (b"attend_lut_build", b"attend", b"attend_combine"): L.vqkv_profile_collect(nm, None, None)
for _ in range(5): f()
torch.cuda.synchronize()
byts = pairs * (kb + vb) + pairs * (n_init + n_local) * D * 4 * 2
print(f"attention ctx={ctx} pairs={pairs}: {ms:.3f} ms/layer-step, {B*ctx/ms/1e6:.2f} G cache-tok/s (B*L/t), "
      f"HBM-equiv {byts/ms/1e6:.1f} GB/s ({byts/ms/1e6/6548.8*100:.1f}% of 6548.8)")
for nm in (b"attend_lut_build", b"attend", b"attend_combine"):
    t = ctypes.c_double(); n = ctypes.c_uint64()
    L.vqkv_profile_collect(nm, ctypes.byref(t), ctypes.byref(n))
    print(f"  {nm.decode():18s} {t.value/max(n.value,1):.3f} ms/launch")
