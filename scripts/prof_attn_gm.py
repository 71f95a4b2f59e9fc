"""configs[2] decode-attention for ncu: 128 pairs, 128K context, attention-record key codes."""
import sys
import torch
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_2603_16435_b200 import codebook as P, device as Dv
D, G, B, HKV = 128, 4, 16, 8
pairs = int(sys.argv[1]) if len(sys.argv) > 1 else B * HKV
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n_init, n_comp, n_local = 4, 131072 - 1028, 1024
ok, ov = O.Rng(1).stack(56, 1024, D, O.KEY), O.Rng(2).stack(16, 512, D, O.VALUE)
ks = P.CodebookStack.from_arrays([ok.entries(s) for s in range(56)], [ok.projection(s) for s in range(56)], 0)
vs = P.CodebookStack.from_arrays([ov.entries(s) for s in range(16)], [ov.projection(s) for s in range(16)], 1)
gen = torch.Generator(device='cuda').manual_seed(1234)
kb, vb = ks.device.payload_bytes(n_comp), vs.device.payload_bytes(n_comp)
kc = torch.randint(0, 256, (pairs, kb), dtype=torch.uint8, device='cuda', generator=gen)
vc = torch.randint(0, 256, (pairs, vb), dtype=torch.uint8, device='cuda', generator=gen)
cap = -(-n_comp // Dv.GM_ALIGN) * Dv.GM_ALIGN
kg = Dv.keycodes_to_gm(ks, kc, n_comp, cap=cap)
del kc
rnd = lambda n: torch.randn(pairs, n, D, device='cuda', generator=gen)
ik, iv, lk, lv = rnd(n_init), rnd(n_init), rnd(n_local), rnd(n_local)
q = torch.randn(pairs, G, D, device='cuda', generator=gen)
f = lambda: Dv.attend_decode(ks, vs, q, kg, vc, n_comp, ik, iv, lk, lv, kcodes_gm_cap=cap)
for _ in range(iters): f()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): f()
e.record(); torch.cuda.synchronize()
print(f"{s.elapsed_time(e)/10:.3f} ms per layer-step ({pairs} pairs)")
import ctypes
from paper_2603_16435_b200 import _lib
L = _lib.load()
L.vqkv_profile_enable(1)
for nm in (b"attend_lut_build", b"attend", b"attend_combine"):
    L.vqkv_profile_collect(nm, None, None)
for _ in range(5): f()
torch.cuda.synchronize()
parts = []
for nm in (b"attend_lut_build", b"attend", b"attend_combine"):
    t, n = ctypes.c_double(), ctypes.c_uint64()
    L.vqkv_profile_collect(nm, ctypes.byref(t), ctypes.byref(n))
    parts.append(f"{nm.decode()} {t.value / max(n.value, 1):.3f}")
L.vqkv_profile_enable(0)
print("  kernels (ms/launch): " + ", ".join(parts))
