"""Decode attention with G = 8 query heads per KV head: grouped LUT path vs the generic kernel (dev aid)."""
import os, sys
import torch
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_2603_16435_b200 import codebook as P, device as Dv
D, G, pairs = 128, int(sys.argv[1]) if len(sys.argv) > 1 else 8, 64
n_init, n_comp, n_local = 4, 32768 - 1028, 1024
ok, ov = O.Rng(1).stack(56, 1024, D, O.KEY), O.Rng(2).stack(16, 512, D, O.VALUE)
ks = P.CodebookStack.from_arrays([ok.entries(s) for s in range(56)], [ok.projection(s) for s in range(56)], 0)
vs = P.CodebookStack.from_arrays([ov.entries(s) for s in range(16)], [ov.projection(s) for s in range(16)], 1)
gen = torch.Generator(device='cuda').manual_seed(1)
kc = torch.randint(0, 256, (pairs, ks.device.payload_bytes(n_comp)), dtype=torch.uint8, device='cuda', generator=gen)
vc = torch.randint(0, 256, (pairs, vs.device.payload_bytes(n_comp)), dtype=torch.uint8, device='cuda', generator=gen)
rnd = lambda n: torch.randn(pairs, n, D, device='cuda', generator=gen)
ik, iv, lk, lv = rnd(n_init), rnd(n_init), rnd(n_local), rnd(n_local)
q = torch.randn(pairs, G, D, device='cuda', generator=gen)
f = lambda: Dv.attend_decode(ks, vs, q, kc, vc, n_comp, ik, iv, lk, lv)
res = []
for path in ("0", "1"):
    os.environ["VQKV_ATTEND_PATH"] = path
    for _ in range(3): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5): f()
    e.record(); torch.cuda.synchronize()
    res.append(f"{'LUT (grouped)' if path == '0' else 'generic'} {s.elapsed_time(e)/5:.3f} ms")
print(f"G={G}, {pairs} pairs, 32K context: " + ", ".join(res))
