"""Small decode-attention run for ncu (config-3 geometry, fewer pairs)."""
import sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2603_16435_b200 import codebook as P, device as Dv
D, G = 128, 4
pairs = int(sys.argv[1]) if len(sys.argv) > 1 else 16
n_init, n_comp, n_local = 4, 130044, 1024
def stack(seed, n, S):
    g = np.random.default_rng(seed)
    return P.CodebookStack.from_arrays([g.standard_normal((S, D), dtype=np.float32) for _ in range(n)],
        [(g.standard_normal((D, D), dtype=np.float32) / np.sqrt(D)).astype(np.float32) for _ in range(n)])
ks, vs = stack(1, 56, 1024), stack(2, 16, 512)
kc = torch.randint(0, 256, (pairs, ks.device.payload_bytes(n_comp)), dtype=torch.uint8, device='cuda')
vc = torch.randint(0, 256, (pairs, vs.device.payload_bytes(n_comp)), dtype=torch.uint8, device='cuda')
ik, iv = torch.randn(pairs, n_init, D, device='cuda'), torch.randn(pairs, n_init, D, device='cuda')
lk, lv = torch.randn(pairs, n_local, D, device='cuda'), torch.randn(pairs, n_local, D, device='cuda')
q = torch.randn(pairs, G, D, device='cuda')
for _ in range(2): Dv.attend_decode(ks, vs, q, kc, vc, n_comp, ik, iv, lk, lv)
torch.cuda.synchronize(); print("ok")
