import numpy as np, torch, time, sys
sys.path.insert(0,'.')
from oracle import oracle as O
from paper_2603_16435_b200 import codebook as P, device as Dv
rng=O.Rng(3); o=rng.stack(2,256,128)
p=P.CodebookStack.from_arrays([o.entries(s) for s in range(o.n)],[o.projection(s) for s in range(o.n)])
xs=rng.matrix(200,128)
Dv.set_encode_path(2)
x=torch.from_numpy(xs).cuda().reshape(1,200,128)
pay,nrm=Dv.quantize_streams(p,x); torch.cuda.synchronize()
ref_pay,ref_norm=o.quantize_batch(xs)
got=o.unpack(pay[0].cpu().numpy(),200); ref=o.unpack(ref_pay,200)
print("rows differing:", int((got!=ref).any(1).sum()), "norm bitexact:", np.array_equal(nrm[0].cpu().numpy().view(np.uint32), ref_norm.view(np.uint32)))
print(got[:3], ref[:3])
print(Dv.encode_counters(p))
