"""configs[3] sweep for ncu (tensor-pipe utilisation per point): each (S, N) point encodes the same
1,048,576 vectors once (no warm-up: ncu replays every launch with its own cache control).  Run as
  ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
      -k regex:encode_tc_kernel --csv --log-file gpurun_out/sweep_ncu.csv python scripts/sweep_ncu.py > gpurun_out/sweep_points.log
then python scripts/sweep_ncu_summary.py gpurun_out/sweep_points.log gpurun_out/sweep_ncu.csv"""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2603_16435_b200 import codebook as P, device as Dv
from paper_2603_16435_b200 import _lib
rows = 1 << 20
x = torch.randn(32, rows // 32, 128, device='cuda')
L = _lib.load()
L.vqkv_profile_enable(1)
for S in (256, 512, 1024, 2048, 4096):
    for N in (2, 4, 8):
        g = np.random.default_rng(S * 10 + N)
        st = P.CodebookStack.from_arrays([g.standard_normal((S, 128), dtype=np.float32) for _ in range(N)],
                                         [(g.standard_normal((128, 128), dtype=np.float32) / np.sqrt(128)).astype(np.float32) for _ in range(N)])
        torch.cuda.synchronize()
        L.vqkv_profile_collect(b"encode_tc", None, None)
        Dv.quantize_streams(st, x)
        torch.cuda.synchronize()
        ms, n = ctypes.c_double(), ctypes.c_uint64()
        L.vqkv_profile_collect(b"encode_tc", ctypes.byref(ms), ctypes.byref(n))
        print(f"POINT {S} {N} {n.value}", flush=True)
