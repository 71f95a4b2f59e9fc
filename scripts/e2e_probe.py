"""Where the e2e step's time goes (dev aid): kernel time inside the host-buffer pipeline vs device-only."""
import sys, ctypes, time
import numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_2603_16435_b200 import _lib, device as Dv
L = _lib.load()
kst, vst = bench.make_stacks(0)
ns = 256
Kh, Vh = bench.gen_inputs(torch, ns, bench.PREFILL, 0)
mid = Kh.shape[1]
kph = torch.empty((ns, kst.device.payload_bytes(mid)), dtype=torch.uint8, pin_memory=True)
vph = torch.empty((ns, vst.device.payload_bytes(mid)), dtype=torch.uint8, pin_memory=True)
knh = torch.empty((ns, mid), dtype=torch.float32, pin_memory=True)
vnh = torch.empty((ns, mid), dtype=torch.float32, pin_memory=True)
def step():
    Dv.quantize_streams_host(kst, Kh, payload_host=kph, norms_host=knh, blocking=False)
    Dv.quantize_streams_host(vst, Vh, payload_host=vph, norms_host=vnh, blocking=False)
step(); torch.cuda.synchronize()
names = [b"encode_tc", b"pack", b"encode_exact"]
L.vqkv_profile_enable(1)
for nm in names: L.vqkv_profile_collect(nm, None, None)
t0 = time.perf_counter(); s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); step(); e.record(); torch.cuda.synchronize()
print(f"e2e step {s.elapsed_time(e):.1f} ms (host wall {1e3*(time.perf_counter()-t0):.1f} ms)")
for nm in names:
    t = ctypes.c_double(); c = ctypes.c_uint64()
    L.vqkv_profile_collect(nm, ctypes.byref(t), ctypes.byref(c))
    print(f"  {nm.decode():12s} {t.value:8.1f} ms in {c.value} launches")
Kd, Vd = Kh.cuda(), Vh.cuda()
for nm in names: L.vqkv_profile_collect(nm, None, None)
s.record(); Dv.quantize_streams(kst, Kd); Dv.quantize_streams(vst, Vd); e.record(); torch.cuda.synchronize()
print(f"device-only step {s.elapsed_time(e):.1f} ms")
for nm in names:
    t = ctypes.c_double(); c = ctypes.c_uint64()
    L.vqkv_profile_collect(nm, ctypes.byref(t), ctypes.byref(c))
    print(f"  {nm.decode():12s} {t.value:8.1f} ms in {c.value} launches")
for nm, st, Xh, ph, nh, Xd in (("K", kst, Kh, kph, knh, Kd), ("V", vst, Vh, vph, vnh, Vd)):
    s.record(); Dv.quantize_streams_host(st, Xh, payload_host=ph, norms_host=nh, blocking=False); e.record()
    torch.cuda.synchronize(); a = s.elapsed_time(e)
    s.record(); Dv.quantize_streams(st, Xd); e.record(); torch.cuda.synchronize(); b = s.elapsed_time(e)
    print(f"{nm}: host-buffer call {a:.1f} ms, device-only {b:.1f} ms")
