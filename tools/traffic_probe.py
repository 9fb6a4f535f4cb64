"""Achievable HBM bandwidth for the SVD kernels' traffic shape (4 trains
read through the TMA ring, 11 written with streaming stores, no math)."""
import ctypes, os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2005_07403_b200 import _lib
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _diag
L = _diag.load()
L.b2s_ring_probe.argtypes = [ctypes.c_int64, _lib._PA, _lib._PA, ctypes.c_int, ctypes.c_void_p]
n = 1 << 28
a = torch.randn(4, n, dtype=torch.float64, device="cuda")
o = torch.empty(11, n, dtype=torch.float64, device="cuda")
ap, k1 = _lib.ptr_array([a[t].data_ptr() for t in range(4)])
op, k2 = _lib.ptr_array([o[t].data_ptr() for t in range(11)])
s = torch.cuda.current_stream().cuda_stream
ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
for k in range(5):
    ev[k].record()
    L.b2s_ring_probe(n, ap, op, 1000000, s)
ev[5].record()
torch.cuda.synchronize()
ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(5)]
print("traffic probe 4R+11W n=2^28: ms", ["%.3f" % m for m in ms], "GB/s %.1f" % (120 * n / min(ms[1:]) / 1e6))
L.b2s_traffic_bulk.argtypes = [ctypes.c_int64, _lib._PA, _lib._PA, ctypes.c_void_p]
for k in range(5):
    ev[k].record()
    L.b2s_traffic_bulk(n, ap, op, s)
ev[5].record()
torch.cuda.synchronize()
ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(5)]
ok = all(torch.equal(o[t], a[t % 4]) for t in range(8))
print("bulk-store probe 4R+11W n=2^28: ms", ["%.3f" % m for m in ms], "GB/s %.1f" % (120 * n / min(ms[1:]) / 1e6), "ok", ok)
