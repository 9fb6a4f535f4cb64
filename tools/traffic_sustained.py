"""Sustained achievable HBM bandwidth for the real SVD kernel's traffic shape
at the bench's size: 4 trains read through the TMA ring, 11 written with
streaming stores, no math (k_ring_probe), n = 2^30, 25 back-to-back launches
as in bench.py's 20 timed + 5 warm-up steps.  Compare with the bench line's
roofline.achieved (same bytes, same launch shape, plus the SVD arithmetic)."""
import ctypes, json, os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_07403_b200 import _lib
import bench
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _diag
L = _diag.load()
L.b2s_ring_probe.argtypes = [ctypes.c_int64, _lib._PA, _lib._PA, ctypes.c_int, ctypes.c_void_p]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
a = torch.ones(4, n, dtype=torch.float64, device="cuda")
o = torch.empty(11, n, dtype=torch.float64, device="cuda")
ap, k1 = _lib.ptr_array([a[t].data_ptr() for t in range(4)])
op, k2 = _lib.ptr_array([o[t].data_ptr() for t in range(11)])
s = torch.cuda.current_stream().cuda_stream
for _ in range(5):
    L.b2s_ring_probe(n, ap, op, 1000000, s)   # 1000000: all 11 output trains
torch.cuda.synchronize()
clk = bench.Clocks(0)
time.sleep(0.3)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
for k in range(20):
    ev[k].record()
    L.b2s_ring_probe(n, ap, op, 1000000, s)   # 1000000: all 11 output trains
ev[20].record()
torch.cuda.synchronize()
c = clk.stop()
ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(20)]
avg = sum(ms) / len(ms)
print(json.dumps({"probe": "k_ring_probe 4R+11W (no math)", "n": n, "ms_mean": round(avg, 3),
                  "gbs_mean": round(120 * n / avg / 1e6, 1), "gbs_best": round(120 * n / min(ms) / 1e6, 1),
                  "clocks": c}))
