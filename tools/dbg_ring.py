import ctypes, os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2005_07403_b200 import _lib
L = ctypes.CDLL(_lib.LIB_PATH)
L.b2s_ring_probe.argtypes = [ctypes.c_int64, _lib._PA, _lib._PA, ctypes.c_int, ctypes.c_void_p]
for n in (1 << 22, (1 << 22) + 256 * 37):
    for spin in (0, 3, 50, -20, -200):
        a = torch.randn(4, n, dtype=torch.float64, device="cuda")
        o = torch.zeros_like(a)
        ap, k1 = _lib.ptr_array([a[t].data_ptr() for t in range(4)])
        op, k2 = _lib.ptr_array([o[t].data_ptr() for t in range(4)])
        rc = L.b2s_ring_probe(n, ap, op, spin, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        tiles = n // 256 * 256
        bad = (a[:, :tiles].view(torch.int64) != o[:, :tiles].view(torch.int64)).sum().item()
        print("n", n, "spin", spin, "rc", rc, "mismatches", bad)
