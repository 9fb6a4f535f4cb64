"""Why pageable host trains are bounced, not pinned or accessed in place:
on the GPU box, probes the device's pageable-memory access attributes
(HMM / ATS: would let kernels read a caller's malloc'd trains directly) and
times cudaHostRegister / cudaHostUnregister of 1 and 4 GiB arrays (pinning
a caller's trains for the duration of one call).

  python tools/host_memory_probe.py > gpurun_out/host_memory_probe.json
"""
import ctypes
import json
import time

import numpy as np

rt = ctypes.CDLL("libcudart.so.12")
rt.cudaHostRegister.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint]
rt.cudaHostUnregister.argtypes = [ctypes.c_void_p]
rt.cudaFree(None)


def attr(a):
    v = ctypes.c_int()
    rc = rt.cudaDeviceGetAttribute(ctypes.byref(v), a, 0)
    return v.value if rc == 0 else None


res = {"attributes": {"cudaDevAttrPageableMemoryAccess": attr(88),
                      "cudaDevAttrConcurrentManagedAccess": attr(89),
                      "cudaDevAttrHostRegisterSupported": attr(99),
                      "cudaDevAttrPageableMemoryAccessUsesHostPageTables": attr(100)},
       "host_register": {}}
for gib in (1, 4):
    a = np.ones(gib << 27)                       # touched pages, as a filled train block
    t0 = time.perf_counter()
    rc = rt.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    t1 = time.perf_counter()
    rc2 = rt.cudaHostUnregister(a.ctypes.data)
    t2 = time.perf_counter()
    res["host_register"]["%d GiB" % gib] = {"register_s": round(t1 - t0, 4),
                                            "unregister_s": round(t2 - t1, 4),
                                            "register_GBps": round(gib * 1.073741824 / (t1 - t0), 2),
                                            "rc": [rc, rc2]}
print(json.dumps(res))
