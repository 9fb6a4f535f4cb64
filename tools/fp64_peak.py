"""Measured FP64 peak of this B200 (the roofline's FP64 term).

  python tools/fp64_peak.py [--out profiles/fp64_peak.json]

Builds tools/csrc/fp64_peak.cu (sm_100a) into tools/_build/, runs DFMA,
DMUL and DADD throughput kernels (8 independent chains per thread, a
resident grid), samples nvidia-smi clocks during the DFMA run, and writes
the peaks: DFMA counts 2 flops per instruction.
"""
import argparse
import ctypes
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SRC = os.path.join(ROOT, "tools", "csrc", "fp64_peak.cu")
OUT = os.path.join(ROOT, "tools", "_build", "libfp64_peak.so")


def build():
    if not os.path.exists(OUT) or os.path.getmtime(OUT) < os.path.getmtime(SRC):
        os.makedirs(os.path.dirname(OUT), exist_ok=True)
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-fmad=false",
                        "-Xcompiler", "-fPIC", "-shared", "-o", OUT, SRC], check=True)
    L = ctypes.CDLL(OUT)
    L.fp64_peak.argtypes = [ctypes.c_int, ctypes.c_longlong, ctypes.c_int,
                            ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_float)]
    return L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--iters", type=int, default=200000)
    a = ap.parse_args()
    import bench
    L = build()
    res = {}
    for op, name in ((0, "dfma"), (1, "dmul"), (2, "dadd")):
        best = None
        for ctas in (4, 8):
            v, ms = ctypes.c_double(), ctypes.c_float()
            clocks = bench.Clocks(0) if op == 0 and ctas == 8 else None
            if clocks:
                time.sleep(0.2)
            rc = L.fp64_peak(op, a.iters, ctas, ctypes.byref(v), ctypes.byref(ms))
            clk = clocks.stop() if clocks else None
            assert rc == 0, rc
            rec = {"ops_per_s": v.value, "ms": ms.value, "ctas_per_sm": ctas}
            if clk:
                rec["clocks"] = clk
            if best is None or v.value > best["ops_per_s"]:
                best = rec
        res[name] = best
    out = {"dfma_tflops": round(2 * res["dfma"]["ops_per_s"] / 1e12, 3),
           "dmul_tops": round(res["dmul"]["ops_per_s"] / 1e12, 3),
           "dadd_tops": round(res["dadd"]["ops_per_s"] / 1e12, 3),
           "fp64_instr_per_s": res["dfma"]["ops_per_s"],
           "detail": res,
           "how": "tools/fp64_peak.py: 8 independent DFMA/DMUL/DADD chains per thread, "
                  "SMs x {4,8} CTAs x 256 threads, best of the two, CUDA events"}
    print(json.dumps(out))
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
