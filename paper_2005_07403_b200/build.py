"""Build the native engine in-tree: ``python paper_2005_07403_b200/build.py``.

One nvcc invocation compiles the CUDA sources for sm_100a only
(``-gencode arch=compute_100a,code=sm_100a``) into ``_native/libb2s.so``.
``-fmad=false`` forbids silent fma contraction: every fused multiply-add in
the kernels is an explicit ``__fma_rn`` so rounding matches the reference.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SOURCES = ["csrc/b2s_kernels.cu", "csrc/b2s_synth.cu", "csrc/b2s_host.cu",
           "csrc/b2s_verify.cu", "csrc/b2s_phases.cu"]
HEADERS = ["csrc/b2s_lane.cuh", "csrc/b2s_svd2.cuh", "csrc/b2s_fast.cuh", "csrc/b2s_tma.cuh", "csrc/b2s_common.cuh",
           "csrc/b2s_sort_variant.cuh",
           "../include/b2s.h"]
OUT = os.path.join(HERE, "_native", "libb2s.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3",
              "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler",
              "-fPIC,-fopenmp", "-shared", "-lgomp"]


def _stale():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = SOURCES + HEADERS + ["build.py"]
    return any(os.path.getmtime(os.path.join(HERE, p)) > t for p in deps)


def build(force=False, verbose=False, out=None, defines=()):
    """Compile the library (to `out` with extra -D `defines` for A/B
    variants; those are always rebuilt)."""
    if out is None and not force and not _stale():
        return OUT
    target = out or OUT
    os.makedirs(os.path.dirname(os.path.abspath(target)), exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    if not os.path.exists("/usr/local/cuda/bin/nvcc") and nvcc == "nvcc":
        pass
    elif nvcc == "nvcc" and os.path.exists("/usr/local/cuda/bin/nvcc"):
        nvcc = "/usr/local/cuda/bin/nvcc"
    cmd = [nvcc] + NVCC_FLAGS + (["-Xptxas", "-v"] if verbose else []) + list(defines) + \
        ["-o", target + ".tmp"] + [os.path.join(HERE, s) for s in SOURCES]
    subprocess.run(cmd, check=True)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    argv = sys.argv[1:]
    out = argv[argv.index("--out") + 1] if "--out" in argv else None
    print(build(force="--force" in argv, verbose="-v" in argv, out=out,
                defines=[a for a in argv if a.startswith("-D")]))
