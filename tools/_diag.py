"""The diagnostic build of the engine (tools only): the same sources with
-DB2S_DIAGNOSTICS=1, which adds the no-math traffic probes (k_ring_probe,
k_traffic_bulk) the product library does not export."""
import ctypes
import importlib.util
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tools", "_build", "libb2s_diag.so")


def load():
    if not os.path.exists(OUT):
        spec = importlib.util.spec_from_file_location(
            "_b2s_build", os.path.join(ROOT, "paper_2005_07403_b200", "build.py"))
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        mod.build(out=OUT, defines=["-DB2S_DIAGNOSTICS=1"])
    return ctypes.CDLL(OUT)
