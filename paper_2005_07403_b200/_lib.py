"""ctypes binding of the native engine ``_native/libb2s.so`` (include/b2s.h).

The CUDA library is the only compute path.  It is mapped on first use
(``_lib.lib``), not at import, so that processes which only need the
package's host-side helpers -- the layout types, the NumPy input generator
of the CPU baseline -- never load it; the first compute call raises
``NativeLibraryMissing`` if it is not built.  There is no CPU fallback.
Build it with
``python -c "import __graft_entry__ as g; g.build()"`` (or
``python paper_2005_07403_b200/build.py``).
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# B2S_LIBRARY selects another build of the same ABI (A/B kernel variants
# from `build.py --out PATH -DNAME=VALUE`); the default is the in-tree build.
LIB_PATH = os.environ.get("B2S_LIBRARY") or os.path.join(_HERE, "_native", "libb2s.so")

BACKSCALE = {"none": 0, "safe": 1, "unconditional": 2}
FLAG_SINE_FORM = 1
FLAG_STATES = 2
FLAG_STATES_FULL = 4
STATES_REAL = 16
STATES_COMPLEX = 20

# exported symbols, exactly the functions declared in include/b2s.h
SYMBOLS = (
    "b2s_version", "b2s_last_error", "b2s_svd2_real", "b2s_svd2_complex",
    "b2s_svd2_real_host", "b2s_svd2_complex_host", "b2s_backscale",
    "b2s_synth", "b2s_check_fp_env", "b2s_math_probe",
    "b2s_reserve_workspace", "b2s_hard_lane_count",
    "b2s_svd2_real_records", "b2s_svd2_complex_records", "b2s_metrics",
    "b2s_oracle_svd2", "b2s_svd2_phase", "b2s_lane_op",
)

_P = ctypes.c_void_p
_PA = ctypes.POINTER(ctypes.c_void_p)   # array of train pointers
_i64 = ctypes.c_int64
_int = ctypes.c_int


class NativeLibraryMissing(ImportError):
    pass


def _load():
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryMissing(
            "libb2s.so not built (%s); run __graft_entry__.build()" % LIB_PATH)
    L = ctypes.CDLL(LIB_PATH)
    L.b2s_version.restype = _int
    L.b2s_last_error.restype = ctypes.c_char_p
    L.b2s_svd2_real.argtypes = [_i64, _PA, _PA, _PA, _P, _P, _P, _int, _int,
                                _PA, _P]
    L.b2s_svd2_complex.argtypes = [_i64, _PA, _PA, _PA, _PA, _PA, _PA, _P, _P,
                                   _P, _int, _int, _PA, _P]
    L.b2s_svd2_real_host.argtypes = [_i64, _PA, _PA, _PA, _P, _P, _P, _int,
                                     _int, _int, _i64]
    L.b2s_svd2_complex_host.argtypes = [_i64, _PA, _PA, _PA, _PA, _PA, _PA,
                                        _P, _P, _P, _int, _int, _int, _i64]
    L.b2s_backscale.argtypes = [_i64, _P, _P, _P, _int, _P, _P, _P, _P]
    L.b2s_synth.argtypes = [_int, ctypes.c_uint64, _i64, _i64, _PA, _PA, _P]
    L.b2s_check_fp_env.argtypes = [_int]
    L.b2s_math_probe.argtypes = [_int, _i64, _P, _P, _P, _P]
    L.b2s_reserve_workspace.argtypes = [_int, _i64, _P]
    L.b2s_metrics.argtypes = [_i64, _PA, _PA, _PA, _PA, _PA, _PA, _P, _P, _P,
                              _P, _int, _P, _P, _P, _P]
    L.b2s_svd2_real_records.argtypes = [_i64, _P, _PA, _PA, _P, _P, _P, _int,
                                        _int, _P]
    L.b2s_svd2_complex_records.argtypes = [_i64, _P, _PA, _PA, _PA, _PA, _P,
                                           _P, _P, _int, _int, _P]
    L.b2s_hard_lane_count.argtypes = [_int]
    L.b2s_oracle_svd2.argtypes = [_i64, _PA, _PA, _PA, _P]
    L.b2s_svd2_phase.argtypes = [_int, _int, _int, _i64, _int, _PA, _int, _PA, _P]
    L.b2s_lane_op.argtypes = [_int, _i64, _int, _PA, _int, _PA, _P]
    for name in SYMBOLS:
        if name not in ("b2s_version", "b2s_last_error"):
            getattr(L, name).restype = _int
    L.b2s_hard_lane_count.restype = ctypes.c_longlong
    return L


_loaded = None
_load_lock = threading.Lock()


def get():
    """The mapped library (maps it on first call)."""
    global _loaded
    with _load_lock:
        if _loaded is None:
            _loaded = _load()
            globals()["lib"] = _loaded
    return _loaded


def __getattr__(name):
    # PEP 562: `_lib.lib` maps libb2s.so the first time it is touched from
    # outside; code in this module calls get() (module globals bypass this).
    if name != "lib":
        raise AttributeError(name)
    return get()


def loaded():
    """True once libb2s.so has been mapped into this process."""
    return _loaded is not None


def ptr_array(ptrs):
    """A C array of raw addresses (ints)."""
    arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
    return ctypes.cast(arr, _PA), arr


def check(rc, what):
    """Map a C-ABI return code onto the reference's exception classes."""
    if rc == 0:
        return
    msg = "%s: %s" % (what, get().b2s_last_error().decode(errors="replace"))
    if rc > 0:
        raise ValueError(msg)
    raise RuntimeError(msg)


_env_checked = set()
_env_lock = threading.Lock()


def assert_device_fp_env(device):
    """GPU analogue of lanes.assert_fp_env (lanes.py:274-302), once per
    device: round-to-nearest-even, gradual underflow, fused fma."""
    with _env_lock:
        if device in _env_checked:
            return
        check(get().b2s_check_fp_env(int(device)), "device FP environment")
        _env_checked.add(device)
