"""paper_2005_07403_b200 -- batched 2x2 SVDs (real and complex fp64) on B200.

The hot path of ``lanesvd`` 0.1.0 (arXiv 2005.07403), rebuilt as sm_100a
CUDA behind the reference's own Python API and SoA layout: exact
power-of-two prescaling, URV reduction to a non-negative triangle, the
closed-form triangle SVD and the U/V assembly run fused in one kernel per
field, one matrix per thread, with results bit-identical to the reference.

Compute happens only in ``_native/libb2s.so`` (C ABI: ``include/b2s.h``),
mapped by the first compute call, which raises if it is not built -- there
is no CPU path.  Importing the package loads no native code (the
reference checks its FP environment at import; here ``assert_fp_env()``
checks the GPU's and runs before a device's first launch).
"""

from ._lib import LIB_PATH, assert_device_fp_env
from .driver import RunConfig, run_batch, run_batch_into, shards, svd2_chunk, svd2_single
from .lanes import assert_fp_env
from .layout import (LANE_WIDTH, Batch2x2, MatrixSvd, SvdBatchOut, aligned_zeros,
                     from_trains, pack, padded_len, unpack, unpack_inputs)
from .svd2 import ScaleResult, Svd2, TriangleSvd, UrvState, backscale, svd2_lanes
from .verify import Metrics, metrics, oracle_svd2

# lanesvd's package namespace (lanesvd/__init__.py) plus this engine's extras
__all__ = sorted([
    "LANE_WIDTH", "padded_len", "Batch2x2", "SvdBatchOut", "MatrixSvd",
    "RunConfig", "run_batch", "svd2_chunk", "svd2_single", "Metrics", "metrics",
    "aligned_zeros", "pack", "unpack", "unpack_inputs", "from_trains",
    "run_batch_into", "shards", "Svd2", "svd2_lanes", "backscale",
    "ScaleResult", "UrvState", "TriangleSvd", "oracle_svd2",
    "assert_fp_env", "assert_device_fp_env", "LIB_PATH",
])

__version__ = "0.1.0"
