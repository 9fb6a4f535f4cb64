"""B200-native batched SVD of 2x2 real and complex fp64 matrices.

A from-scratch GPU engine for the batched algorithm of arXiv 2005.07403
(Novakovic), exposing the API of the reference package ``lanesvd`` 0.1.0:
exact power-of-two prescaling, URV reduction to a non-negative triangle,
closed-form triangle SVD and U/V assembly, fused in one sm_100a kernel per
field that runs one SVD per thread over structure-of-arrays trains.
Results are bit-identical to the reference's CPU pipeline.

The native library ``_native/libb2s.so`` (C-ABI: ``include/b2s.h``) is the
only compute path; importing this package without it raises.
"""

from ._lib import LIB_PATH, assert_device_fp_env
from .layout import (LANE_WIDTH, Batch2x2, MatrixSvd, SvdBatchOut,
                     aligned_zeros, from_trains, pack, padded_len, unpack,
                     unpack_inputs)
from .driver import (RunConfig, run_batch, run_batch_into, shards,
                     svd2_chunk, svd2_single)
from .svd2 import Svd2, backscale, svd2_lanes

__all__ = [
    "LANE_WIDTH", "padded_len", "aligned_zeros", "Batch2x2", "SvdBatchOut",
    "MatrixSvd", "pack", "unpack", "from_trains", "unpack_inputs",
    "RunConfig", "run_batch", "run_batch_into", "svd2_chunk", "svd2_single", "shards",
    "Svd2", "svd2_lanes", "backscale", "assert_device_fp_env", "LIB_PATH",
]

__version__ = "0.1.0"
