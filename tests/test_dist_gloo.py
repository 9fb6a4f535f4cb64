"""The N>1 path on CPU: two gloo ranks, each owning one contiguous shard.

Covers the host-side multi-rank logic bench.py uses on GPUs (shard
assignment, barrier, max-over-ranks timing, per-shard digests combined
into a checksum of checksums) with the CPU oracle standing in for the
device kernel.  The GPU path itself is exercised by bench.py under torchrun.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, config, n, q):
    import oracle
    from paper_2005_07403_b200 import dist as bd
    from paper_2005_07403_b200 import synth
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port,
                            rank=rank, world_size=world)
    try:
        lo, hi = bd.rank_span(n, rank, world)
        re, im = synth.generate(config, 77, lo, hi - lo)
        out = oracle.svd2(re, im, threads=1)
        bd.barrier()
        t = bd.max_over_ranks(float(rank + 1))
        total = bd.sum_over_ranks(hi - lo)
        digs = bd.gather(bd.shard_digest({k: np.ascontiguousarray(v).view(np.uint64)
                                          for k, v in out.trains().items()}))
        spans = bd.gather((lo, hi))
        if rank == 0:
            q.put((t, total, digs, spans))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("config,n", [(3, 5000), (4, 3000)])
def test_two_rank_shards_match_single_batch(config, n):
    import oracle
    from paper_2005_07403_b200 import dist as bd
    from paper_2005_07403_b200 import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, config, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    t, total, digs, spans = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == 2.0                      # max over ranks
    assert total == n                    # every lane owned exactly once
    assert spans[0][0] == 0 and spans[0][1] == spans[1][0] and spans[1][1] == n
    # partition invariance: the whole batch split at the same boundaries
    re, im = synth.generate(config, 77, 0, n)
    whole = oracle.svd2(re, im, threads=1)
    expect = []
    for lo, hi in spans:
        expect.append(bd.shard_digest({k: np.ascontiguousarray(v[..., lo:hi]).view(np.uint64)
                                       for k, v in whole.trains().items()}))
    assert digs == expect
    assert bd.combine_digests(digs) == bd.combine_digests(expect)


def test_rank_span_more_ranks_than_units():
    from paper_2005_07403_b200 import dist as bd
    spans = [bd.rank_span(300, r, 4) for r in range(4)]
    assert spans[0] == (0, 256) and spans[1] == (256, 300)
    assert spans[2] == (300, 300) and spans[3] == (300, 300)


def test_single_process_helpers_are_identity():
    from paper_2005_07403_b200 import dist as bd
    assert bd.max_over_ranks(3.5) == 3.5
    assert bd.sum_over_ranks(2) == 2.0
    assert bd.gather("x") == ["x"]
    os.environ.pop("WORLD_SIZE", None)
    assert bd.world_info()[0] == 1
