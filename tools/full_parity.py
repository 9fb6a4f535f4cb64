"""Full-size parity: every lane of BASELINE configs 3 (real, n = 2^30) and 4
(complex, n = 2^28) -- the bench's own seeded workloads -- through the
streaming kernels on the GPU, compared bit for bit with the CPU oracle
(oracle/svd2_oracle.c, pinned to the reference by tests/golden/).

Inputs are generated on the device (b2s_synth, equal to the host generator:
tests/test_gpu_parity.py::test_device_synth_equals_host_synth) and copied to
the host for the oracle, 2^26 lanes at a time.  Prints one JSON line per
config: lanes compared, differing lanes per output train, hard lanes fixed
up, and a checksum of checksums of the outputs (SHA-256 over the per-chunk
train digests), so two runs or two implementations can be compared.

  python tools/full_parity.py [--configs 3 4] [--chunk 67108864]
"""
import argparse
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: the checker)
import paper_2005_07403_b200 as b2s  # noqa: E402
from paper_2005_07403_b200 import _lib, synth  # noqa: E402
from paper_2005_07403_b200.svd2 import launch_device  # noqa: E402

SEED = 20250705                      # bench.py's workload seed


def run(config, chunk, dev):
    cfg = synth.CONFIGS[config]
    n, cplx = cfg["n"], cfg["field"] == "complex"
    threads = os.cpu_count() or 1
    diff, hard, lanes = {}, 0, 0
    top = hashlib.sha256()
    t0 = time.time()
    for lo in range(0, n, chunk):
        m = min(chunk, n - lo)
        re, im = synth.generate_device(config, SEED, lo, m, device=dev)
        out = b2s.SvdBatchOut.empty(m, cplx, device=dev)
        outd = {"u_re": list(out.u_re), "v_re": list(out.v_re),
                "u_im": list(out.u_im) if cplx else None, "v_im": list(out.v_im) if cplx else None,
                "smax": out.smax, "smin": out.smin, "shift": out.shift}
        launch_device(m, list(re), list(im) if cplx else None, outd, 0)
        torch.cuda.synchronize(dev)
        hard += int(_lib.lib.b2s_hard_lane_count(dev.index or 0))
        got = out.cpu().trains()
        ref = oracle.svd2(re.cpu().numpy(), im.cpu().numpy() if cplx else None, threads=threads).trains()
        del re, im, out, outd
        for k in sorted(ref):
            g = np.ascontiguousarray(got[k]).view(np.uint64)
            r = np.ascontiguousarray(ref[k]).view(np.uint64)
            bad = g != r
            if bad.ndim == 2:
                bad = bad.any(axis=0)
            diff[k] = diff.get(k, 0) + int(np.count_nonzero(bad))
            top.update(k.encode())
            top.update(hashlib.sha256(g.tobytes()).digest())
        lanes += m
        del got, ref
    return {"config": config, "field": cfg["field"], "n": n, "lanes_compared": lanes,
            "seed": SEED, "chunk": chunk, "differing_lanes": diff,
            "bit_identical": all(v == 0 for v in diff.values()),
            "hard_lanes_fixed_up": hard, "checksum_of_checksums": top.hexdigest(),
            "oracle_threads": threads, "wall_s": round(time.time() - t0, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[3, 4])
    ap.add_argument("--chunk", type=int, default=1 << 26)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    ok = True
    for c in a.configs:
        r = run(c, a.chunk, dev)
        ok &= r["bit_identical"]
        print(json.dumps(r), flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
