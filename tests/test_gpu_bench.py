"""GPU: bench.py's own multi-rank launcher (`--gpus N` outside torchrun).

On a one-GPU box the two ranks share cuda:0 over gloo
(B2S_DIST_BACKEND=gloo), which exercises the launcher, sharding, barrier,
max over ranks and the rank-0 line; the timings are not scaling numbers.
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus_2_launches_two_ranks():
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "LOCAL_WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    if torch.cuda.device_count() < 2:
        env["B2S_DIST_BACKEND"] = "gloo"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--config", "1", "--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu"],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout          # rank 0 alone prints
    line = lines[0]
    assert line["n_gpus"] == 2 and len(line["devices"]) == 2
    assert line["config"]["n"] == 1 << 20 and line["value"] > 0
    if torch.cuda.device_count() >= 2:
        assert len({d["pci"] for d in line["devices"]}) == 2
