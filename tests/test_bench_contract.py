"""bench.py's driver contract on CPU: the reference arm's JSON line (it runs
the CPU oracle only, so it works without a GPU) and the pure helpers that
assemble the device arm's roofline object."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_reference_arm_json_line():
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0", "--ref-sample", str(1 << 18)],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"] == bench.METRIC and line["unit"] == "SVD/s"
    assert line["higher_is_better"] is True and line["n_gpus"] == 1
    assert line["steps"] == 1 and line["warmup"] == 0 and line["value"] > 0
    assert line["config"]["n"] == 1 << 30 and line["config"]["field"] == "real"
    cb = line["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert cb["value_1thread"] > 0 and cb["sample_lanes"] == 1 << 18
    assert "cpu_model" in cb
    # the reference arm maps no engine code (it used to load libb2s.so)
    assert not any("libb2s" in x for x in line["native_libs"]), line["native_libs"]
    assert "timed_sample" in line["config"]
    e2e = line["e2e"]
    assert e2e["value"] == line["value"] and e2e["unit"] == line["unit"]
    assert e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0


def test_package_import_maps_no_native_code():
    code = ("import paper_2005_07403_b200 as b, paper_2005_07403_b200.synth as s, bench;"
            "from paper_2005_07403_b200 import _lib;"
            "s.generate(3, 1, 0, 64);"
            "assert not _lib.loaded();"
            "assert not any('libb2s' in x for x in bench.repo_native_libs())")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                       timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr


def test_roofline_object():
    res = {"field": "real", "n_shard": 1 << 30, "avg_kernel_ms": 25.0}
    rf = bench.roofline(res, 3, 6454.3, "measured")
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["peak"] == 6454.3
    algo = 120 * (1 << 30)
    assert rf["algorithmic_bytes_per_launch"] == algo
    assert abs(rf["achieved"] - algo / 0.025 / 1e9) < 0.1
    assert abs(rf["frac"] - rf["achieved"] / 6454.3) < 1e-3
    assert rf["traffic"] is None or 0.9 * algo < rf["traffic"] < 1.1 * algo
    cres = {"field": "complex", "n_shard": 1 << 28, "avg_kernel_ms": 16.0}
    assert bench.roofline(cres, 4, 6454.3, "measured")["algorithmic_bytes_per_launch"] == 216 * (1 << 28)


def test_roofline_fp64_term():
    """Both roofline terms: 70 / 178 algorithmic flops per SVD over the
    measured FP64 peak, the binding term named, the issued FP64-pipe
    fraction from the committed ncu capture."""
    peak, how = bench.fp64_peak()
    assert peak and 20 < peak < 60, (peak, how)       # B200 DFMA ~37 TFLOP/s
    res = {"field": "complex", "n_shard": 1 << 28, "avg_kernel_ms": 16.0}
    rf = bench.roofline(res, 4, 6454.3, "measured", (peak, how))
    fp = rf["fp64"]
    assert abs(fp["algorithmic_tflops"] - 178 * (1 << 28) / 0.016 / 1e12) < 1e-3
    assert abs(fp["frac"] - fp["algorithmic_tflops"] / peak) < 1e-3
    assert rf["bound"] == "hbm" and 0 < fp["issued_fp64_pipe_frac"] < 1
    slow = bench.roofline(res, 4, 6454.3, "measured", (0.01, "tiny"))
    assert slow["bound"] == "fp64"


def test_workload_configs():
    for config, field, n in ((3, "real", 1 << 30), (4, "complex", 1 << 28)):
        c = bench.workload_config(config, 1)
        assert c["field"] == field and c["n"] == n and c["workload"].startswith("config%d" % config)
        assert "model" not in c


def test_gpus_flag_refuses_when_gpus_are_missing():
    """`bench.py --gpus 2` outside torchrun launches two ranks itself; with
    fewer visible GPUs it refuses instead of timing one GPU as two."""
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "B2S_DIST_BACKEND"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 2 and "needs 2 visible GPUs" in r.stderr, r.stderr
    assert r.stdout.strip() == ""
