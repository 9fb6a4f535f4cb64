set -o pipefail
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 3 1 4 2; do python tools/prof_kernel.py --config $c --lanes 67108864 --reps 4; done > gpurun_out/prof.log 2>&1
