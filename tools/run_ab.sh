for v in 0 1 0 1; do
  echo "== NO_TMA=$v" >> gpurun_out/ab_bench.log
  B2S_NO_TMA=$v python bench.py --no-complex --no-e2e --no-cpu 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value']/1e9, d['roofline']['frac'], d['clocks'])" >> gpurun_out/ab_bench.log 2>&1
done
