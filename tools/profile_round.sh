# Refresh the measured evidence under gpurun_out/ (copied to profiles/ after review).
# usage: bash tools/profile_round.sh TAG
T=${1:-r1}
python bench.py > gpurun_out/bench_$T.log 2> gpurun_out/bench_$T.err
python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_small_$T.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch_$T.log 2>&1
python tools/prof_kernel.py --config 3 --lanes 67108864 --reps 2 > gpurun_out/p3_$T.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_svd2|k_fix" -c 2 -f -o gpurun_out/prof_${T}_cfg3 \
    python tools/prof_kernel.py --config 3 --lanes 67108864 --reps 1 > gpurun_out/ncu3_$T.log 2>&1
python tools/prof_kernel.py --config 4 --lanes 33554432 --reps 2 > gpurun_out/p4_$T.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_svd2|k_fix" -c 2 -f -o gpurun_out/prof_${T}_cfg4 \
    python tools/prof_kernel.py --config 4 --lanes 33554432 --reps 1 > gpurun_out/ncu4_$T.log 2>&1
echo done
