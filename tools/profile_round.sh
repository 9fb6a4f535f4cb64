# Refresh the measured evidence under gpurun_out/ (copied to profiles/ after review).
# usage: bash tools/profile_round.sh TAG
# The .ncu-rep captures stay in /tmp on the box (gpurun copies back <= 64 MiB);
# their summaries, stall/opcode mixes and per-lane traffic come back as text.
T=${1:-r2}
python bench.py > gpurun_out/bench_$T.log 2> gpurun_out/bench_$T.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv \
    python bench.py > gpurun_out/ncu_launch_$T.log 2>&1
python tools/prof_kernel.py --config 3 --lanes 67108864 --reps 2 > gpurun_out/p3_$T.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_svd2|k_fix" -c 2 -f -o /tmp/prof_${T}_cfg3 \
    python tools/prof_kernel.py --config 3 --lanes 67108864 --reps 1 > gpurun_out/ncu3_$T.log 2>&1
python tools/prof_kernel.py --config 4 --lanes 33554432 --reps 2 > gpurun_out/p4_$T.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_svd2|k_fix" -c 2 -f -o /tmp/prof_${T}_cfg4 \
    python tools/prof_kernel.py --config 4 --lanes 33554432 --reps 1 > gpurun_out/ncu4_$T.log 2>&1
for c in 3 4; do
  python tools/ncu_summary.py /tmp/prof_${T}_cfg$c.ncu-rep > gpurun_out/${T}_ncu_cfg$c.txt 2>&1
  python tools/ncu_stalls.py /tmp/prof_${T}_cfg$c.ncu-rep >> gpurun_out/${T}_ncu_cfg$c.txt 2>&1
done
python tools/ncu_traffic.py 3 67108864 /tmp/prof_${T}_cfg3.ncu-rep 4 33554432 /tmp/prof_${T}_cfg4.ncu-rep > gpurun_out/${T}_traffic.log 2>&1
cp profiles/ncu_traffic.json gpurun_out/${T}_ncu_traffic.json
echo done
