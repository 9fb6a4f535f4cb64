# Multi-rank bench path on one GPU (2 ranks sharing cuda:0 over gloo): the
# torchrun launch the driver uses, and bench.py's own launcher (--gpus 2
# outside torchrun).  A plumbing check; the timings are time-shared.
B2S_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu \
  --e2e-lanes 16777216 > gpurun_out/mr_bench.log 2> gpurun_out/mr_bench.err
echo "rc=$?" >> gpurun_out/mr_bench.log
B2S_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-e2e \
  > gpurun_out/mr_launcher.log 2> gpurun_out/mr_launcher.err
echo "rc=$?" >> gpurun_out/mr_launcher.log
B2S_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 \
  > gpurun_out/mr_ref.log 2> gpurun_out/mr_ref.err
echo "rc=$?" >> gpurun_out/mr_ref.log
