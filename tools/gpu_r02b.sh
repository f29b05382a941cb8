#!/bin/bash
# round-2 check: GPU tests, multi-process sharded runs on one GPU (gloo), bench C3 N=2 (gloo)
mkdir -p gpurun_out
T=${1:-r02b}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
for ex in nccl p2p; do
  for n in 2 3; do
    HX_DIST_BACKEND=gloo HX_EXCHANGE=$ex timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
      --master-addr 127.0.0.1 --master-port $((29500 + n)) tools/check_sharded.py >> gpurun_out/${T}_sharded.txt 2>&1
    echo "exchange=$ex n=$n rc=$?" >> gpurun_out/${T}_sharded.txt
  done
done
HX_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --workload C3 --steps 3 --warmup 3 > gpurun_out/${T}_bench_c3_n2_gloo.json 2> gpurun_out/${T}_bench_c3_n2_gloo.err
HX_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29512 bench.py --gpus 2 --workload C5 --steps 3 --warmup 3 --no-e2e > gpurun_out/${T}_bench_c5_n2_gloo.json 2> gpurun_out/${T}_bench_c5_n2_gloo.err
echo done
