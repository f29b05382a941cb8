#!/bin/bash
# multi-process sharded checks on one GPU (gloo, ranks sharing the device): check_sharded.py for both
# exchanges at 2 and 3 ranks, and bench.py --gpus 2 (C3) with its in-bench digest parity
mkdir -p gpurun_out
T=${1:-mp}
for ex in nccl p2p; do
  for n in 2 3; do
    HX_DIST_BACKEND=gloo HX_EXCHANGE=$ex timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
      --master-addr 127.0.0.1 --master-port $((29500 + n)) tools/check_sharded.py >> gpurun_out/${T}_sharded.txt 2>&1
    echo "exchange=$ex n=$n rc=$?" >> gpurun_out/${T}_sharded.txt
  done
done
HX_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --workload C3 --steps 3 --warmup 3 > gpurun_out/${T}_bench_c3_n2_gloo.json 2> gpurun_out/${T}_bench_c3_n2_gloo.err
echo done
