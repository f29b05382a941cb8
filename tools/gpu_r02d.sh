#!/bin/bash
# round-2 pass: GPU tests, multi-process sharded checks (gloo, ranks sharing one GPU), ncu --set full
# of the integration kernel (C3) and of pattern + emit (C4), with source-level SASS
mkdir -p gpurun_out
T=${1:-r02d}
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
for ex in nccl p2p; do
  for n in 2 3; do
    HX_DIST_BACKEND=gloo HX_EXCHANGE=$ex timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
      --master-addr 127.0.0.1 --master-port $((29500 + n)) tools/check_sharded.py >> gpurun_out/${T}_sharded.txt 2>&1
    echo "exchange=$ex n=$n rc=$?" >> gpurun_out/${T}_sharded.txt
  done
done
HX_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus 2 --workload C3 --steps 3 --warmup 3 > gpurun_out/${T}_bench_c3_n2_gloo.json 2> gpurun_out/${T}_bench_c3_n2_gloo.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:integrate_mesh_kernel -c 1 \
  -o gpurun_out/${T}_full_ke_c3 python tools/profile_step.py C3 > gpurun_out/${T}_ncu_ke.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"pattern_kernel|emit_kernel" -c 2 \
  -o gpurun_out/${T}_full_asm_c4 python tools/profile_step.py C4 > gpurun_out/${T}_ncu_asm.log 2>&1
echo done
