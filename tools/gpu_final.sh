#!/bin/bash
# Round-end evidence on one B200: tests, smoke, bench lines (C4 headline, C3, C5, fast mode),
# reference arm, launch lists and ncu --set full captures.  Usage: bash tools/gpu_final.sh TAG
T=${1:-r01}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err
timeout 600 python bench.py --impl reference > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
timeout 600 python bench.py --workload C3 --no-cpu-baseline > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err
timeout 600 python bench.py --workload C5 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_c5.json 2> gpurun_out/${T}_bench_c5.err
timeout 600 python bench.py --mode fast --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_c4_fast.json 2> gpurun_out/${T}_bench_c4_fast.err
for W in C3 C4; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/${T}_launches_${W,,}.csv python tools/profile_step.py $W > /dev/null 2>&1
done
# launch list of the bench command itself (the recipe's --metrics gpu__time_duration.sum pass)
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 120 \
  --csv --log-file gpurun_out/${T}_launches_bench_c4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/${T}_launches_bench_c4.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"integrate_mesh_kernel|pattern_kernel|emit_kernel|adjacency_kernel" -c 4 \
  -o gpurun_out/${T}_full_c3 python tools/profile_step.py C3 > gpurun_out/${T}_ncu_c3.log 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:integrate_mesh_kernel -c 1 \
  -o gpurun_out/${T}_ke_c4 python tools/profile_step.py C4 > gpurun_out/${T}_ncu_c4.log 2>&1
echo done
