#!/bin/bash
# Round-2 evidence pass: GPU parity tests, smoke, bench lines (C4 headline, C3, C5, fast C4, reference arm),
# launch lists of one C4 and one C5 step.  Usage (repo root, under gpurun): bash tools/gpu_r02.sh TAG [steps...]
TAG=${1:-r02}
shift
STEPS=${*:-"tests smoke bench bench5 bench3 fast ref launches4 launches5"}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
nproc >> gpurun_out/${TAG}_gpu.txt; free -g >> gpurun_out/${TAG}_gpu.txt
for s in $STEPS; do
  echo "== $s $(date +%T)" >> gpurun_out/${TAG}_timeline.txt
  case $s in
    tests) timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1 ;;
    bench) timeout 900 python bench.py > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err ;;
    bench3) timeout 600 python bench.py --workload C3 --no-cpu-baseline > gpurun_out/${TAG}_bench_c3.json 2> gpurun_out/${TAG}_bench_c3.err ;;
    bench5) timeout 600 python bench.py --workload C5 --no-cpu-baseline > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err ;;
    fast) timeout 600 python bench.py --mode fast --no-cpu-baseline > gpurun_out/${TAG}_bench_c4_fast.json 2> gpurun_out/${TAG}_bench_c4_fast.err ;;
    ref) timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err ;;
    launches4) timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
        --csv --log-file gpurun_out/${TAG}_launches_c4.csv python tools/profile_step.py C4 > gpurun_out/${TAG}_launches4.log 2>&1 ;;
    launches5) timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
        --csv --log-file gpurun_out/${TAG}_launches_c5.csv python tools/profile_step.py C5 > gpurun_out/${TAG}_launches5.log 2>&1 ;;
    ncu5) timeout 1200 ncu --set full --clock-control none --import-source on \
        -k regex:"pattern_kernel|emit_kernel|adjacency" -c 4 \
        -o gpurun_out/${TAG}_full_c5 python tools/profile_step.py C5 > gpurun_out/${TAG}_ncu_full5.log 2>&1 ;;
    ncu4) timeout 1200 ncu --set full --clock-control none --import-source on \
        -k regex:"integrate_mesh_kernel|pattern_kernel|emit_kernel" -c 3 \
        -o gpurun_out/${TAG}_full_c4 python tools/profile_step.py C4 > gpurun_out/${TAG}_ncu_full4.log 2>&1 ;;
  esac
done
echo "== done $(date +%T)" >> gpurun_out/${TAG}_timeline.txt
echo done
