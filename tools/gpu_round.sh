#!/bin/bash
# One gpurun call: GPU parity tests, bench lines, launch list and full ncu captures.
# Usage (from the repo root, under gpurun): bash tools/gpu_round.sh TAG [steps...]
TAG=${1:-r01}
shift
STEPS=${*:-"tests bench launches ncu"}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
for s in $STEPS; do
  case $s in
    fp64) timeout 120 ./tools/fp64_peak > gpurun_out/${TAG}_fp64.txt 2>&1 ;;
    tests) timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1 ;;
    bench) timeout 900 python bench.py > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err ;;
    bench3) timeout 600 python bench.py --workload C3 --no-cpu-baseline > gpurun_out/${TAG}_bench_c3.json 2> gpurun_out/${TAG}_bench_c3.err ;;
    bench5) timeout 600 python bench.py --workload C5 --no-cpu-baseline > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err ;;
    ref) timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err ;;
    launches) timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
        --csv --log-file gpurun_out/${TAG}_launches_c3.csv python tools/profile_step.py C3 > gpurun_out/${TAG}_launches.log 2>&1 ;;
    ncu) timeout 1200 ncu --set full --clock-control none --import-source on \
        -k regex:"integrate_mesh_kernel|pattern_kernel|emit_kernel|adjacency_kernel" -c 5 \
        -o gpurun_out/${TAG}_full_c3 python tools/profile_step.py C3 > gpurun_out/${TAG}_ncu_full.log 2>&1 ;;
  esac
done
echo done
