mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/e1_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e1_smoke.log 2>&1
for W in C3 C4; do for B in 4 3 2; do
HX_KE_BLOCKS_PER_SM=$B timeout 300 python tools/step_time.py $W >> gpurun_out/e1_steps.txt 2>&1
done; done
echo done
