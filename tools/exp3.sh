mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/e3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e3_pytest.log
for W in C3 C4 C5; do
  HX_FUSED_ADJACENCY=0 timeout 300 python tools/step_time.py $W >> gpurun_out/e3_steps.txt 2>&1
  timeout 300 python tools/step_time.py $W >> gpurun_out/e3_steps.txt 2>&1
done
echo done
