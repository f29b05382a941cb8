mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_distributed.py -x -q > gpurun_out/g15_tests.log 2>&1; echo rc=$? >> gpurun_out/g15_tests.log
for lam in 0 0.5 1 2 4; do
  echo "lambda=$lam" >> gpurun_out/g15_c5.txt
  HX_BALANCE_TOUCH=$lam timeout 600 python tools/shard_rank_time.py C5 8 >> gpurun_out/g15_c5.txt 2>&1
done
for lam in 0 1 2; do
  echo "lambda=$lam" >> gpurun_out/g15_c4.txt
  HX_BALANCE_TOUCH=$lam timeout 900 python tools/shard_rank_time.py C4 8 >> gpurun_out/g15_c4.txt 2>&1
done
