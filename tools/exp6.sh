mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/e6_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e6_pytest.log
for W in C3 C4 C5; do timeout 600 python tools/asm_variants.py $W >> gpurun_out/e6_asm.txt 2>&1; done
for W in C3 C4 C5; do timeout 300 python tools/step_time.py $W >> gpurun_out/e6_steps.txt 2>&1; done
echo done
