mkdir -p gpurun_out
for W in C3 C4; do timeout 600 python tools/ke_variants.py $W >> gpurun_out/e14_ke.txt 2>&1; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/e14_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e14_pytest.log
echo done
