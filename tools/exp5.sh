mkdir -p gpurun_out
for W in C3 C4; do timeout 600 python tools/ke_variants.py $W >> gpurun_out/e5_ke.txt 2>&1; done
for W in C3 C4 C5; do timeout 300 python tools/step_time.py $W >> gpurun_out/e5_steps.txt 2>&1; done
echo done
