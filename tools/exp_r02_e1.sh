mkdir -p gpurun_out
timeout 300 python tools/ke_variants.py C3 > gpurun_out/e1_ke_c3.txt 2>&1
timeout 400 python tools/ke_variants.py C4 > gpurun_out/e1_ke_c4.txt 2>&1
for n in 384 399 400 401; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:emit_kernel \
    --csv --log-file gpurun_out/e1_emit_$n.csv python tools/profile_cube.py $n > /dev/null 2>&1
done
echo done
