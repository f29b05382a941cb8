mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"integrate_mesh_kernel|pattern_kernel|emit_kernel" -c 3 \
  -o gpurun_out/e4_full_c3 python tools/profile_step.py C3 > gpurun_out/e4_ncu.log 2>&1
echo done
