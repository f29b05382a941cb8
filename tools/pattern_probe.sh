#!/bin/bash
# ncu launch list of the pattern kernel for the default library and each variant (C4 and C5 cold builds)
for wl in C4 C5; do
for lib in default paper_1501_04784_b200/_lib/variants/*.so; do
  if [ "$lib" = default ]; then unset HEXFEM_B200_LIB; else export HEXFEM_B200_LIB=$lib; fi
  n=$(basename $lib .so)
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:pattern_kernel -c 2 --csv --log-file gpurun_out/pp_${wl}_$n.csv python tools/profile_step.py $wl > /dev/null 2>&1
  echo "== $wl $n"; python tools/launches.py gpurun_out/pp_${wl}_$n.csv | grep pattern
done
done
