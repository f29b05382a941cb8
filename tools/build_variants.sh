#!/bin/bash
# Build alternate libhexfem_b200.so variants: tools/build_variants.sh name "-DFOO=1" [name "-D..."]...
set -e -o pipefail
cd "$(dirname "$0")/.."
OUT=paper_1501_04784_b200/_lib/variants
rm -rf $OUT; mkdir -p $OUT
while [ $# -gt 1 ]; do
  name=$1; defs=$2; shift 2
  d=/tmp/hxvar_$name; rm -rf $d; mkdir -p $d
  python -c "from paper_1501_04784_b200.build import SOURCES; print(\"\\n\".join(SOURCES))" | xargs -P 8 -I{} \
    nvcc -std=c++17 -O3 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude $defs \
      -gencode arch=compute_100a,code=sm_100a -c paper_1501_04784_b200/csrc/{} -o $d/{}.o
  nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $OUT/$name.so $d/*.o -cudart static
done
ls -la $OUT
