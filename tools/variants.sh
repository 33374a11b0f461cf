#!/bin/bash
# Build libcil.so variants (extra nvcc -D flags) into tools/ubench/var_<name>/ for A/B timing.
# usage: tools/variants.sh name "-DFOO=1" [name2 "-D..."] ...
set -e
cd "$(dirname "$0")/.."
while [ $# -gt 0 ]; do
  name=$1; flags=$2; shift 2
  d=tools/ubench/var_$name/paper_1807_00399_b200
  mkdir -p $d
  cp paper_1807_00399_b200/__init__.py $d/
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
      -Xcompiler -fvisibility=hidden -Iinclude --expt-relaxed-constexpr $flags -shared -o $d/libcil.so \
      paper_1807_00399_b200/csrc/*.cu -lcudart
  echo "built $name ($flags)"
done
