#!/bin/bash
# Build libsbr variants with extra -D flags for A/B timing: tools/build_variants.sh NAME "-DFOO" ...
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_2504_21719_b200/_lib/variants
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -fmad=false \
    -Xcompiler -fPIC -shared --expt-relaxed-constexpr $flags \
    paper_2504_21719_b200/csrc/*.cu -o paper_2504_21719_b200/_lib/variants/libsbr_$name.so &
done
wait
