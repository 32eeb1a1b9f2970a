#!/bin/bash
# A/B of k_cir_visibility library variants on config 3: tools/vis_ab_run.sh VAR ... (built by build_variants.sh)
L=$PWD/paper_2504_21719_b200/_lib/variants
for v in default "$@" default "$@"; do
  if [ $v = default ]; then unset SBR_LIB_PATH; else export SBR_LIB_PATH=$L/libsbr_$v.so; fi
  echo "$v $(timeout 300 python tools/vis_ab.py --repeat ${VIS_REPEAT:-3} 2>&1 | tail -1)"
done
