#!/bin/bash
# A/B: bench the radio map with each libsbr variant (k_map_trace / k_map_shade split)
for v in default "$@"; do
  if [ "$v" = default ]; then unset SBR_LIB_PATH; else export SBR_LIB_PATH=$PWD/paper_2504_21719_b200/_lib/variants/libsbr_$v.so; fi
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-cir 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernels']; print('$v', '%.3e'%d['value'], {n: round(x['ms_per_step'],2) for n,x in k.items()})"
done
