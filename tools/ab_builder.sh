#!/bin/bash
# radio map (canyon) + CIR (city) with each BVH builder
for b in ploc lbvh; do
  export SBR_BVH_BUILDER=$b
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-config4 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernels']; print('$b', 'map %.3e rb/s'%d['value'], {n: round(x['ms_per_step'],2) for n,x in k.items()}, 'cir ms %.1f'%d['cir']['ms_per_solve'], d['cir']['kernel_ms_per_solve'], 'paths', d['cir']['paths'])"
done
