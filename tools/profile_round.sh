#!/bin/bash
# ncu evidence for the current build: launch list of one bench run + full captures of
# the hot kernels.  Outputs -> gpurun_out/ (summarise with tools/ncu_summary.py).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
   > gpurun_out/ncu_launches.log 2>&1
for k in k_map_trace k_map_shade; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
     -o gpurun_out/$k -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-cir \
     > gpurun_out/ncu_$k.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cir_visibility -c 1 \
   -o gpurun_out/k_cir_visibility -f python tools/cir_city.py --samples 100000 --repeat 1 \
   > gpurun_out/ncu_k_cir_visibility.log 2>&1
echo profile done
