#!/bin/bash
# ncu evidence for the current build: launch list of one bench run + full captures of
# the hot kernels.  Outputs -> gpurun_out/ (summarise with tools/ncu_summary.py).
# k_map_trace / k_map_shade: all 12 launches of one radio-map step (segments 0-5 of
# both 2^23-sample chunks), so traffic per launch is the step's mean like `achieved`.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
   > gpurun_out/ncu_launches.log 2>&1
for k in k_map_trace k_map_shade; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 12 \
     -o gpurun_out/$k -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-cir \
     --no-config4 > gpurun_out/ncu_$k.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cir_visibility -c 1 \
   -o gpurun_out/k_cir_visibility -f python tools/cir_city.py --samples 100000 --repeat 1 \
   > gpurun_out/ncu_k_cir_visibility.log 2>&1
echo profile done
# summaries on the box (the .ncu-rep files are too large to bring back together)
R=${ROUND:-r01}
for k in k_map_trace k_map_shade k_cir_visibility; do
  python tools/ncu_summary.py full gpurun_out/$k.ncu-rep > gpurun_out/${R}_${k}_ncu_full.txt 2>&1
  python tools/ncu_hotlines.py gpurun_out/$k.ncu-rep 40 > gpurun_out/${R}_${k}_hotlines.txt 2>&1
  python tools/ncu_summary.py traffic gpurun_out/$k.ncu-rep > gpurun_out/traffic_$k.json 2>&1
done
python tools/ncu_summary.py launches gpurun_out/launches.csv > gpurun_out/${R}_bench_launches.txt
rm -f gpurun_out/k_map_shade.ncu-rep gpurun_out/k_map_trace.ncu-rep gpurun_out/launches.csv
echo summaries done
