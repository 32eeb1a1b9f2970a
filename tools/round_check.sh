#!/bin/bash
# One gpurun call for the round's evidence (run from the repo root on the box):
#   GPU tests, smoke, bench (both arms), config-4 / config-3 / config-2 ncu captures.
# Outputs in gpurun_out/ (copy the summaries into profiles/).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
R=${ROUND:-r02}
if [ "${SKIP_TESTS:-0}" != 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/${R}_pytest_gpu.log 2>&1
  tail -3 gpurun_out/${R}_pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1
  tail -1 gpurun_out/${R}_smoke.log
fi
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
tail -c 300 gpurun_out/${R}_bench.json
if [ "${SKIP_REF:-0}" != 1 ]; then
  timeout 1200 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${R}_bench_ref.json 2> gpurun_out/${R}_bench_ref.err
  tail -c 300 gpurun_out/${R}_bench_ref.json
fi
if [ "${SKIP_NCU:-0}" != 1 ]; then
  bash tools/profile_c4.sh
  # config-3 visibility and config-2 shade/trace full captures
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cir_visibility -c 1 \
     -o gpurun_out/c3_k_cir_visibility -f python tools/cir_city.py --samples 1000000 --repeat 1 \
     > gpurun_out/ncu_c3_vis.log 2>&1
  k=k_cir_visibility
  python tools/ncu_summary.py full gpurun_out/c3_$k.ncu-rep > gpurun_out/${R}_c3_${k}_ncu_full.txt 2>&1
  python tools/ncu_hotlines.py gpurun_out/c3_$k.ncu-rep 40 > gpurun_out/${R}_c3_${k}_hotlines.txt 2>&1
  python tools/ncu_summary.py traffic gpurun_out/c3_$k.ncu-rep > gpurun_out/traffic_c3_$k.json 2>&1
  for k in k_map_trace k_map_shade; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 6 \
       -o gpurun_out/c2_$k -f python tools/map_time.py > gpurun_out/ncu_c2_$k.log 2>&1
    python tools/ncu_summary.py full gpurun_out/c2_$k.ncu-rep > gpurun_out/${R}_c2_${k}_ncu_full.txt 2>&1
    python tools/ncu_summary.py traffic gpurun_out/c2_$k.ncu-rep > gpurun_out/traffic_c2_$k.json 2>&1
  done
  rm -f gpurun_out/c2_*.ncu-rep gpurun_out/c4_*.ncu-rep
fi
echo round_check done
