#!/bin/bash
# ncu evidence for the config-4 headline (run under gpurun, one GPU):
#   launch list of one whole 1e9-ray map, full captures of the 6 segment
#   launches of k_map_trace and k_map_shade of one 2^24-sample pass,
#   summaries -> gpurun_out/${R}_c4_*.txt and traffic_c4_<kernel>.json
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
R=${ROUND:-r02}
python tools/c4_probe.py > gpurun_out/c4_probe.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
   --log-file gpurun_out/c4_launches.csv python tools/c4_probe.py --full \
   > gpurun_out/ncu_c4_launches.log 2>&1
python tools/ncu_summary.py launches gpurun_out/c4_launches.csv > gpurun_out/${R}_c4_launches.txt
for k in ${KERNELS:-k_map_trace k_map_shade}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 6 \
     -o gpurun_out/c4_$k -f python tools/c4_probe.py > gpurun_out/ncu_c4_$k.log 2>&1
  python tools/ncu_summary.py full gpurun_out/c4_$k.ncu-rep > gpurun_out/${R}_c4_${k}_ncu_full.txt 2>&1
  python tools/ncu_hotlines.py gpurun_out/c4_$k.ncu-rep 40 > gpurun_out/${R}_c4_${k}_hotlines.txt 2>&1
  python tools/ncu_summary.py traffic gpurun_out/c4_$k.ncu-rep > gpurun_out/traffic_c4_$k.json 2>&1
done
rm -f gpurun_out/c4_launches.csv
echo profile_c4 done
