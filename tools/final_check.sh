NCU=0 bash tools/gpu_check.sh
R=r01
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
python tools/ncu_summary.py launches gpurun_out/launches.csv > gpurun_out/${R}_bench_launches.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cir_visibility -c 1 -o gpurun_out/k_cir_visibility -f python tools/cir_city.py --samples 100000 --repeat 1 > gpurun_out/ncu_k_cir_visibility.log 2>&1
k=k_cir_visibility
python tools/ncu_summary.py full gpurun_out/$k.ncu-rep > gpurun_out/${R}_${k}_ncu_full.txt 2>&1
python tools/ncu_hotlines.py gpurun_out/$k.ncu-rep 40 > gpurun_out/${R}_${k}_hotlines.txt 2>&1
python tools/ncu_summary.py traffic gpurun_out/$k.ncu-rep > gpurun_out/traffic_$k.json 2>&1
timeout 400 python tools/cir_breakdown.py > gpurun_out/cir_breakdown.txt 2>&1
rm -f gpurun_out/launches.csv
echo final done
