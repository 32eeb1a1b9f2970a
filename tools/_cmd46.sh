python -m pytest tests -m gpu -q -x > gpurun_out/t46.log 2>&1; tail -2 gpurun_out/t46.log
python bench.py --steps 10 --warmup 3 --no-config2 --no-cir --no-config5 --no-cpu-baseline > gpurun_out/b46.json 2> gpurun_out/b46.err; tail -c 600 gpurun_out/b46.json
for k in k_map_shade k_map_trace; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 6 -o gpurun_out/c2_$k -f python tools/map_time.py > gpurun_out/ncu46_$k.log 2>&1
python tools/ncu_summary.py full gpurun_out/c2_$k.ncu-rep > gpurun_out/c2_${k}_46.txt 2>&1
python tools/ncu_hotlines.py gpurun_out/c2_$k.ncu-rep 40 > gpurun_out/c2_${k}_46_hot.txt 2>&1
done
