python -m pytest tests/test_gpu_radiomap.py tests/test_gpu_configs.py tests/test_gpu_cir.py tests/test_gpu_edge.py -q -x > gpurun_out/t48.log 2>&1; tail -2 gpurun_out/t48.log
for k in k_map_shade; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -c 6 -o gpurun_out/c2_$k -f python tools/map_time.py > gpurun_out/ncu48_$k.log 2>&1
python tools/ncu_summary.py full gpurun_out/c2_$k.ncu-rep > gpurun_out/c2_${k}_48.txt 2>&1
python tools/ncu_hotlines.py gpurun_out/c2_$k.ncu-rep 60 > gpurun_out/c2_${k}_48_hot.txt 2>&1
done
