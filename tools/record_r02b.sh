# round-2 (second session) record: bench, per-config throughput, C4 parity with the fused
# k = 4 Poisson kernel, the C4 launch list and a full capture of k_K4_fused, with nvidia-smi
# clocks sampled alongside every ncu run
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python paper_1607_03936_b200/build.py > gpurun_out/g15_build.log 2>&1
Q="--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
timeout 600 python bench.py > gpurun_out/g15_bench.json 2> gpurun_out/g15_bench.err
timeout 600 python tools/configs_report.py > gpurun_out/g15_configs.jsonl 2> gpurun_out/g15_configs.err
timeout 1200 python tools/parity_report.py --configs C4 --out gpurun_out/g15_parity_C4.json > gpurun_out/g15_parity.log 2>&1
nvidia-smi $Q --format=csv -lms 200 > gpurun_out/g15_clocks_launches.csv & CP=$!
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/g15_launches_C4.csv python tools/configs_report.py C4 > gpurun_out/g15_ncu_launch.log 2>&1
kill $CP
nvidia-smi $Q --format=csv -lms 200 > gpurun_out/g15_clocks_k4.csv & CP=$!
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_K4_fused -s 4 -c 1 -o gpurun_out/g15_k4 -f python tools/k4_once.py 1 > gpurun_out/g15_ncu_k4.log 2>&1
kill $CP
nvidia-smi $Q --format=csv -lms 200 > gpurun_out/g15_clocks_bt4.csv & CP=$!
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_BT4_tile -c 1 -o gpurun_out/g15_bt4 -f python tools/k4_bbt.py > gpurun_out/g15_ncu_bt4.log 2>&1
kill $CP
echo done > gpurun_out/g15_done
