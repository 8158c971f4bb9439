# round-2 (second session, final): bench, the ncu launch list of the same bench command and
# full captures of the z-march B / B^T kernels, with nvidia-smi clocks sampled alongside
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python paper_1607_03936_b200/build.py > gpurun_out/g28_build.log 2>&1
Q="--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
timeout 600 python bench.py > gpurun_out/g28_bench.json 2> gpurun_out/g28_bench.err
nvidia-smi $Q --format=csv -lms 200 > gpurun_out/g28_clocks_launches.csv & CP=$!
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/g28_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c4 --comp-reps 3 > gpurun_out/g28_ncu_launch.log 2>&1
kill $CP
nvidia-smi $Q --format=csv -lms 200 > gpurun_out/g28_clocks_zc.csv & CP=$!
timeout 600 ncu --set full --clock-control none --import-source on -k regex:_zc2 -s 2 -c 2 -o gpurun_out/g28_zc -f python tools/zc_once.py 4 > gpurun_out/g28_ncu_zc.log 2>&1
kill $CP
echo done > gpurun_out/g28_done
