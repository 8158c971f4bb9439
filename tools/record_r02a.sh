# round-2 profiling: launch list of the bench step and full captures of the dominant kernels,
# each with nvidia-smi clocks sampled while it runs
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python paper_1607_03936_b200/build.py > gpurun_out/g14_build.log 2>&1
Q="--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --comp-reps 3 > gpurun_out/g14_plain.json 2> gpurun_out/g14_plain.err && \
python tools/k_once.py > gpurun_out/g14_kplain.log 2>&1 && {
nvidia-smi $Q --format=csv -lms 200 > gpurun_out/g14_clocks_launches.csv & CP=$!
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/g14_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --comp-reps 3 > gpurun_out/g14_ncu_launch.log 2>&1
kill $CP
nvidia-smi $Q --format=csv -lms 200 > gpurun_out/g14_clocks_k2tma.csv & CP=$!
ncu --set full --clock-control none --import-source on -k regex:k_K2_tma -s 20 -c 1 -o gpurun_out/g14_k2tma -f python tools/k_once.py > gpurun_out/g14_ncu_k.log 2>&1
kill $CP
nvidia-smi $Q --format=csv -lms 200 > gpurun_out/g14_clocks_upd.csv & CP=$!
ncu --set full --clock-control none --import-source on -k regex:k_pcg_upd -s 20 -c 1 -o gpurun_out/g14_upd -f python tools/k_once.py > gpurun_out/g14_ncu_upd.log 2>&1
kill $CP
}
echo done > gpurun_out/g14_done
