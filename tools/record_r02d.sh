# round-2 final session: bench, the reference arm, the ncu launch list of the same bench command and
# full captures of k_K2_tma / k_pcg_upd / k_A_tile, with nvidia-smi clocks sampled alongside
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
Q="--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
timeout 600 python bench.py > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err; echo "bench rc=$?" >> gpurun_out/r02d_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02d_bench_ref.json 2> gpurun_out/r02d_bench_ref.err
nvidia-smi $Q --format=csv -lms 200 > gpurun_out/r02d_clocks_launches.csv & CP=$!
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r02d_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c4 --comp-reps 3 > gpurun_out/r02d_ncu_launch.log 2>&1
kill $CP
nvidia-smi $Q --format=csv -lms 200 > gpurun_out/r02d_clocks_ncu.csv & CP=$!
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_K2_tma -s 40 -c 1 -o gpurun_out/r02d_k2tma -f python tools/tma_check.py C5 > gpurun_out/r02d_ncu_k.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pcg_upd -s 40 -c 2 -o gpurun_out/r02d_upd -f python tools/tma_check.py C5 > gpurun_out/r02d_ncu_upd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_A_tile -s 3 -c 1 --cache-control all -o gpurun_out/r02d_atile -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c4 --comp-reps 3 > gpurun_out/r02d_ncu_a.log 2>&1
kill $CP
python tools/configs_report.py > gpurun_out/r02d_configs.jsonl 2> gpurun_out/r02d_configs.err
echo done > gpurun_out/r02d_done
