#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, the ncu launch list of the same bench
# command, then one full ncu capture of the fused K kernel.
# usage: tools/gpu_round.sh <tag> [pytest-args...]
TAG=${1:-r}; shift
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -rf "$@" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; rc=$?
echo "bench rc=$rc" >> gpurun_out/${TAG}_bench.err
if [ $rc -eq 0 ]; then
  timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 3000 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 > gpurun_out/${TAG}_ncu_launch.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_K2_tma -s 40 -c 1 \
    -o gpurun_out/${TAG}_k2tma -f python tools/tma_check.py C5 > gpurun_out/${TAG}_ncu_full.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_A_tile -s 3 -c 1 --cache-control all \
    -o gpurun_out/${TAG}_atile -f python bench.py --steps 3 --warmup 3 > gpurun_out/${TAG}_ncu_a.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg_upd -s 40 -c 2 \
    -o gpurun_out/${TAG}_upd -f python tools/tma_check.py C5 > gpurun_out/${TAG}_ncu_upd.log 2>&1
fi
