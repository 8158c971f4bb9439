mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python paper_1607_03936_b200/build.py > gpurun_out/g1_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf -x --durations=25 > gpurun_out/g1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g1_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err; echo "bench rc=$?" >> gpurun_out/g1_bench.err
timeout 2400 python tools/parity_report.py --out gpurun_out/parity_r02.json > gpurun_out/g1_parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/g1_parity.log
