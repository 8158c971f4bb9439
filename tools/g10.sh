mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python paper_1607_03936_b200/build.py > gpurun_out/g10_build.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/g10_bench.json 2> gpurun_out/g10_bench.err; echo "bench rc=$?" >> gpurun_out/g10_bench.err
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/g10_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g10_pytest.log
