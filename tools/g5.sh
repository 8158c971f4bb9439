mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python paper_1607_03936_b200/build.py > gpurun_out/g5_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_mg.py -m gpu -q -rf -x -s --durations=10 > gpurun_out/g5_mg.log 2>&1; echo "mg rc=$?" >> gpurun_out/g5_mg.log
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=10 --deselect tests/test_gpu_mg.py > gpurun_out/g5_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g5_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/g5_bench.json 2> gpurun_out/g5_bench.err; echo "bench rc=$?" >> gpurun_out/g5_bench.err
