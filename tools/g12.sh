mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python paper_1607_03936_b200/build.py > gpurun_out/g12_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_mg.py tests/test_gpu_vmg.py tests/test_gpu_schur.py -m gpu -q -rf -s --durations=8 > gpurun_out/g12_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g12_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/g12_bench.json 2> gpurun_out/g12_bench.err; echo "bench rc=$?" >> gpurun_out/g12_bench.err
