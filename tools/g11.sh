mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python paper_1607_03936_b200/build.py > gpurun_out/g11_build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_vmg.py -m gpu -q -k restart > gpurun_out/g11_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g11_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/g11_bench.json 2> gpurun_out/g11_bench.err; echo "bench rc=$?" >> gpurun_out/g11_bench.err
timeout 300 python tools/san_case.py small > gpurun_out/g11_san_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python tools/san_case.py small > gpurun_out/g11_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/g11_memcheck.log
