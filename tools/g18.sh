mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g18_build.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g18_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/g18_smoke.log
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=12 > gpurun_out/g18_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g18_pytest.log
timeout 900 python bench.py > gpurun_out/g18_bench.json 2> gpurun_out/g18_bench.err; echo "bench rc=$?" >> gpurun_out/g18_bench.err
