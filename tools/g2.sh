mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python paper_1607_03936_b200/build.py > gpurun_out/g2_build.log 2>&1
timeout 600 python tools/zm_check.py 44 46 64 > gpurun_out/g2_zm.log 2>&1; echo "zm rc=$?" >> gpurun_out/g2_zm.log
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/g2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g2_pytest.log
