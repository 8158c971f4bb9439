mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python paper_1607_03936_b200/build.py > gpurun_out/g21_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_mg.py -m gpu -q -rf -s --durations=10 > gpurun_out/g21_mg.log 2>&1; echo "mg rc=$?" >> gpurun_out/g21_mg.log
