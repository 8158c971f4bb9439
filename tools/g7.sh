mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python paper_1607_03936_b200/build.py > gpurun_out/g7_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_schur.py -m gpu -q -rf -s --durations=10 > gpurun_out/g7_schur.log 2>&1; echo "schur rc=$?" >> gpurun_out/g7_schur.log
timeout 900 python tools/stokes_exp.py C2 6 20 > gpurun_out/g7_stokes_C2.log 2>&1
timeout 900 python tools/stokes_exp.py C5 20 > gpurun_out/g7_stokes_C5.log 2>&1
