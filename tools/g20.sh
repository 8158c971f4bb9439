mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python paper_1607_03936_b200/build.py > gpurun_out/g20_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_api.py -m gpu -q -rf -k "failure or ragged" > gpurun_out/g20_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g20_pytest.log
timeout 3000 python tools/mg_report.py --out gpurun_out/mg_stokes_r02.json > gpurun_out/g20_mg.log 2>&1; echo "mg rc=$?" >> gpurun_out/g20_mg.log
