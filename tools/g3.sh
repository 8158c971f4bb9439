mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python paper_1607_03936_b200/build.py > gpurun_out/g3_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -rf -k "one_step or lumped" > gpurun_out/g3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g3_pytest.log
python tools/k_once.py k_zm=1 zm_zc=8 > gpurun_out/g3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_K2_zm -s 3 -c 1 -o gpurun_out/g3_zm -f python tools/k_once.py k_zm=1 zm_zc=8 > gpurun_out/g3_ncu.log 2>&1
