mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python paper_1607_03936_b200/build.py > gpurun_out/g6_build.log 2>&1
timeout 3000 python tools/parity_report.py --out gpurun_out/parity_r02.json > gpurun_out/g6_parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/g6_parity.log
