mkdir -p gpurun_out
for ne in 5 4 8 10; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared --expt-relaxed-constexpr -DA4_NE=$ne -o paper_1607_03936_b200/libwbfbt.so paper_1607_03936_b200/csrc/wbfbt.cu
  echo "NE=$ne" >> gpurun_out/g16_a4.log
  timeout 300 python tools/ab.py C4 2>&1 | head -2 >> gpurun_out/g16_a4.log
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "apply_A" >> gpurun_out/g16_a4.log 2>&1
