#!/bin/bash
# k_K2_ws: role probes, then per-iteration times (plain build), producer warps from WS_PWS
set -x
for pw in ${WS_PWS:-4}; do
  WS_FLAGS="-DWS_PW=$pw" timeout 300 python tools/wsphase.py 2>&1 | grep -v warning | tail -9
  python -c "
import sys; sys.path.insert(0,'paper_1607_03936_b200'); import build; build.FLAGS += ['-DWS_PW=$pw']; build.build(force=True)" > /dev/null 2>&1
  timeout 300 python -m pytest tests/test_gpu_api.py -q -x -k "ragged" 2>&1 | tail -1
  timeout 300 python tools/opt_ab.py C5 "k_ws=0,kz=0" "k_ws=1,kz=0" "k_ws=1,kz=1" 2>&1 | tail -3
done
