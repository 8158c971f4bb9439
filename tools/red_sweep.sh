#!/bin/bash
# PCG vector-kernel grid (RED_MULT blocks per SM): per-iteration time at C5
for r in ${RED_MULTS:-2 4 8}; do
  python -c "
import sys; sys.path.insert(0,'paper_1607_03936_b200'); import build; build.FLAGS += ['-DRED_MULT=$r']; build.build(force=True)" > /dev/null 2>&1
  echo "RED_MULT=$r"; timeout 300 python tools/opt_ab.py C5 "kz=0" 2>&1 | tail -1
done
