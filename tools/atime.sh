#!/bin/bash
# per-kernel durations of the A pair (ncu launch list, cold caches) over tools/ab.py's 21 applies
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_A_ -c 42 --csv \
  --log-file gpurun_out/${1:-a}_atime.csv python tools/ab.py C5 > gpurun_out/${1:-a}_ab.log 2>&1
python tools/atime_parse.py gpurun_out/${1:-a}_atime.csv
