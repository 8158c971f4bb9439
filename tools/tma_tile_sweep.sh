mkdir -p gpurun_out
cp paper_1607_03936_b200/libwbfbt.so /tmp/base.so
for v in base tz4m1 tz4m2; do
  if [ $v != base ]; then cp paper_1607_03936_b200/libwbfbt_$v.so paper_1607_03936_b200/libwbfbt.so; else cp /tmp/base.so paper_1607_03936_b200/libwbfbt.so; fi
  touch paper_1607_03936_b200/libwbfbt.so
  echo "== $v" >> gpurun_out/g27_tz.log
  timeout 300 python tools/configs_report.py C2 C3 C5 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print(d['config'], round(d['wbfbt_applies_per_s'],1))
    except Exception: print(l.strip()[:200])" >> gpurun_out/g27_tz.log
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "C2 or C3" 2>&1 | tail -1 >> gpurun_out/g27_tz.log
done
cp /tmp/base.so paper_1607_03936_b200/libwbfbt.so
