#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, then the ncu launch list of the same bench command.
# usage: tools/gpu_round.sh <tag> [pytest-args...]
TAG=${1:-r}; shift
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -rf "$@" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
