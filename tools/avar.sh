#!/bin/bash
# A tile-shape sweep: rebuild with -DA_TX/-DA_TY/-DA_TZ/-DA_MINB and time the A pair (ncu launch list)
# usage: tools/avar.sh TAG "TX TY TZ MINB" ...
TAG=$1; shift
for v in "$@"; do
  set -- $v
  python -c "
import sys; sys.path.insert(0,'paper_1607_03936_b200'); import build
build.FLAGS += ['-DA_TX=$1', '-DA_TY=$2', '-DA_TZ=$3', '-DA_MINB=$4']; build.build(force=True)" > /dev/null 2>&1
  echo "== tile $1x$2x$3, $4 CTAs/SM"
  bash tools/atime.sh ${TAG}_$1$2$3
done
python -c "
import sys; sys.path.insert(0,'paper_1607_03936_b200'); import build; build.build(force=True)" > /dev/null 2>&1
