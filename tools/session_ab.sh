#!/bin/bash
# GPU parity suite under each variant library, then the A/B bench on CFG5.
# usage: tools/session_ab.sh <tag> <variant...>
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
for v in "$@"; do
  [ "$v" = u1 ] && continue
  ZEUS_SIM_LIB=$PWD/build/libzs_$v.so timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $OUT/pytest_$v.log 2>&1
  echo "$v tests rc=$? $(tail -1 $OUT/pytest_$v.log)"
done
AB_TRIALS=${AB_TRIALS:-10000000} bash tools/ab_session.sh $TAG "$@"
