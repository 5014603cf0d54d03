#!/bin/bash
# ncu launch lists (gpu__time_duration only) of the CFG5 bench step under each variant library
# usage: tools/session_launches_ab.sh <tag> <variant...>
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
for v in "$@"; do
  ZEUS_SIM_LIB=$PWD/build/libzs_$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_$v.csv python bench.py ${LAUNCH_ARGS:-} --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > $OUT/launches_$v.json 2>&1
  echo "ncu $v rc=$?"
done
