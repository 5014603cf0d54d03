#!/bin/bash
# ncu --set full of the Thompson-phase kernel with source-level stall sampling (2M trials of CFG5).
# usage: tools/sessions/session_ncu_src.sh <tag> [lib variant]
set -u
TAG=$1; V=${2:-}
OUT=gpurun_out/$TAG; mkdir -p $OUT
[ -n "$V" ] && export ZEUS_SIM_LIB=$PWD/build/libzs_$V.so
timeout -s KILL 800 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -s 1 -c 1 \
  -o $OUT/replay python bench.py --trials ${NCU_TRIALS:-2000000} --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 \
  > $OUT/ncu_bench.json 2> $OUT/ncu.err
echo "ncu rc=$?"
