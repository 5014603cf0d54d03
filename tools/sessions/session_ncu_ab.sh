#!/bin/bash
# ncu --set full of the Thompson-phase kernel for each variant library in build/
# usage: tools/sessions/session_ncu_ab.sh <tag> <variant...>
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
for v in "$@"; do
  ZEUS_SIM_LIB=$PWD/build/libzs_$v.so timeout -s KILL 900 ncu --set full --clock-control none --import-source on \
    -k regex:replay_kernel -s 1 -c 1 -o $OUT/replay_$v python bench.py --trials ${NCU_TRIALS:-2000000} --steps 1 --warmup 0 \
    --no-cpu-baseline --e2e-steps 1 > $OUT/ncu_$v.json 2> $OUT/ncu_$v.err; echo "$v ncu rc=$?"
done
