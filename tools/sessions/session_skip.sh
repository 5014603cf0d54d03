#!/bin/bash
# Bound-skip statistics: counters of the stats variant minus the product build.
OUT=gpurun_out/skip; mkdir -p $OUT
for cfg in cfg5 cfg3 cfg2; do
  for v in u1 skipstats; do
    T=""; [ $cfg = cfg5 ] && T="--trials 1000000"
    ZEUS_SIM_LIB=$PWD/build/libzs_$v.so timeout -s KILL 300 python bench.py --config $cfg $T --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/${cfg}_$v.json 2> $OUT/${cfg}_$v.err
    echo "$cfg $v $(python -c "import json,sys;d=json.loads(open('$OUT/${cfg}_$v.json').read().splitlines()[-1]);print(d['counters_per_step'])")"
  done
done
