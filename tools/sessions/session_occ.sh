#!/bin/bash
# Occupancy lever probe: the same kernel under register caps, on a config whose shared memory
# does not limit residency (CFG3, B <= 9) and on CFG5.  usage: tools/sessions/session_occ.sh <tag> <config> <variant...>
set -u
TAG=$1; CFG=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
for v in "$@"; do
  ZEUS_SIM_LIB=$PWD/build/libzs_$v.so timeout -s KILL 300 python bench.py --config $CFG ${TRIALS:+--trials $TRIALS} --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 1 > $OUT/bench_${CFG}_$v.json 2> $OUT/bench_${CFG}_$v.err
  python - "$v" "$OUT/bench_${CFG}_$v.json" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(f"{sys.argv[1]:10s} {d['value']:.4g} dec/s  replay {d['replay_ms_per_step']:.2f} ms  frac {d['roofline']['frac']:.3f} clk {d['clocks']['sm_mhz']}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
