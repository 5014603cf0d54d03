#!/bin/bash
# A/B of the early split (phase A stops each lane at its first pure Thompson decision):
# GPU parity suite under the candidate libraries, then CFG5 / CFG3 / CFG4 bench lines per library.
# usage: tools/session_split_ab.sh <tag> <test-variants> -- <bench-variants>
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
TV=(); while [ $# -gt 0 ] && [ "$1" != "--" ]; do TV+=("$1"); shift; done; shift || true
for v in "${TV[@]}"; do
  ZEUS_SIM_LIB=$PWD/build/libzs_$v.so timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $OUT/pytest_$v.log 2>&1
  echo "$v tests rc=$? $(tail -1 $OUT/pytest_$v.log)"
done
for rep in 1 2; do
for c in ${AB_CONFIGS:-cfg5 cfg3}; do
  for v in "$@"; do
    ZEUS_SIM_LIB=$PWD/build/libzs_$v.so timeout -s KILL 300 python bench.py --config $c ${AB_ARGS:-} --steps ${AB_STEPS:-5} --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/bench_${c}_${v}_$rep.json 2> $OUT/bench_${c}_${v}_$rep.err
    python - "$c $v $rep" "$OUT/bench_${c}_${v}_$rep.json" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(f"{sys.argv[1]:24s} {d['value']:.4g} dec/s  ms {d['ms_per_step']:.2f} frac {d['roofline']['frac']:.3f} clk {d['clocks']['sm_mhz']}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
  done
done
done
