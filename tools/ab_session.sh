#!/bin/bash
# Kernel A/B on one GPU: parity smoke + short bench per variant library in build/.
# usage: tools/ab_session.sh <tag> <variant...>
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
for v in "$@"; do
  LIB=build/libzs_$v.so
  ZEUS_SIM_LIB=$PWD/$LIB timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$v.log 2>&1
  echo "$v smoke rc=$? $(tail -1 $OUT/smoke_$v.log)"
  ZEUS_SIM_LIB=$PWD/$LIB timeout -s KILL 300 python bench.py --trials ${AB_TRIALS:-2000000} --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 1 > $OUT/bench_$v.json 2> $OUT/bench_$v.err
  python - "$v" "$OUT/bench_$v.json" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    r = d["roofline"]
    c = d["counters_per_step"]
    fb = c[13] / max(1, c[12] + c[13]) if len(c) > 13 else float("nan")
    print(f"{sys.argv[1]:10s} {d['value']:.4g} dec/s  replay {d['replay_ms_per_step']:.1f} ms  frac {r['frac']:.3f} fallback {fb:.2e} clk {d['clocks']['sm_mhz']}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
