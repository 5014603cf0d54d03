#!/bin/bash
# A/B of variant libraries over several configs (short benches), plus the GPU suite on the first.
# usage: tools/sessions/session_cfgab.sh <tag> "<configs>" <variants...>
TAG=$1; CFGS=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
ZEUS_SIM_LIB=$PWD/build/libzs_$1.so timeout -s KILL 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_$1.log 2>&1; echo "pytest[$1] rc=$? $(tail -1 $OUT/pytest_$1.log)"
for c in $CFGS; do
  for v in "$@"; do
    ZEUS_SIM_LIB=$PWD/build/libzs_$v.so timeout -s KILL 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/${c}_$v.json 2> $OUT/${c}_$v.err
    python -c "import json;d=json.loads(open('$OUT/${c}_$v.json').read().splitlines()[-1]);c=d['counters_per_step'];print('%-6s %-6s %.4g dec/s  %.3f ms  bm/dec %.3f'%('$c','$v',d['value'],d['ms_per_step'],c[9]/c[0]))" 2>/dev/null || echo "$c $v FAILED"
  done
done
