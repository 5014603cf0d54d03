#!/bin/bash
# GPU parity suite against one variant library, then an A/B bench of variants.
# usage: tools/sessions/session_var.sh <tag> <variant-under-test> <ab variants...>
TAG=$1; V=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
ZEUS_SIM_LIB=$PWD/build/libzs_$V.so timeout -s KILL 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_$V.log 2>&1; echo "pytest[$V] rc=$? $(tail -1 $OUT/pytest_$V.log)"
AB_TRIALS=${AB_TRIALS:-4000000} bash tools/ab_session.sh $TAG "$@" | grep -v smoke
for v in "$@"; do python -c "import json;d=json.loads(open('$OUT/bench_$v.json').read().splitlines()[-1]);c=d['counters_per_step'];print('$v', 'bm/dec %.3f'%(c[9]/c[0]), 'screened/dec %.3f'%(c[11]/c[0]))"; done
