#!/bin/bash
# Layout check of the latency-bound configs on the current build: auto (0), one pass (1),
# two phases (2), lane groups (3).   usage: tools/sessions/session_layouts2.sh <tag>
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
for c in cfg2 f1 f2 cfg4 cfg1; do
  for l in 0 1 2 3; do
    timeout 300 python bench.py --config $c --layout $l --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/bench_${c}_l$l.json 2> $OUT/bench_${c}_l$l.err
    python -c "import json; d=json.loads(open('$OUT/bench_${c}_l$l.json').read().splitlines()[-1]); print('$c layout $l', '%.4g'%d['value'], 'ms %.3f'%d['ms_per_step'])" 2>/dev/null || echo "$c layout $l failed"
  done
done
