#!/bin/bash
# bench lines with and without CUDA-graph runs (zeus_run_opts.graph) for the given configs
# usage: tools/graph_ab.sh <tag> <config...>
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
for c in "$@"; do
  for g in 0 1; do
    timeout 600 python bench.py --config $c --graph $g --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 10 > $OUT/bench_${c}_g$g.json 2> $OUT/bench_${c}_g$g.err
    python -c "import json; d=json.loads(open('$OUT/bench_${c}_g$g.json').read().splitlines()[-1]); print('$c graph=$g', '%.4g dec/s'%d['value'], 'e2e %.4g'%d['e2e']['value'], 'ratio %.2f'%(d['e2e']['value']/d['value']))" || tail -3 $OUT/bench_${c}_g$g.err
  done
done
