#!/bin/bash
# GPU suite, then every config with and without the CUDA-graph run.
OUT=gpurun_out/graph; mkdir -p $OUT
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $OUT/pytest.log)"
for c in ${CFGS:-cfg1 cfg2 cfg4 cfg4_38 f1 f2 f2v f3 cfg3 cfg5}; do
  for g in 0 1; do
    timeout -s KILL 300 python bench.py --config $c --graph $g --steps 10 --warmup 3 --no-cpu-baseline > $OUT/${c}_g$g.json 2> $OUT/${c}_g$g.err
    python -c "import json;d=json.loads(open('$OUT/${c}_g$g.json').read().splitlines()[-1]);print('%-8s graph=$g %.4g dec/s  %.4f ms  e2e %.4g'%('$c',d['value'],d['ms_per_step'],d['e2e']['value']))" 2>/dev/null || echo "$c g$g FAILED"
  done
done
