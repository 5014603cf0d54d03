#!/bin/bash
# round 2, first session: build, smoke, GPU tests, peaks, CFG5 bench, the latency configs' e2e
TAG=${1:-r02a}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout -s KILL 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log
timeout -s KILL 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "tests rc=$?"; tail -5 $OUT/pytest_gpu.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peaks tools/peaks.cu && /tmp/peaks > $OUT/peaks.json; cat $OUT/peaks.json
timeout -s KILL 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cat $OUT/bench.json | head -c 3000; echo
for c in cfg2 f1 f3 cfg1 cfg4; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  python -c "import json; d=json.loads(open('$OUT/bench_$c.json').read().splitlines()[-1]); print('$c', '%.4g dec/s'%d['value'], 'ms/step %.3f'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], 'ratio %.2f'%(d['e2e']['value']/d['value']))" || tail -3 $OUT/bench_$c.err
done
