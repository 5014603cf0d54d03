#!/bin/bash
# bench line for every config (documentation table), default library
TAG=$1
mkdir -p gpurun_out/$TAG
for c in cfg1 cfg2 cfg3 cfg4 cfg4_38 cfg5 f1 f2 f2v f3; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/$TAG/bench_$c.json 2> gpurun_out/$TAG/bench_$c.err
  python -c "import json; d=json.loads(open('gpurun_out/$TAG/bench_$c.json').read().splitlines()[-1]); print('$c', '%.4g dec/s'%d['value'], 'ms/step %.3f'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], 'frac %.3f'%d['roofline']['frac'], 'launches', d['gpu_launches'], 'cpu %.3g' % d.get('cpu_baseline', {}).get('value', 0))" || tail -3 gpurun_out/$TAG/bench_$c.err
done
