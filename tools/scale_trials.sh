#!/bin/bash
# per-decision time vs trials (and layout) for the default library
TAG=$1; shift
mkdir -p gpurun_out/$TAG
for spec in "$@"; do
  n=${spec%:*}; lay=${spec#*:}
  timeout 300 python bench.py --trials $n --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 1 --layout $lay > gpurun_out/$TAG/scale_${n}_${lay}.json 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/$TAG/scale_${n}_${lay}.json').read().splitlines()[-1]); print('$n layout $lay', '%.4g dec/s'%d['value'], '%.2f ps/dec'%(1e12*d['replay_ms_per_step']/1e3/($n*1000)))"
done
