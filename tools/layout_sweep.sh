#!/bin/bash
# bench one config under every replay layout
TAG=$1; CFG=$2; shift 2
mkdir -p gpurun_out/$TAG
for lay in 0 1 2 3; do
  timeout 300 python bench.py --config $CFG --layout $lay --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 "$@" > gpurun_out/$TAG/${CFG}_l$lay.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/$TAG/${CFG}_l$lay.json').read().splitlines()[-1]); print('$CFG layout $lay', '%.4g dec/s'%d['value'], 'replay %.3f ms'%d['replay_ms_per_step'], 'launches', d['gpu_launches'])" || tail -2 gpurun_out/$TAG/${CFG}_l$lay.json
done
