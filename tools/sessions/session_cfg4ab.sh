#!/bin/bash
mkdir -p gpurun_out/$1
for v in u1 noquad noslim noboth; do
  ZEUS_SIM_LIB=$PWD/build/libzs_$v.so timeout 300 python bench.py --config cfg4 --layout 2 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/$1/cfg4_$v.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/$1/cfg4_$v.json').read().splitlines()[-1]); print('$v', '%.4g dec/s'%d['value'], 'replay %.3f ms'%d['replay_ms_per_step'])"
done
