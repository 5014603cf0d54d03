#!/bin/bash
tools/gpu_session.sh r01g tests
tools/ab_session.sh r01g u1 u2
ZEUS_SIM_LIB=$PWD/build/libzs_u1.so timeout 300 python bench.py --trials 2000000 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 1 --layout 1 > gpurun_out/r01g/bench_u1_layout1.json 2>&1; python -c "import json; d=json.loads(open('gpurun_out/r01g/bench_u1_layout1.json').read().splitlines()[-1]); print('layout1', d['value'], d['replay_ms_per_step'])"
tools/gpu_session.sh r01g ncu
