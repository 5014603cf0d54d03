#!/bin/bash
tools/gpu_session.sh r01f tests
tools/ab_session.sh r01f u1 u2 u1_r96
ZEUS_SIM_LIB=$PWD/build/libzs_u1.so timeout 300 python bench.py --trials 2000000 --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 1 --layout 1 > gpurun_out/r01f/bench_u1_layout1.json 2>&1; tail -c 400 gpurun_out/r01f/bench_u1_layout1.json
tools/gpu_session.sh r01f ncu
