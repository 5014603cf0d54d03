#!/bin/bash
# multi-rank bench path on one GPU (2 ranks share it over gloo) + the reference arm under torchrun
mkdir -p gpurun_out/$1
ZEUS_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --trials 1000000 > gpurun_out/$1/bench_2rank.json 2> gpurun_out/$1/bench_2rank.err; echo "2rank rc=$?"; tail -c 600 gpurun_out/$1/bench_2rank.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 1 --warmup 0 > gpurun_out/$1/ref_2rank.json 2> gpurun_out/$1/ref_2rank.err; echo "ref2 rc=$?"; tail -c 300 gpurun_out/$1/ref_2rank.json
