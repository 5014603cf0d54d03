#!/bin/bash
# One gpurun session: smoke, GPU tests, bench, ncu launch list + full capture of the replay kernel.
# usage: tools/gpu_session.sh <tag> [what...]   (what: smoke tests bench launches ncu; default all)
# NCU_KERNEL / NCU_SKIP select the captured kernel (default: the first thompson_kernel launch)
set -u
TAG=${1:-r01}; shift || true
WHAT=${*:-smoke tests bench launches ncu}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
lscpu > $OUT/lscpu.txt 2>&1
for w in $WHAT; do
  case $w in
    smoke) timeout -s KILL 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" ;;
    tests) timeout -s KILL 1500 python -m pytest tests -m gpu -q --maxfail=10 -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "tests rc=$?"; tail -5 $OUT/pytest_gpu.log ;;
    bench) timeout -s KILL 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cat $OUT/bench.json ;;
    launches) timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > $OUT/launches_bench.json 2> $OUT/launches.err; echo "launches rc=$?" ;;
    ncu) timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-thompson_kernel} -s ${NCU_SKIP:-0} -c 1 -o $OUT/replay python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 1 > $OUT/ncu_bench.json 2> $OUT/ncu.err; echo "ncu rc=$?" ;;
  esac
done
