#!/bin/bash
# quick A/B loop: GPU tests (optional), CFG5 bench, a few latency configs
TAG=${1:-quick}; shift
WHAT=${*:-tests bench}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
for w in $WHAT; do
  case $w in
    tests) timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --maxfail=5 > $OUT/pytest_gpu.log 2>&1; echo "tests rc=$?"; tail -8 $OUT/pytest_gpu.log ;;
    bench) timeout -s KILL 900 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; python -c "import json; d=json.loads(open('$OUT/bench.json').read().splitlines()[-1]); print('cfg5 %.4g dec/s ms %.2f frac %.3f e2e %.4g'%(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value']))" || tail -5 $OUT/bench.err ;;
    lat) for c in cfg2 f1 f3 cfg3 cfg4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err; python -c "import json; d=json.loads(open('$OUT/bench_$c.json').read().splitlines()[-1]); print('$c', '%.4g dec/s'%d['value'], 'ms/step %.3f'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], 'ratio %.2f'%(d['e2e']['value']/d['value']))" || tail -3 $OUT/bench_$c.err; done ;;
  esac
done
