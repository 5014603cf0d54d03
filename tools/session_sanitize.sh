#!/bin/bash
# compute-sanitizer over small runs of every kernel family: memcheck (out-of-bounds / misaligned
# accesses), racecheck (shared-memory hazards), synccheck.  usage: tools/session_sanitize.sh <tag>
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
cat > /tmp/zs_small.py <<'PY'
import sys
sys.path.insert(0, ".")
from paper_2208_06102_b200 import synth
from paper_2208_06102_b200.zeus_sim import Simulation
# one-cell (RK kernels, two phases), multi-cell, windowed one pass, lane groups, baselines,
# ablations, variant readings, concurrent submissions
# (layout 4: the early split, thompson_kernel<..., EARLY>; draw 0: the certified Thompson kernel; 1: the exact-screen phase B; 2: certified, all fallbacks)
runs = [("cfg5", 600, 0, 0), ("cfg5", 300, 2, 1), ("cfg5", 300, 2, 2), ("cfg5", 400, 4, 0), ("cfg5", 300, 4, 2),
        ("cfg3", 300, 0, 0), ("cfg3", 300, 4, 0), ("cfg4", 400, 4, 0),
        ("cfg4", 400, 0, 0), ("cfg4", 300, 0, 2), ("cfg4_38", 500, 0, 0), ("cfg1", 100, 3, 0), ("f1", 200, 0, 0), ("f2", 200, 0, 0),
        ("f2v", 200, 0, 0), ("f3", 200, 0, 0)]
for name, trials, layout, draw in runs:
    for job in synth.config(name, trials=trials)[:2]:
        R = min(job.recurrences, 120)
        sim = Simulation(job.workload, job.cells, job.trials, R, layout=layout, draw=draw).load_profile()
        sim.run().results()
        sim.close()
    print("ok", name, flush=True)
PY
for tool in memcheck racecheck synccheck; do
  timeout -s KILL 1200 compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/zs_small.py > $OUT/sanitizer_$tool.log 2>&1
  echo "$tool rc=$? $(grep -c '^ok' $OUT/sanitizer_$tool.log) runs ok; $(grep -m1 'ERROR SUMMARY' $OUT/sanitizer_$tool.log)"
done
