#!/bin/bash
OUT=gpurun_out/clk; mkdir -p $OUT
ZEUS_SIM_LIB=$PWD/build/libzs_clk.so timeout -s KILL 300 python bench.py --trials 4000000 --steps 1 --warmup 2 --no-cpu-baseline --e2e-steps 1 > $OUT/bench_clk.json 2> $OUT/bench_clk.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/clk/bench_clk.json").read().splitlines()[-1])
c = d["counters_per_step"]
names = ["loop top", "leader", "screen", "residual", "step3/4", "curves", "observe"]
tot = sum(c[4:11])
for n, v in zip(names, c[4:11]):
    print(f"{n:10s} {100 * v / tot:5.1f}%  {v / c[0]:8.1f} cyc/decision(lane-summed)")
print("value", d["value"])
PY
