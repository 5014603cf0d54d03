#!/bin/bash
# A/B: CFG5 bench + CFG4 in layouts 0/1/2 for two libraries
OUT=gpurun_out/r02al; mkdir -p $OUT
for v in prev u1; do
  L=$PWD/build/libzs_$v.so
  ZEUS_SIM_LIB=$L timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 1 > $OUT/cfg5_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('$OUT/cfg5_$v.json').read().splitlines()[-1]); print('$v cfg5', '%.4g'%d['value'])"
  for lay in 0 2; do for c in cfg4 cfg4_38; do
    ZEUS_SIM_LIB=$L timeout 300 python bench.py --config $c --layout $lay --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $OUT/${c}_${v}_l$lay.json 2>/dev/null
    python -c "import json; d=json.loads(open('$OUT/${c}_${v}_l$lay.json').read().splitlines()[-1]); print('$v $c layout $lay', '%.4g'%d['value'], 'ms %.3f'%d['ms_per_step'])"
  done; done
done
