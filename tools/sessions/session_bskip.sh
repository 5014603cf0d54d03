#!/bin/bash
OUT=gpurun_out/bskip; mkdir -p $OUT
ZEUS_SIM_LIB=$PWD/build/libzs_bskip.so timeout -s KILL 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_bskip.log 2>&1; echo "pytest rc=$? $(tail -1 $OUT/pytest_bskip.log)"
AB_TRIALS=${AB_TRIALS:-4000000} bash tools/ab_session.sh bskip u1 bskip u1 bskip
