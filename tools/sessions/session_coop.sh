set -u
OUT=gpurun_out/r02c; mkdir -p $OUT
ZEUS_SIM_LIB=$PWD/build/libzs_coop.so timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $OUT/pytest_coop.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/pytest_coop.log
AB_TRIALS=10000000 bash tools/ab_session.sh r02c u1 coop
