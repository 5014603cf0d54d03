#!/bin/bash
# A/B of the record read cache in the lane-group, concurrent and variant kernels: GPU tests under
# the variant, then the configs those kernels run (CFG1 lane groups, f3 concurrent, f2v variants).
set -u
ZEUS_SIM_LIB=$PWD/build/libzs_kc.so timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for c in cfg1 f3 f2v; do bash tools/sessions/session_occ.sh r02u $c u1 kc; done
