"""Builds kernel A/B variants of the same ABI into build/ (experiments; the product
library is paper_2208_06102_b200/libzeus_sim.so)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_06102_b200 import build as B  # noqa: E402

VARIANTS = {
    "u1": ([], []),
    "qc": (["ZS_QCACHE=1"], []),
    "noqc": (["ZS_QCACHE=0"], []),
    "wb": (["ZS_WRITE_BACK=1"], []),
    "diet": (["ZS_DIET=1"], []),
    "nodiet": (["ZS_DIET=0"], []),
    "opc": (["ZS_ONEPASS_CACHE=1"], []),
    "noopc": (["ZS_ONEPASS_CACHE=0"], []),
    "kc": (["ZS_KERNEL_CACHE=1"], []),
    "nowb": (["ZS_WRITE_BACK=0"], []),
    "sall": (["ZS_SCREEN_ALL=1"], []),
    "lred": (["ZS_LANE_RED=1"], []),
    "clk": (["ZS_REGION_CLOCKS=1"], []),
    "minmu": (["ZS_LEAD_MINMU=1"], []),
    "skipstats": (["ZS_SKIP_STATS=1"], []),
    "bskip": (["ZS_BOUND_SKIP=1"], []),
    "b1": (["ZS_BOUND_SKIP=1", "ZS_BSKIP_SLOTS=1"], []),
    "b1l": (["ZS_BOUND_SKIP=1", "ZS_BSKIP_SLOTS=1", "ZS_RUB_LINE=1"], []),
    "b1_6": (["ZS_BOUND_SKIP=1", "ZS_BSKIP_SLOTS=1", "ZS_P2_MIN_BLOCKS=6"], []),
    "b1l_6": (["ZS_BOUND_SKIP=1", "ZS_BSKIP_SLOTS=1", "ZS_RUB_LINE=1", "ZS_P2_MIN_BLOCKS=6"], []),
    "bl": (["ZS_BOUND_SKIP=1", "ZS_RUB_LINE=1"], []),
    "blr": (["ZS_BOUND_SKIP=1", "ZS_RUB_LINE=1", "ZS_REDUX=1"], []),
    "blp": (["ZS_BOUND_SKIP=1", "ZS_RUB_LINE=1", "ZS_SCREEN_PREFETCH=1"], []),
    "blpr": (["ZS_BOUND_SKIP=1", "ZS_RUB_LINE=1", "ZS_SCREEN_PREFETCH=1", "ZS_REDUX=1"], []),
    "ur": (["ZS_REDUX=1"], []),
    "noquad": (["ZS_QUAD_LOOP=0"], []),
    "noslim": (["ZS_SLIM_B=0"], []),
    "noboth": (["ZS_QUAD_LOOP=0", "ZS_SLIM_B=0"], []),
    "slim": (["ZS_SLIM_B=1"], []),
    "slim_b6": (["ZS_SLIM_B=1", "ZS_P2_MIN_BLOCKS=6"], []),
    "b6": (["ZS_P2_MIN_BLOCKS=6"], []),
    "occ20": (["ZS_EXPERIMENT_SMEM_PAD=2500"], []),
    "occ16": (["ZS_EXPERIMENT_SMEM_PAD=12000"], []),
    "quad": (["ZS_QUAD_LOOP=1"], []),
    "quad_r96": (["ZS_QUAD_LOOP=1", "ZS_MAXNREG=96"], []),
    "carve0": (["ZS_DEFAULT_CARVEOUT"], []),
    "mb6": (["ZS_P2_MIN_BLOCKS=6"], []),
    "mb6c0": (["ZS_P2_MIN_BLOCKS=6", "ZS_DEFAULT_CARVEOUT"], []),
    "win512": (["ZS_REGROUP_WINDOW=512"], []),
    "win8k": (["ZS_REGROUP_WINDOW=8192"], []),
    "win1m": (["ZS_REGROUP_WINDOW=1048576"], []),
    "norecip": (["ZS_RECIP_TABLE=0"], []),
    "p2b6": (["ZS_P2_MIN_BLOCKS=6"], []),
    "p2b5": (["ZS_P2_MIN_BLOCKS=5"], []),
    "pipe": (["ZS_PIPELINE=1"], []),
    "hoist": (["ZS_HOIST_REPLICA=1"], []),
    "pipe_hoist": (["ZS_PIPELINE=1", "ZS_HOIST_REPLICA=1"], []),
    "pipe_hoist_r80": (["ZS_PIPELINE=1", "ZS_HOIST_REPLICA=1", "ZS_MAXNREG=80"], []),
    "u1_imm": (["ZS_IMMEDIATE_CONSTANTS"], []),
    "rk": (["ZS_ROUND_KEYS"], []),
    "rk_r88": (["ZS_ROUND_KEYS", "ZS_MAXNREG=88"], []),
    "u2": (["ZS_PAIR_UNROLL=2"], []),
    "u1_r96": (["ZS_MAXNREG=96"], []),
    "u2_r96": (["ZS_PAIR_UNROLL=2", "ZS_MAXNREG=96"], []),
    "u1_r80": (["ZS_MAXNREG=80"], []),
    "u1_r88": (["ZS_MAXNREG=88"], []),
    "u1_r72": (["ZS_MAXNREG=72"], []),
    "u1_r64": (["ZS_MAXNREG=64"], []),
    "u1_r56": (["ZS_MAXNREG=56"], []),
    "u2_r80": (["ZS_PAIR_UNROLL=2", "ZS_MAXNREG=80"], []),
}

if __name__ == "__main__":
    os.makedirs("build", exist_ok=True)
    names = sys.argv[1:] or list(VARIANTS)
    for n in names:
        d, x = VARIANTS[n]
        out = B.build(force=True, out=f"build/libzs_{n}.so", defines=d, extra=x)
        log = open(out + ".ptxas.log").read().split("Compiling entry function")
        for part in log:
            head = part.split("\n")[0]
            if "replay_kernelILb0ELb0E" in head or "replay_kernel_tsILb0ELb0E" in head:
                ph = head.split("ELi")[1][0] if "ELi" in head else "ts"
                print(n, "phase", ph, [l.strip()[-70:] for l in part.splitlines()
                                       if "Used" in l or "spill" in l])
