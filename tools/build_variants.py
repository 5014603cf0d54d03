"""Builds kernel A/B variants of the same ABI into build/ (experiments; the product
library is paper_2208_06102_b200/libzeus_sim.so)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_06102_b200 import build as B  # noqa: E402

VARIANTS = {
    "u1": ([], []),
    "bskip": (["ZS_BOUND_SKIP=1"], []),
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
    "p2b6": (["ZS_P2_MIN_BLOCKS=6"], []),
    "p2b5": (["ZS_P2_MIN_BLOCKS=5"], []),
    "u1_imm": (["ZS_IMMEDIATE_CONSTANTS"], []),
    "u1_r96": (["ZS_MAXNREG=96"], []),
    "u1_r80": (["ZS_MAXNREG=80"], []),
    "u1_r88": (["ZS_MAXNREG=88"], []),
    "u1_r72": (["ZS_MAXNREG=72"], []),
    "u1_r64": (["ZS_MAXNREG=64"], []),
    "u1_r56": (["ZS_MAXNREG=56"], []),
    # round 2: the certified-draw Thompson kernel (thompson.cuh)
    "th_mb5": (["ZS_TH_MIN_BLOCKS=5"], []),
    "th_nowide": (["ZS_PHILOX_WIDE=0"], []),
    "th_noprefix": (["ZS_PHILOX_PREFIX=0"], []),
    "th_mb6": (["ZS_TH_MIN_BLOCKS=6"], []),
    "th_mb7": (["ZS_TH_MIN_BLOCKS=7"], []),
    "th_q1": (["ZS_QUAD2=0"], []),
    "hs4": (["ZS_HSLOT_MAX=4"], []),
    "pa_cert": (["ZS_PHASEA_CERT=1"], []),
    "hs64": (["ZS_HSLOT_MAX=64"], []),
    "diag_nohist": (["ZS_DIAG_NOHIST"], []),   # timing diagnostic only: curves wrong
    "th_q2_mb5": (["ZS_TH_MIN_BLOCKS=5"], []),
    "th_mb8": (["ZS_TH_MIN_BLOCKS=8"], []),
    "nosplit": (["ZS_EARLY_SPLIT=0"], []),       # phase A runs every lane to t_split (round-2 r02ao)
    "split": (["ZS_EARLY_SPLIT=1"], []),
    "split_mb5": (["ZS_EARLY_SPLIT=1", "ZS_TH_MIN_BLOCKS=5"], []),
    "split_pack": (["ZS_EARLY_SPLIT=1", "ZS_T0_PACK=1"], []),
    "sl8": (["ZS_SLOT_MAX=8"], []),
    "sl8_hs4": (["ZS_SLOT_MAX=8", "ZS_HSLOT_MAX=4"], []),
    "sl16_hs8": (["ZS_SLOT_MAX=16", "ZS_HSLOT_MAX=8"], []),
    "remat": (["ZS_CURVES_REMAT=1"], []),
    "winpf": (["ZS_WIN_PREFETCH=1"], []),
    "winfit": (["ZS_WIN_POOL_FIT=1"], []),
    "qdesc": (["ZS_QUADS_DESC=1"], []),
    "redpred": (["ZS_RED_PRED=1"], []),
    "rec32": (["ZS_REC32=1"], []),
    "hist32": (["ZS_HIST32=1"], []),
    "actreg": (["ZS_ACT_REG=1"], []),
    "noinit": (["ZS_NOINIT=1"], []),
    "armpack": (["ZS_ARMC_PACK=1"], []),
    "tpb128": (["ZS_TPB_CONST=1"], []),
    "smaxub": (["ZS_SMAX_UB=1"], []),
    "actregA": (["ZS_ACT_REG_A=1"], []),
    "rec32_rp": (["ZS_REC32=1", "ZS_RED_PRED=1"], []),
    "p1b5": (["ZS_P1_MIN_BLOCKS=5"], []),
    "p1b6": (["ZS_P1_MIN_BLOCKS=6"], []),
    "winpf_fit": (["ZS_WIN_PREFETCH=1", "ZS_WIN_POOL_FIT=1"], []),
    "nosplit_mb5": (["ZS_EARLY_SPLIT=0", "ZS_TH_MIN_BLOCKS=5"], []),
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
            if "replay_kernelILb0ELb0E" in head or "thompson_kernelILb0ELb1E" in head:
                ph = head.split("ELi")[1][0] if "ELi" in head else "ts"
                print(n, "phase", ph, [l.strip()[-70:] for l in part.splitlines()
                                       if "Used" in l or "spill" in l])
