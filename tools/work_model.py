"""Per-primitive instruction counts of the contract, from the sm_100a SASS of
tools/work_probe.cu (straight-line main path: NOPs, slow-path subroutines after
EXIT and the probe's own load/store scaffolding excluded).

Writes tools/work_model.json, used by bench.py to turn the replay's event
counters (normal pairs, normals used, decisions, posterior updates) into
algorithmic lane-instructions per launch.
"""
import json
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
NVCC = "/usr/local/cuda/bin/nvcc"
FP64 = re.compile(r"^(DFMA|DADD|DMUL|DSETP|DMNMX|DSET|MUFU\.(RCP|RSQ)64H|F2F\.F64|I2F\.F64|F2I\.F64|I2F\.S64|DMMA)")
FMA_PIPE = re.compile(r"^(IMAD|IMUL|FFMA|FMUL|FADD|HFMA2|HMUL2|HADD2|IDP)")
ALU_PIPE = re.compile(r"^(IADD3|IADD|LOP3|LOP|SHF(?!L)|SHL|SHR|SEL|FSEL|ISETP|FSETP|PRMT|IMNMX|FMNMX|LEA|IABS|"
                      r"PLOP3|P2R|R2P|SGXT|BMSK|VIADD|VIMNMX|I2IP|F2FP)")
SCAFFOLD = ("LDG", "STG", "LDC", "LDCU", "ULDC", "S2R", "S2UR", "EXIT", "RET", "BRA", "NOP", "CALL",
            "UMOV", "MOV ")  # constant materialisation is hoisted out of the replay loop


def sass(cubin, fn):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-sass", "-fun", fn, cubin], text=True)
    ins = []
    for line in out.splitlines():
        m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(.*?);", line)
        if not m:
            continue
        txt = m.group(1).strip()
        if txt.startswith("@"):
            txt = txt.split(None, 1)[1]
        ins.append(txt)
        if txt.startswith("EXIT") and not m.group(1).strip().startswith("@"):
            break
    return ins


def classify(ins):
    """Lane-instructions by pipe: fp64 (the FP64 unit), fma (IMAD/FFMA: the fma pipe), alu
    (LOP3/IADD3/SHF/SEL/ISETP/...: the alu pipe), other (MUFU, XU, shuffles, shared-memory and
    uniform-datapath ops, moves); total = all of them (issue slots)."""
    body = [i for i in ins if not i.startswith(SCAFFOLD)]
    fp64 = sum(1 for i in body if FP64.match(i))
    fma = sum(1 for i in body if not FP64.match(i) and FMA_PIPE.match(i))
    alu = sum(1 for i in body if not FP64.match(i) and not FMA_PIPE.match(i) and ALU_PIPE.match(i))
    return {"fp64": fp64, "fma": fma, "alu": alu, "other": len(body) - fp64 - fma - alu,
            "total": len(body)}


def main():
    cubin = "/tmp/zs_work_probe.cubin"
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "--fmad=false",
                           "-cubin", "-o", cubin, os.path.join(HERE, "work_probe.cu")])
    names = ["philox", "zlog", "sincospi", "sqrt", "div", "bm", "pair", "theta", "observe", "charge",
             "serial", "curves", "screen", "philox_q", "fpair"]
    model = {n: classify(sass(cubin, f"probe_{n}")) for n in names}
    model["_doc"] = ("lane-instructions per primitive on sm_100a (nvcc 12.9, -O3 --fmad=false), main "
                     "path from tools/work_probe.cu; fp64 = FP64-unit ops (DFMA/DADD/DMUL/DSETP/MUFU.*64H/"
                     "conversions), fma = fma-pipe ops (IMAD*, FFMA), alu = alu-pipe ops (LOP3, IADD3, "
                     "SHF, SEL, ISETP, ...), other = everything else (MUFU, shuffles, uniform ops, moves); "
                     "total = issue slots")
    json.dump(model, open(os.path.join(HERE, "work_model.json"), "w"), indent=1)
    json.dump(model, sys.stdout, indent=1)


if __name__ == "__main__":
    main()
