#!/usr/bin/env python
"""Instruction mix of a kernel's basic blocks, grouped by the B200 pipe that
issues them, from `cuobjdump -sass` (no GPU needed).

  python tools/sass_mix.py build/sys_cartpole.o <mangled-name-substring> [--top 3]

Pipe costs measured on the B200 (scratch microbenchmark, warp-instructions per
cycle per SM sub-partition): FFMA/FMUL/FADD 1.0, FFMA2 0.5, IMAD 0.5,
LOP3/IADD3/SHF 0.5, MUFU 0.125.  The per-block estimate `cyc` is the busiest of
issue (1/instr), fma-pipe and alu-pipe cycles, i.e. the block's lower bound
on one SMSP per warp pass.
"""
import re
import subprocess
import sys
from collections import Counter

FMA_FULL = ("FFMA", "FMUL", "FADD", "FSEL", "FSET", "FMNMX", "HFMA2")
FMA_HALF = ("IMAD", "FFMA2", "FMUL2", "FADD2", "I2F", "F2I", "I2FP", "F2IP")
ALU_HALF = ("LOP3", "IADD3", "SHF", "ISETP", "FSETP", "SEL", "LEA", "PRMT", "IABS", "IMNMX", "VIADD", "PLOP3", "P2R", "R2P", "IADD", "FLO", "POPC", "BMSK", "SGXT")
MUFU = ("MUFU",)
MEM = ("LDS", "STS", "LDG", "STG", "LD", "ST", "LDC", "LDSM", "ATOM", "RED", "SHFL")


def klass(op):
    base = op.split(".")[0]
    if base in ("FFMA2", "FMUL2", "FADD2"):
        return "fma2"
    if base in FMA_FULL:
        return "fma"
    if base in FMA_HALF:
        return "imad"
    if base in ALU_HALF:
        return "alu"
    if base in MUFU:
        return "mufu"
    if base in MEM:
        return "mem"
    if base.startswith("U") or base in ("S2UR", "R2UR", "LDCU"):
        return "uniform"
    return "other:" + base


def blocks(sass):
    cur, out, label = [], [], "entry"
    for line in sass.splitlines():
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        lab = re.match(r"\.(L_x_\d+):", line.strip())
        if lab:
            if cur:
                out.append((label, cur))
            cur, label = [], lab.group(1)
            continue
        if not m:
            continue
        ins = m.group(2).strip()
        ins = re.sub(r"^@!?U?P\w+\s+", "", ins)
        op = ins.split()[0]
        cur.append(op)
        if op.startswith("BRA") or op.startswith("EXIT"):
            out.append((label, cur))
            cur, label = [], label + "+"
    if cur:
        out.append((label, cur))
    return out


def main():
    obj, name = sys.argv[1], sys.argv[2]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 3
    sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)
    f = [x for x in funcs if x.split("\n", 1)[0].strip().endswith(name) or name in x.split("\n", 1)[0]]
    if not f:
        sys.exit("no function matching " + name)
    body = f[0]
    print(body.split("\n", 1)[0].strip())
    bl = sorted(blocks(body), key=lambda b: -len(b[1]))[:top]
    for label, ops in bl:
        c = Counter(klass(o) for o in ops)
        n = len(ops)
        fma_cyc = c["fma"] + 2 * (c["imad"] + c["fma2"])
        alu_cyc = 2 * c["alu"]
        print(f"{label}: {n} instr  fma {c['fma']} fma2 {c['fma2']} imad/cvt {c['imad']} alu {c['alu']} "
              f"mufu {c['mufu']} mem {c['mem']} uniform {c['uniform']}  | issue {n} fma-pipe {fma_cyc} "
              f"alu-pipe {alu_cyc} mufu-pipe {8 * c['mufu']}")
        other = {k: v for k, v in c.items() if k.startswith("other")}
        if other:
            print("   other:", other)
        if "-v" in sys.argv:
            print("   ", Counter(ops).most_common(40))


if __name__ == "__main__":
    main()
