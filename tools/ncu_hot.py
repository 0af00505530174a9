"""Hot SASS basic blocks of an ncu report (by executed warp instructions).

    python tools/ncu_hot.py gpurun_out/prof.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys
from collections import Counter


def main(rep, n=25):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[1]
    data = rows[2:]
    iA, iS, iE, iW = (h.index(k) for k in ("Address", "Source", "Instructions Executed",
                                           "Warp Stall Sampling (All Samples)"))
    tot = sum(int(r[iE] or 0) for r in data)
    print("total warp instructions", tot)
    blocks, cur = [], None
    for r in data:
        e = int(r[iE] or 0)
        if cur is None or e != cur[0]:
            cur = [e, 0, r[iA], [], 0]
            blocks.append(cur)
        cur[1] += 1
        src = r[iS].split()
        op = src[1] if src and src[0].startswith("@") and len(src) > 1 else (src[0] if src else "")
        cur[3].append(op.split(".")[0])
        cur[4] += int(r[iW] or 0)
    blocks.sort(key=lambda b: -b[0] * b[1])
    for b in blocks[:n]:
        c = Counter(b[3])
        print(f"{b[0]:>8} x {b[1]:>4} = {b[0]*b[1]:>9} ({100*b[0]*b[1]/tot:4.1f}%) stall {b[4]:>5} {b[2][-6:]} {c.most_common(7)}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
