"""Top SASS lines of an ncu report by warp-stall samples, with the source line they map to.

    python tools/ncu_stalls.py gpurun_out/prof.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys


def main(rep, n=30):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[1]
    data = rows[2:]
    iA, iS, iW = (h.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)"))
    tot = sum(int(r[iW] or 0) for r in data)
    print("total stall samples", tot)
    top = sorted(data, key=lambda r: -int(r[iW] or 0))[:n]
    for r in top:
        print(f"{int(r[iW] or 0):>6} ({100*int(r[iW] or 0)/max(tot,1):4.1f}%) {r[iA][-6:]} {r[iS].strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
