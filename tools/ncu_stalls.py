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


def block_reasons(rep, addr_suffix, n_instr):
    """Stall-reason totals over the n_instr SASS lines starting at the address ending in addr_suffix."""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[1]
    data = rows[2:]
    iA = h.index("Address")
    cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    start = [i for i, r in enumerate(data) if r[iA].endswith(addr_suffix)][0]
    tot = {c: 0 for c in cols}
    for r in data[start:start + n_instr]:
        for c in cols:
            tot[c] += int(r[h.index(c)] or 0)
    s = sum(tot.values()) or 1
    return sorted(((v / s, c) for c, v in tot.items() if v), reverse=True)
