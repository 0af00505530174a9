"""Instructions executed and warp-stall samples per CUDA source line of an ncu
report (SASS rows attributed to the source line above them).

    python tools/ncu_lines.py gpurun_out/x.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main(rep, n=40):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    inst, samp, src = defaultdict(int), defaultdict(int), {}
    f, cur = "?", None
    for r in csv.reader(io.StringIO(txt)):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0].isdigit():
            cur = (f, int(r[0]))
            src[cur] = ",".join(r[1:3])[:70]
            continue
        if len(r) > 7 and r[2].startswith("0x") and cur:
            samp[cur] += int(r[4] or 0)
            inst[cur] += int(r[7] or 0)
    ti, ts = sum(inst.values()), sum(samp.values())
    print(f"total instructions {ti}, stall samples {ts}")
    for k in sorted(inst, key=lambda k: -inst[k])[:n]:
        print(f"{100*inst[k]/ti:5.1f}% inst {100*samp[k]/max(ts,1):5.1f}% samp  {k[0]}:{k[1]}  {src.get(k,'')}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
