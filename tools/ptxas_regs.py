"""Registers / spills per kernel from the build's ptxas logs (make writes build/*.ptxas.log).

    python tools/ptxas_regs.py [filter]
"""
import glob
import re
import subprocess
import sys


def main(flt=""):
    for log in sorted(glob.glob("build/*.ptxas.log")):
        name = None
        spill = ""
        for ln in open(log):
            m = re.search(r"Compiling entry function '([^']+)'", ln)
            if m:
                name = m.group(1)
                continue
            m = re.search(r"(\d+) bytes spill stores", ln)
            if m:
                spill = m.group(1)
            m = re.search(r"Used (\d+) registers", ln)
            if m and name:
                dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
                dem = re.sub(r"jm::|System<|CostDiagQuadratic|RolloutArgs<[a-z]+>", "", dem)
                if flt in dem:
                    print(f"{m.group(1):>4} regs  spill {spill:>3}  {dem[:110]}")
                name = None


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "")
