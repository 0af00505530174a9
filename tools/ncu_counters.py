"""Record an ncu capture's per-launch counters in profiles/kernel_counters.json.

    python tools/ncu_counters.py <report.ncu-rep> <workload>/<precision>/<noise>/K=<K> <source label>

Writes dram bytes (read + write), warp instructions (smsp__inst_executed.sum),
the kernel name and duration, stamped with the hash of the CUDA sources the
capture was taken from (bench.kernel_source_hash: bench.py refuses entries
whose stamp differs from the tree it runs in).  Run on the box that took the
capture (the snapshot's sources are the ones that were compiled).
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return int(round(float(v.replace(",", "")) * scale))


def main():
    rep, key, label = sys.argv[1], sys.argv[2], sys.argv[3]
    out_path = Path(sys.argv[4]) if len(sys.argv) > 4 else ROOT / "profiles" / "kernel_counters.json"
    from bench import kernel_source_hash

    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    raw = list(csv.reader(io.StringIO(txt)))
    h, u, v = raw[0], raw[1], raw[2]
    d = {k: (val, unit) for k, unit, val in zip(h, u, v)}
    entry = {
        "kernel": d.get("Kernel Name", ("?", ""))[0],
        "dram_bytes": to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"]),
        "warp_instructions": int(float(d["smsp__inst_executed.sum"][0].replace(",", ""))),
        "duration": " ".join(d["gpu__time_duration.sum"]),
        "src_hash": kernel_source_hash(),
        "source": label,
    }
    try:
        doc = json.loads(out_path.read_text())
    except (OSError, ValueError):
        doc = {"_note": "per-launch ncu counters of the rollout kernel (ncu --set full --clock-control none, one launch): "
                        "dram__bytes_read.sum + dram__bytes_write.sum, smsp__inst_executed.sum; src_hash = "
                        "bench.kernel_source_hash() of the sources the capture was compiled from",
               "captures": {}}
    doc["captures"][key] = entry
    out_path.write_text(json.dumps(doc, indent=1) + "\n")
    print(key, entry)


if __name__ == "__main__":
    main()
