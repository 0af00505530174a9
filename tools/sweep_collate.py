"""Collate tools/sweep.sh output into sweep_cfg4.json (+ a markdown table on stdout).

    python tools/sweep_collate.py gpurun_out/sweep
"""
import glob
import json
import os
import sys


def main(d):
    rows = []
    for f in sorted(glob.glob(os.path.join(d, "cfg*_K*_T*.json"))):
        try:
            line = [l for l in open(f) if l.startswith("{")][-1]
            j = json.loads(line)
        except (IndexError, ValueError):
            rows.append({"file": os.path.basename(f), "error": open(f[:-5] + ".err").read()[-300:]})
            continue
        r, c = j["roofline"], j["config"]
        rows.append({"system": c["system"], "noise": c["noise"], "K": c["K"], "T": c["T"],
                     "state_steps_per_s": j["value"], "ms_per_iteration": j["ms_per_step"],
                     "rollout_ms": r["kernel_ms"], "kernel": r["kernel"], "fp32_frac": r["frac"],
                     "hbm_frac": r.get("hbm", {}).get("frac"), "sm_mhz": (j.get("clocks") or {}).get("sm_mhz")})
    json.dump(rows, open(os.path.join(d, "sweep_cfg4.json"), "w"), indent=1)
    ok = [r for r in rows if "error" not in r]
    for noise in ("philox", "hbm"):
        for system in ("cartpole", "quadrotor"):
            pts = {(r["K"], r["T"]): r for r in ok if r["noise"] == noise and r["system"] == system}
            if not pts:
                continue
            Ts = sorted({t for _, t in pts})
            frac = "hbm_frac" if noise == "hbm" else "fp32_frac"
            print(f"\n{system}, {noise} noise: state-steps/s ({'HBM' if noise == 'hbm' else 'FP32'} fraction)\n")
            print("| K \\ T | " + " | ".join(str(t) for t in Ts) + " |")
            print("|---|" + "---|" * len(Ts))
            for K in sorted({k for k, _ in pts}):
                cells = []
                for t in Ts:
                    r = pts.get((K, t))
                    cells.append("—" if r is None else f"{r['state_steps_per_s']:.2e} ({100 * (r[frac] or 0):.0f}%)")
                print(f"| 2^{K.bit_length() - 1} | " + " | ".join(cells) + " |")
    bad = [r for r in rows if "error" in r]
    if bad:
        print("\nfailed points:", ", ".join(r["file"] for r in bad))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sweep")
