"""One rank of tests/test_distributed.py (gloo, CPU).  Prints a JSON line."""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import mppi as om  # noqa: E402
from oracle import philox_stream as ps  # noqa: E402
from paper_1807_06108_b200 import distributed as jd  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from conftest import load_golden, oracle_spec

    if os.environ.get("JM_AGREE"):  # transport agreement: rank 1 reports a failed setup
        ok = jd.agree(rank != 1)
        print(json.dumps({"rank": rank, "agree": ok, "all_ok": jd.agree(True)}))
        dist.destroy_process_group()
        return
    g = load_golden(os.environ["JM_CASE"])
    spec = oracle_spec(g["spec"])
    if os.environ.get("JM_K_TOTAL"):  # strong scaling: a fixed global K split over the ranks (ragged)
        off, cnt = jd.shard_for("strong", int(os.environ["JM_K_TOTAL"]), rank, world)
    else:
        off, cnt = jd.shard_for("weak", int(os.environ["JM_K_LOCAL"]), rank, world)
    Ld = np.linalg.cholesky(spec.c * spec.sigma_d)
    Lj = np.linalg.cholesky(spec.sigma_j)
    jthr = ps.jump_threshold(spec.nu * spec.dt) if spec.jump_enabled else 0
    noise = ps.device_noise(7, 3, cnt, spec.T, spec.m, spec.q, Ld, Lj, spec.mark_mean, jthr,
                            jump_channel=spec.jump_channel, sample_offset=off)
    spec.K = cnt
    out = om.mppi_iteration_oracle(spec, g["x0"], g["u_nom"], noise)
    rec = torch.from_numpy(om.partial_record(out["costs"], noise[3], spec.lam))
    gathered = jd.exchange_records(rec).numpy()
    u_new, rho, ess = om.combine_records(gathered, spec.lam, spec.dt, g["u_nom"])
    print(json.dumps({"rank": rank, "u_new": u_new.tolist(), "rho": rho, "ess": ess,
                      "gathered_rho": gathered[:, 0].tolist(), "offset": off, "count": cnt}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
