"""torchrun worker for tests/test_gpu_nccl.py (one rank per GPU, NCCL): runs a
tinynet plan through the drop-in API and rank 0 writes the losses and column
parameters as JSON for the test to compare with the reference's goldens."""

import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    d, m, cross, precision, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4], sys.argv[5]
    cross = tuple(int(c) for c in cross.split(",") if c)
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1312_5853_b200 as P
    from paper_1312_5853_b200.plan import plan_columnized
    from paper_1312_5853_b200.schemes import column_params
    steps = np.load(ROOT / "tests" / "golden" / "steps.npz")
    net = P.load_network(ROOT / "configs" / "tinynet.net")
    plan = P.ParallelPlan(d, m, cross)
    cs = plan_columnized(net, plan)
    fab = P.spawn(plan.workers, precision=precision)
    dense = {i: {k: steps[f"tiny_p0_{i}_{k}"] for k in ("w", "b")} for i in (0, 3, 5, 7)}
    P.setup_workers(fab, plan, cs, dense, P.SgdState())
    losses, ledgers = [], []
    for st in range(3):        # step 1 eager, step 2 captured, step 3 replayed
        r = P.hybrid_step(fab, plan, cs, steps[f"tiny_x{st % 2}"], steps[f"tiny_y{st % 2}"])
        losses.append(r.loss)
        ledgers.append([r.ledger_bytes, r.ledger_messages])
    wrong = P.evaluation_errors(fab, plan, cs, steps["tiny_x0"], steps["tiny_y0"])
    cols = {}
    for j in range(m):
        obj = [column_params(fab, j) if fab.rank == j else None]
        dist.broadcast_object_list(obj, src=j)
        cols[j] = {str(i): {k: v.tolist() for k, v in t.items()} for i, t in obj[0].items()}
    if fab.rank == 0:
        Path(out).write_text(json.dumps({"losses": losses, "ledgers": ledgers, "cols": cols, "wrong": wrong,
                                         "graphs": fab._runner.replays}))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
