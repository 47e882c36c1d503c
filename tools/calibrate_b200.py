"""B200 recalibration of the cost model (the paper's Table-1
methodology on this hardware): time the device step of the dense AlexNet plan
d1m1 at several per-device batches (CUDA-graph replay, CUDA events, inputs
resident), fit the compute term with costmodel.calibrate_compute, and write
configs/b200.cost (the reference's cost-parameter format; measured rows kept
as comments). Needs a GPU:  python tools/calibrate_b200.py [out]
"""

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_1312_5853_b200 as P  # noqa: E402
from paper_1312_5853_b200 import costmodel as CM, rng as R, schemes as S  # noqa: E402
from paper_1312_5853_b200.data import synthetic_rows  # noqa: E402
from paper_1312_5853_b200.plan import plan_columnized  # noqa: E402

BATCHES = (32, 64, 128, 256, 512)


def step_seconds(net, batch, steps=20, warmup=5):
    plan = P.ParallelPlan(1, 1)
    cs = plan_columnized(net, plan)
    order = R.permutation(0, 0, 1000 * max(1, -(-batch // 1000)))[:batch]
    xb, yb = synthetic_rows(1000, max(1, -(-batch // 1000)), net.input_shape, 0, order)
    fab = P.spawn(1, precision="bf16")
    P.setup_workers(fab, plan, cs, P.init_dense_params(net, 0, std=0.01), P.SgdState())
    P.hybrid_step(fab, plan, cs, torch.from_numpy(xb).to(torch.bfloat16), yb.astype(np.int32))
    run = S._runner(fab, plan, cs, batch)
    for _ in range(warmup):
        run.program(1.0 / batch)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        run.program(1.0 / batch)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps / 1e3


def main():
    out = Path(sys.argv[1]) if len(sys.argv) > 1 else ROOT / "configs" / "b200.cost"
    net = P.load_network(ROOT / "configs" / "alexnet.net")
    rows = []
    for b in BATCHES:
        sec = step_seconds(net, b)
        rows.append((b, sec))
        print(f"batch {b}: {sec * 1e3:.3f} ms/step ({b / sec:.0f} img/s)", flush=True)
    cp = CM.calibrate_compute(rows, net)
    CM.save_cost_params(cp, out)
    lines = ["# B200 cost parameters (tools/calibrate_b200.py): throughput and b_half fitted to the",
             "# measured d1m1 AlexNet-227 device step (bf16, CUDA graph, inputs resident);",
             "# bandwidth / latency = NVLink 5 per-direction bandwidth and an NCCL call latency",
             "# (stated, not fitted: one GPU per measurement call); memory = 180 GB HBM3e.",
             "# rows: '# step <batch> <seconds>'"]
    lines += [f"# step {b} {sec!r}" for b, sec in rows]
    out.write_text("\n".join(lines) + "\n" + out.read_text())
    print(out.read_text())


if __name__ == "__main__":
    main()
