"""One eager AlexNet-227 b256 training step through the drop-in API (for ncu
captures of a single step's kernels): python tools/prof_step_once.py [net] [precision]"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1312_5853_b200 as P  # noqa: E402
from paper_1312_5853_b200.data import synthetic_rows  # noqa: E402

net = P.load_network(sys.argv[1] if len(sys.argv) > 1 else ROOT / "configs" / "alexnet.net")
prec = sys.argv[2] if len(sys.argv) > 2 else "bf16"
plan = P.ParallelPlan(1, 1)
cs = P.columnize(net, 1)
x, y = synthetic_rows(1000, 1, net.input_shape, 0, np.arange(256))
fab = P.spawn(1, precision=prec)
P.setup_workers(fab, plan, cs, P.init_dense_params(net, 0, std=0.01), P.SgdState())
xb = torch.from_numpy(x).to(torch.bfloat16 if prec == "bf16" else torch.float32).pin_memory()
P.hybrid_step(fab, plan, cs, xb, y)
torch.cuda.synchronize()
print("loss", P.hybrid_step(fab, plan, cs, xb, y).loss)
torch.cuda.synchronize()
