"""Multi-GPU torchrun path (one process per GPU, NCCL column / replica groups,
CUDA-graph-captured collectives) vs the reference's own trajectories (golden
steps.npz, `pkg/src/parconv/schemes.py:500-569`) at the fp32 bound, and bf16
vs the single-GPU run of the same plan. Needs >= 2 GPUs: skipped on a one-GPU
box (the same plans run there through the single-process fabrics, which are
bit-identical to each other: tests/test_gpu_multidev.py)."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

from conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu

STEPS = np.load(GOLDEN / "steps.npz")
PLANS = {"d1m2x3": (1, 2, "3"), "d2m1": (2, 1, ""), "d2m2x3": (2, 2, "3")}


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(d, m, cross, precision, out):
    n = d * m
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "tests" / "nccl_parity_worker.py"),
           str(d), str(m), cross, precision, str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=dict(os.environ))
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(out.read_text())


@pytest.mark.parametrize("pname", sorted(PLANS))
def test_nccl_plans_fp32_match_reference(pname, tmp_path):
    d, m, cross = PLANS[pname]
    if torch.cuda.device_count() < d * m:
        pytest.skip(f"needs {d * m} GPUs")
    res = _torchrun(d, m, cross, "fp32", tmp_path / "out.json")
    for st in range(2):
        ref = float(STEPS[f"hyb_{pname}_loss{st}"])
        assert abs(res["losses"][st] - ref) / abs(ref) < 1e-5
        led = STEPS[f"hyb_{pname}_ledger{st}"]
        assert res["ledgers"][st] == [int(led[0]), int(led[1])]
    assert res["graphs"] >= 1          # the third step replayed the captured graph


@pytest.mark.parametrize("pname", sorted(PLANS))
def test_nccl_plans_bf16_match_single_gpu(pname, tmp_path):
    import paper_1312_5853_b200 as P
    from paper_1312_5853_b200.plan import plan_columnized
    d, m, cross = PLANS[pname]
    if torch.cuda.device_count() < d * m:
        pytest.skip(f"needs {d * m} GPUs")
    res = _torchrun(d, m, cross, "bf16", tmp_path / "out.json")
    net = P.load_network(ROOT / "configs" / "tinynet.net")
    plan = P.ParallelPlan(d, m, tuple(int(c) for c in cross.split(",") if c))
    cs = plan_columnized(net, plan)
    fab = P.spawn(plan.workers, precision="bf16", devices=[0] * plan.workers)
    dense = {i: {k: STEPS[f"tiny_p0_{i}_{k}"] for k in ("w", "b")} for i in (0, 3, 5, 7)}
    P.setup_workers(fab, plan, cs, dense, P.SgdState())
    for st in range(3):
        loss = P.hybrid_step(fab, plan, cs, STEPS[f"tiny_x{st % 2}"], STEPS[f"tiny_y{st % 2}"]).loss
        # NCCL's reduction order may differ from the ascending single-process sum
        assert abs(loss - res["losses"][st]) <= 1e-3 * abs(loss)
