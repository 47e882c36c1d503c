"""Single-process multi-GPU fabric (multidev.PeerRunner): one host thread and
stream per worker, peer-memory exchange and reduce-scatter / all-gather replica
reduction — the reference's ``Fabric.run`` execution model
(`pkg/src/parconv/fabric.py:280-339`).

On a one-GPU box every worker is pinned to GPU 0 (``devices=[0] * n``): the
same threads, streams, events and peer-pointer kernels run, and the results
must be BIT-identical to the single-stream path (same kernels, same ascending
summation orders), which is itself pinned to the reference (test_gpu_step.py).
With two or more GPUs visible the workers spread over them and the same
assertions hold.
"""

import numpy as np
import pytest
import torch

from conftest import CONFIGS, GOLDEN

pytestmark = pytest.mark.gpu

STEPS = np.load(GOLDEN / "steps.npz")


def _devices(n):
    count = torch.cuda.device_count()
    return [w * min(n, count) // n for w in range(n)] if count > 1 else [0] * n


def _run(net, plan, dense, batches, precision, devices):
    import paper_1312_5853_b200 as P
    from paper_1312_5853_b200.plan import plan_columnized
    from paper_1312_5853_b200.schemes import column_params
    cs = plan_columnized(net, plan)
    fab = P.spawn(plan.workers, precision=precision, devices=devices)
    P.setup_workers(fab, plan, cs, dense, P.SgdState())
    losses, ledger = [], []
    for x, y in batches:
        r = P.hybrid_step(fab, plan, cs, x, y)
        losses.append(r.loss)
        ledger.append((r.ledger_bytes, r.ledger_messages))
    cols = [column_params(fab, plan.worker_of(0, j)) for j in range(plan.model_columns)]
    p32 = {w: e.p32.cpu() for w, e in fab._engines.items()}
    return fab, losses, ledger, cols, p32


PLANS = {"d2m1": (2, 1, ()), "d1m2x3": (1, 2, (3,)), "d2m2x3": (2, 2, (3,)), "d1m4x3": (1, 4, (3,)),
         "d4m1": (4, 1, ())}


@pytest.mark.parametrize("pname", sorted(PLANS))
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_peer_fabric_bit_identical_to_single_stream(pname, precision):
    import paper_1312_5853_b200 as P
    net = P.load_network(CONFIGS / "tinynet.net")
    plan = P.ParallelPlan(*PLANS[pname])
    dense = {i: {k: STEPS[f"tiny_p0_{i}_{k}"] for k in ("w", "b")} for i in (0, 3, 5, 7)}
    batches = [(STEPS[f"tiny_x{s}"], STEPS[f"tiny_y{s}"]) for s in range(3)]
    fab, l_multi, led_m, cols_m, p_m = _run(net, plan, dense, batches, precision, _devices(plan.workers))
    assert fab.multi and type(fab._runner).__name__ == "PeerRunner"
    _, l_one, led_1, cols_1, p_1 = _run(net, plan, dense, batches, precision, None)
    assert l_multi == l_one
    assert led_m == led_1
    for w in p_m:
        assert torch.equal(p_m[w], p_1[w]), w
    # replicas hold bit-identical parameters (the reference's broadcast)
    d, m = plan.data_shards, plan.model_columns
    for r in range(1, d):
        for j in range(m):
            assert torch.equal(p_m[r * m + j], p_m[j])
    if precision == "fp32" and pname in ("d2m1", "d1m2x3", "d2m2x3", "d1m4x3"):
        for st in range(2):
            ref = float(STEPS[f"hyb_{pname}_loss{st}"])
            assert abs(l_multi[st] - ref) / abs(ref) < 1e-5


def test_peer_fabric_alexnet_hybrid_bf16():
    """AlexNet-227 Krizhevsky cross(6), d2 x m2 (the paper's hybrid on 4 workers),
    two steps: bit-identical to the single-stream path."""
    import paper_1312_5853_b200 as P
    from paper_1312_5853_b200.data import synthetic_rows
    net = P.load_network(CONFIGS / "alexnet.net")
    plan = P.ParallelPlan(2, 2, (6,))
    dense = P.init_dense_params(net, 0, std=0.01)
    x, y = synthetic_rows(1000, 1, net.input_shape, 0, np.arange(16) * 61)
    batches = [(x, y), (x[::-1].copy(), y[::-1].copy())]
    _, l_multi, _, _, p_m = _run(net, plan, dense, batches, "bf16", _devices(4))
    _, l_one, _, _, p_1 = _run(net, plan, dense, batches, "bf16", None)
    assert l_multi == l_one
    for w in p_m:
        assert torch.equal(p_m[w], p_1[w]), w


def test_peer_fabric_evaluation_and_errors():
    import paper_1312_5853_b200 as P
    from paper_1312_5853_b200.plan import plan_columnized
    net = P.load_network(CONFIGS / "tinynet.net")
    plan = P.ParallelPlan(2, 2, (3,))
    cs = plan_columnized(net, plan)
    dense = {i: {k: STEPS[f"tiny_p0_{i}_{k}"] for k in ("w", "b")} for i in (0, 3, 5, 7)}
    x, y = STEPS["tiny_x0"], STEPS["tiny_y0"]
    counts = []
    for devices in (_devices(4), None):
        fab = P.spawn(4, precision="fp32", devices=devices)
        P.setup_workers(fab, plan, cs, dense, P.SgdState())
        P.hybrid_step(fab, plan, cs, x, y)
        counts.append(P.evaluation_errors(fab, plan, cs, x, y))
        with pytest.raises(P.ValidationError):      # out-of-range label
            P.hybrid_step(fab, plan, cs, x, np.full(len(y), 10))
    assert counts[0] == counts[1]
    with pytest.raises(P.ValidationError):
        P.spawn(4, devices=[0, 0])


@pytest.mark.parametrize("sched", ["lockstep", "threads"])
def test_fabric_run_moves_device_tensors_between_workers(sched):
    """Fabric.run with CUDA tensor payloads (mailbox.py): the copy lands on the
    receiver's GPU, ordered after the sender's stream; reduce_to_root sums on the
    root's device in ascending worker order, bit-identical to the float64 host
    program rounded the same way."""
    import torch
    import paper_1312_5853_b200 as P
    n = 4
    fab = P.spawn(n, scheduling=sched, devices=_devices(n))
    rs = np.random.RandomState(7)
    host = [rs.randn(1 << 16).astype(np.float32) for _ in range(n)]

    def program(ctx):
        dev = fab.device_of(ctx.wid)
        x = torch.from_numpy(host[ctx.wid]).to(dev)
        x = x * 2 + 1                               # produced on this worker's stream
        ctx.send((ctx.wid + 1) % n, "ring", x)
        y = ctx.recv((ctx.wid - 1) % n, "ring")
        assert y.device == dev
        tot = ctx.reduce_to_root(range(n), 0, x + y)
        return ctx.broadcast_from_root(range(n), 0, tot if ctx.wid == 0 else None).cpu()

    res = fab.run(program)
    xs = [torch.from_numpy(h) * 2 + 1 for h in host]
    want = None
    for w in range(n):
        v = xs[w] + xs[(w - 1) % n]
        want = v.clone() if want is None else want.add_(v)
    for r in res:
        assert torch.equal(r, want)
    assert fab.ledger.total_messages == n + (n - 1) * 2
