"""Ragged batch sizes through one fabric (the reference accepts any batch its
plan can shard, `schemes.py:500-570`): the device buffers, the per-shape CUDA
graphs and the split-K / tile plans change with every size, including batches
of one image and sizes that are not multiples of any tile. Every step is
checked against the float64 oracle from the parameters the device held before
it (tests/parity.py replays the device's max-pool and ReLU decisions), so a
wrong graph or stale buffer for one size shows up at that step.
"""

import numpy as np
import pytest

from conftest import CONFIGS
from parity import rel_l2

pytestmark = pytest.mark.gpu


def _columns(fab, plan):
    from paper_1312_5853_b200.schemes import column_params
    return [column_params(fab, plan.worker_of(0, j)) for j in range(plan.model_columns)]


def _check_sequence(net_name, plan_args, sizes, precision, loss_tol, upd_tol, std=None):
    import paper_1312_5853_b200 as P
    from oracle.ref_engine import OracleFabric
    from parity import assert_near_ties, assert_relu_near_ties, device_argmax, device_relu_masks
    from paper_1312_5853_b200.data import synthetic_rows
    from paper_1312_5853_b200.plan import plan_columnized
    net = P.load_network(CONFIGS / f"{net_name}.net")
    plan = P.ParallelPlan(*plan_args)
    cs = plan_columnized(net, plan)
    dense = {i: {k: v.astype(np.float32).astype(np.float64) for k, v in t.items()}
             for i, t in P.init_dense_params(net, 0, std=std).items()}
    fab = P.spawn(plan.workers, precision=precision)
    # momentum 0: each step's update depends only on the parameters before it (no
    # velocity to carry into the oracle)
    P.setup_workers(fab, plan, cs, dense, P.SgdState(momentum=0.0))
    tie_tol = 1e-5 if precision == "fp32" else 2e-2
    for step, b in enumerate(sizes):
        x, y = synthetic_rows(net.classes, 1, net.input_shape, step, (np.arange(b) * 7 + step) % net.classes)
        x = x.astype(np.float64)
        before = _columns(fab, plan)
        res = P.hybrid_step(fab, plan, cs, x, y)
        of = OracleFabric(net, plan, dense, momentum=0.0)
        of.params = [{i: {k: v.copy() for k, v in t.items()} for i, t in c.items()} for c in before]
        forced, relu, trace = device_argmax(fab, plan), device_relu_masks(fab, plan), {}
        oloss = of.step(x, y, trace=trace, force_argmax=forced, force_relu=relu)
        assert_near_ties(trace, forced, of.cs, tie_tol)
        assert_relu_near_ties(trace, relu, tie_tol)
        assert abs(res.loss - oloss) / abs(oloss) < loss_tol, (step, b, res.loss, oloss)
        after = _columns(fab, plan)
        for j in range(plan.model_columns):
            for i in after[j]:
                for k in ("w", "b"):
                    if precision == "fp32":
                        # the update (~1e-7) is a few float32 ulps of a weight (~1e-2): compare
                        # the stored parameters, within upd_tol ulps of the oracle's plus 1e-5
                        # of the update (biases start at 0: there the update is the value)
                        want = of.params[j][i][k].astype(np.float32)
                        upd = float(np.max(np.abs(of.params[j][i][k] - before[j][i][k])))
                        slack = upd_tol * np.spacing(np.abs(want)) + 1e-5 * upd
                        excess = np.abs(after[j][i][k] - want) - slack
                        assert float(excess.max()) <= 0, (step, b, j, i, k, float(excess.max()), upd)
                    else:
                        err = rel_l2(after[j][i][k] - before[j][i][k], of.params[j][i][k] - before[j][i][k])
                        assert err < upd_tol, (step, b, j, i, k, err)


def test_alexnet_bf16_ragged_batches_one_fabric():
    """AlexNet-227 d1m1 bf16: 3, 1, 16, 3 images (the second 3 replays the graph
    captured for the first)."""
    _check_sequence("alexnet", (1, 1, ()), [3, 1, 16, 3], "bf16", 1e-2, 0.3, std=0.01)


@pytest.mark.parametrize("precision,loss_tol,upd_tol", [("fp32", 1e-5, 1.0), ("bf16", 1e-2, 0.3)])
def test_small64_hybrid_ragged_batches_one_fabric(precision, loss_tol, upd_tol):
    """alexnet_small64, d2 x m2 cross(6): 2, 6, 34, 2 images (one per replica
    at the smallest)."""
    _check_sequence("alexnet_small64", (2, 2, (6,)), [2, 6, 34, 2], precision, loss_tol, upd_tol, std=0.01)
