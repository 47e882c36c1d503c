"""GPU tests of the rows around the step:

* evaluation_errors (`pkg/src/parconv/schemes.py:600-645`) on the device vs the
  reference's own counts and exchange ledger (golden eval.npz), cached engines;
* the device reference_step (`schemes.py:439-458`) vs the oracle's, threading
  the SgdState velocity through two calls;
* on-device synthetic data (pc_synthetic_rows) vs the host restatement of
  `data.py:52-96` (itself pinned to the reference's host.npz vectors), and the
  device batch gather (pc_gather_rows).
"""

import numpy as np
import pytest

from conftest import CONFIGS, GOLDEN
from parity import rel

pytestmark = pytest.mark.gpu

EVAL = np.load(GOLDEN / "eval.npz")
CASES = {"tiny_d1m2x3": ("tinynet", (1, 2, (3,))), "tiny_d2m2x3": ("tinynet", (2, 2, (3,))),
         "tiny_d2m1": ("tinynet", (2, 1, ())), "small64_d1m2x6": ("alexnet_small64", (1, 2, (6,)))}


def f32_params(params):
    return {i: {k: v.astype(np.float32).astype(np.float64) for k, v in t.items()} for i, t in params.items()}


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_evaluation_errors_match_reference(name, precision):
    import paper_1312_5853_b200 as P
    from paper_1312_5853_b200.plan import plan_columnized
    net_name, (d, m, cross) = CASES[name]
    net = P.load_network(CONFIGS / f"{net_name}.net")
    plan = P.ParallelPlan(d, m, cross)
    cs = plan_columnized(net, plan)
    fab = P.spawn(plan.workers, precision=precision)
    P.setup_workers(fab, plan, cs, f32_params(P.init_dense_params(net, 3)), P.SgdState())
    P.hybrid_step(fab, plan, cs, EVAL[f"{name}_x"].astype(np.float64), EVAL[f"{name}_y"])
    tx, ty = EVAL[f"{name}_tx"].astype(np.float64), EVAL[f"{name}_ty"]
    b0, m0 = fab.ledger.total_bytes, fab.ledger.total_messages
    wrong = P.evaluation_errors(fab, plan, cs, tx, ty)
    assert [fab.ledger.total_bytes - b0, fab.ledger.total_messages - m0] == list(EVAL[f"{name}_ledger"])
    want = int(EVAL[f"{name}_wrong"])
    if precision == "fp32":
        assert wrong == want
    else:   # bf16 logits may rank a near-tie differently
        assert abs(wrong - want) <= max(1, len(ty) // 10)
    # the engines are cached per batch size and refreshed from the training engines
    cache = dict(fab._eval_cache)
    again = P.evaluation_errors(fab, plan, cs, tx, ty)
    assert again == wrong and all(fab._eval_cache[k] is v for k, v in cache.items())
    P.hybrid_step(fab, plan, cs, EVAL[f"{name}_x"].astype(np.float64), EVAL[f"{name}_y"])
    P.evaluation_errors(fab, plan, cs, tx, ty)      # refreshed parameters, same engines
    eng = next(iter(fab._eval_cache.values()))[0]
    assert P.evaluation_errors(fab, plan, cs, tx[:0], ty[:0]) == 0
    import torch
    assert torch.equal(eng.p32, fab._engines[eng.wid].p32)


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-5), ("bf16", 2e-2)])
def test_device_reference_step_matches_oracle(precision, tol):
    """Two chained reference_step calls (params and SgdState velocity threaded
    through, `schemes.py:439-458`) vs the oracle's reference_step."""
    import paper_1312_5853_b200 as P
    from oracle.ref_engine import reference_step as oracle_step
    from paper_1312_5853_b200.plan import lists_as_params
    net = P.load_network(CONFIGS / "tinynet.net")
    steps = np.load(GOLDEN / "steps.npz")
    params = {i: {k: steps[f"tiny_p0_{i}_{k}"] for k in ("w", "b")} for i in (0, 3, 5, 7)}
    sgd = P.SgdState()
    oparams, ovel = params, None
    cs = P.columnize(net, 1)
    for st in range(2):
        x, y = steps[f"tiny_x{st}"], steps[f"tiny_y{st}"]
        res = P.reference_step(net, params, (x, y), sgd, precision=precision)
        wloss, wparams, wvel = oracle_step(net, oparams, (x, y), velocity=ovel)
        assert abs(res.loss - wloss) / abs(wloss) < tol
        assert abs(res.loss - float(steps[f"tiny_loss{st}"])) / abs(wloss) < tol
        for i in res.params:
            for k in ("w", "b"):
                d_got = res.params[i][k] - params[i][k]
                d_want = wparams[i][k] - oparams[i][k]
                assert rel(d_got, d_want) < (tol if precision == "fp32" else 0.3), (st, i, k)
        got_v = lists_as_params(list(res.sgd.velocity), cs)
        want_v = lists_as_params(list(wvel), cs)
        for i in got_v:
            for k in ("w", "b"):
                assert rel(got_v[i][k], want_v[i][k]) < (tol if precision == "fp32" else 0.3)
        params, sgd = res.params, res.sgd
        oparams, ovel = wparams, wvel


@pytest.mark.parametrize("shape,classes,per_class,split", [((3, 227, 227), 1000, 1, "train"),
                                                           ((3, 64, 64), 100, 4, "train"),
                                                           ((2, 4, 4), 3, 2, "test")])
def test_synthetic_rows_on_device_match_host(shape, classes, per_class, split):
    import torch
    from paper_1312_5853_b200 import rng
    from paper_1312_5853_b200.data import synthetic_rows, synthetic_rows_device, gen_synthetic
    n = classes * per_class
    idx = rng.permutation(0, 0, n)[: min(n, 24)]
    dev = synthetic_rows_device(classes, per_class, shape, 11, idx, split=split).cpu().numpy()
    if split == "train":
        host, _ = synthetic_rows(classes, per_class, shape, 11, idx)
    else:
        _, te = gen_synthetic(classes, 4 * per_class, shape, seed=11, test_per_class=per_class)
        host = te.images[idx].astype(np.float32)
    assert dev.dtype == np.float32 and dev.shape == host.shape
    diff = dev != host
    # CUDA's and numpy's double log/sin/cos may differ in the last bit; that moves the
    # float32 image by one ulp only at a float32 rounding boundary
    ulp = np.abs(dev.view(np.int32).astype(np.int64) - host.view(np.int32).astype(np.int64))
    assert ulp.max() <= 1 and diff.mean() < 1e-5, (int(diff.sum()), diff.size)
    bf = synthetic_rows_device(classes, per_class, shape, 11, idx, dtype=torch.bfloat16, split=split)
    assert torch.equal(bf, torch.as_tensor(dev).cuda().bfloat16())


def test_gather_rows_matches_index_select():
    import torch
    from paper_1312_5853_b200.trainer import _gather
    for row in ((3, 227, 227), (3, 64, 64), (5,)):
        src = torch.randn((37,) + row, device="cuda")
        idx = np.array([5, 0, 36, 5, 17, 2])
        assert torch.equal(_gather(src, idx), src.index_select(0, torch.as_tensor(idx).cuda()))


@pytest.mark.parametrize("plan_args", [(1, 1, ()), (2, 1, ()), (1, 2, (6,))])
def test_train_device_resident_test_split_matches_host(plan_args):
    """train() with device_data evaluates the test split from HBM (evaluation_errors
    on device tensors): the per-epoch test errors and losses equal the host-fed run's,
    and evaluation_errors on a CUDA tensor equals the numpy call."""
    import torch
    import paper_1312_5853_b200 as P
    net = P.load_network(CONFIGS / "alexnet_small64.net")
    train_set, test_set = P.gen_synthetic(100, 2, net.input_shape, seed=4)
    plan = P.ParallelPlan(*plan_args)
    runs = []
    for dev in (True, False):
        cfg = P.TrainConfig(net=net, plan=plan, epochs=2, batch=32, seed=3, train_data=train_set, test_data=test_set,
                            precision="bf16", device_data=dev, sgd=P.SgdState(learning_rate=0.001))
        res = P.train(cfg)
        runs.append([(r.train_loss, r.test_error) for r in res.records])
        if dev:
            fab = res.fabric
            cs = P.columnize(net, plan.model_columns, plan.cross_layers)
            xd = torch.as_tensor(np.ascontiguousarray(test_set.images[:50], dtype=np.float32)).cuda()
            a = P.evaluation_errors(fab, plan, cs, xd, test_set.labels[:50])
            b = P.evaluation_errors(fab, plan, cs, test_set.images[:50], test_set.labels[:50])
            assert a == b
    assert runs[0] == runs[1]
    assert any(e is not None for _, e in runs[0])
