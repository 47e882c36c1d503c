"""Step-level parity on the B200: the drop-in scheme API vs the reference's
trajectories (golden fixtures written by the reference itself) and vs the
float64 oracle, layer by layer.

fp32 mode bound (north_star): <= 1e-5 relative (max-normalised)
on losses and parameters / parameter updates. bf16 mode: activations and
loss <= 1e-2 rel-L2, weight gradients / updates <= 0.3 rel-L2.
"""

import numpy as np
import pytest

from conftest import CONFIGS, GOLDEN
from oracle.ref_engine import OracleFabric, column_fwd_bwd

pytestmark = pytest.mark.gpu

STEPS = np.load(GOLDEN / "steps.npz")
TOL = 1e-5


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def tree(prefix, idxs):
    return {i: {k: STEPS[f"{prefix}_{i}_{k}"] for k in ("w", "b")} for i in idxs}


def test_library_reports_device():
    from paper_1312_5853_b200._lib import lib
    assert lib().dll.pc_version() == 1


def test_tinynet_trajectory_fp32():
    import paper_1312_5853_b200 as P
    net = P.load_network(CONFIGS / "tinynet.net")
    plan = P.ParallelPlan(1, 1)
    cs = P.columnize(net, 1)
    fab = P.spawn(1, precision="fp32")
    P.setup_workers(fab, plan, cs, tree("tiny_p0", (0, 3, 5, 7)), P.SgdState())
    for st in range(3):
        res = P.hybrid_step(fab, plan, cs, STEPS[f"tiny_x{st}"], STEPS[f"tiny_y{st}"])
        ref = float(STEPS[f"tiny_loss{st}"])
        assert abs(res.loss - ref) / abs(ref) < TOL
    got = P.gather_dense_params(fab, plan, cs)
    p0, p3 = tree("tiny_p0", (0, 3, 5, 7)), tree("tiny_p3", (0, 3, 5, 7))
    for i in p3:
        for k in ("w", "b"):
            assert rel(got[i][k], p3[i][k]) < TOL
            assert rel(got[i][k] - p0[i][k], p3[i][k] - p0[i][k]) < 1e-4


PLANS = {"d2m1": (2, 1, ()), "d1m2x3": (1, 2, (3,)), "d2m2x3": (2, 2, (3,)), "d1m4x3": (1, 4, (3,)),
         "d1m2grp": (1, 2, ())}


@pytest.mark.parametrize("pname", sorted(PLANS))
def test_hybrid_plans_fp32_match_reference(pname):
    import paper_1312_5853_b200 as P
    d, m, cross = PLANS[pname]
    net = P.load_network(CONFIGS / "tinynet.net")
    plan = P.ParallelPlan(d, m, cross)
    cs = P.plan_columnized(net, plan) if hasattr(P, "plan_columnized") else P.columnize(net, m, cross)
    fab = P.spawn(plan.workers, precision="fp32")
    P.setup_workers(fab, plan, cs, tree("tiny_p0", (0, 3, 5, 7)), P.SgdState())
    for st in range(2):
        res = P.hybrid_step(fab, plan, cs, STEPS[f"tiny_x{st}"], STEPS[f"tiny_y{st}"])
        ref = float(STEPS[f"hyb_{pname}_loss{st}"])
        assert abs(res.loss - ref) / abs(ref) < TOL
        led = STEPS[f"hyb_{pname}_ledger{st}"]
        assert (res.ledger_bytes, res.ledger_messages) == (int(led[0]), int(led[1]))
    from paper_1312_5853_b200.schemes import column_params
    for j in range(m):
        got = column_params(fab, j)
        for i in (0, 3, 5, 7):
            for k in ("w", "b"):
                assert rel(got[i][k], STEPS[f"hyb_{pname}_col{j}_{i}_{k}"]) < TOL


def test_small64_layer_by_layer_fp32():
    """Forward activations, input gradients and parameter gradients of every
    layer vs the oracle (config #1 net, B=4)."""
    import paper_1312_5853_b200 as P
    from paper_1312_5853_b200.plan import plan_columnized
    net = P.load_network(CONFIGS / "alexnet_small64.net")
    plan = P.ParallelPlan(1, 2, (6,))
    cs = plan_columnized(net, plan)
    dense = {i: {k: v.astype(np.float32).astype(np.float64) for k, v in t.items()}
             for i, t in P.init_dense_params(net, 3).items()}
    x, y = STEPS["small64_x0"], STEPS["small64_y0"]
    trace = {}
    ofab = OracleFabric(net, plan, dense)
    oloss = ofab.step(x, y, trace=trace)
    fab = P.spawn(2, precision="fp32")
    P.setup_workers(fab, plan, cs, dense, P.SgdState())
    res = P.hybrid_step(fab, plan, cs, x, y)
    assert abs(res.loss - oloss) / abs(oloss) < TOL
    for j in range(2):
        eng = fab._engines[j]
        for i, cl in enumerate(cs.col_layers):
            st = eng.layers[i]
            if st.kind == "softmax" or (st.kind == "relu" and st.relu_fused_fwd):
                continue
            # conv/FC outputs are stored after their fused ReLU: compare with the ReLU output
            ref_idx = cl.index + 1 if st.relu_after else cl.index
            assert rel(eng.activation_host(i, "out"), trace["fwd"][ref_idx][j]) < TOL, cl.index
            if st.kind == "pool":
                # end to end, fp32-vs-float64 rounding may legitimately move a near-tie
                # (bit-exactness is asserted at kernel level in test_gpu_kernels.py)
                got = eng.layers[i].argmax[: st.out.numel()].cpu().numpy().reshape(
                    (4,) + st.out_nhwc).transpose(0, 3, 1, 2)
                assert np.mean(got != trace["argmax"][cl.index][j]) < 1e-3
        for i, t in eng.grads_host().items():
            for k in ("w", "b"):
                assert rel(t[k], trace["grads"][j][i][k]) < TOL, (i, k)


def test_alexnet_b2_fp32_matches_reference_digest():
    import paper_1312_5853_b200 as P
    g = np.load(GOLDEN / "alexnet.npz")
    net = P.load_network(CONFIGS / "alexnet.net")
    dense = {i: {k: v.astype(np.float32).astype(np.float64) for k, v in t.items()}
             for i, t in P.init_dense_params(net, 0).items()}
    res = P.reference_step(net, dense, (g["x"].astype(np.float64), g["y"]), P.SgdState())
    assert abs(res.loss - float(g["loss"])) / float(g["loss"]) < TOL
    # First step from zero velocity: the new velocity IS the update p1 - p0, computed
    # in fp32 on the device (p1 - p0 itself would measure fp32 storage of p, ~4e-4 of
    # the update on conv1, not the step's arithmetic).
    from paper_1312_5853_b200.plan import lists_as_params
    vel = lists_as_params(res.sgd.velocity, P.columnize(net, 1))
    for i in dense:
        for k in ("w", "b"):
            d = vel[i][k]
            dig = g[f"d_{i}_{k}"]
            assert abs(d.sum() - dig[0]) <= TOL * dig[1] * np.sqrt(d.size) + 1e-12, (i, k)
            assert abs(np.sqrt((d ** 2).sum()) - dig[1]) <= TOL * dig[1] + 1e-12, (i, k)
            assert abs(np.abs(d).max() - dig[2]) <= TOL * dig[2] * 10 + 1e-12, (i, k)


def test_alexnet_krizhevsky_columns_bf16_bounds():
    """AlexNet-227 two-column cross(6) plan, bf16 tensor-core mode vs the
    float64 oracle: loss and update bounds of the bf16 contract."""
    import paper_1312_5853_b200 as P
    from paper_1312_5853_b200.plan import plan_columnized
    net = P.load_network(CONFIGS / "alexnet.net")
    plan = P.ParallelPlan(1, 2, (6,))
    cs = plan_columnized(net, plan)
    dense = {i: {k: v.astype(np.float32).astype(np.float64) for k, v in t.items()}
             for i, t in P.init_dense_params(net, 0).items()}
    tr, _ = P.gen_synthetic(4, 1, net.input_shape, seed=1)
    x, y = tr.images, np.array([0, 17, 999, 500])
    ofab = OracleFabric(net, plan, dense)
    oloss = ofab.step(x, y)
    fab = P.spawn(2, precision="bf16")
    P.setup_workers(fab, plan, cs, dense, P.SgdState())
    res = P.hybrid_step(fab, plan, cs, x, y)
    assert abs(res.loss - oloss) / oloss < 1e-2
    from paper_1312_5853_b200.plan import split_params
    from paper_1312_5853_b200.schemes import column_params
    for j in range(2):
        got = column_params(fab, j)
        start = split_params(dense, cs, j)
        for i in got:
            d_got = got[i]["w"] - start[i]["w"]
            d_ref = ofab.params[j][i]["w"] - start[i]["w"]
            assert rel_l2(d_got, d_ref) < 0.3, (j, i)


def test_label_out_of_range_raises():
    import paper_1312_5853_b200 as P
    net = P.load_network(CONFIGS / "tinynet.net")
    plan = P.ParallelPlan(1, 1)
    cs = P.columnize(net, 1)
    fab = P.spawn(1, precision="fp32")
    P.setup_workers(fab, plan, cs, tree("tiny_p0", (0, 3, 5, 7)), P.SgdState())
    with pytest.raises(P.ValidationError):
        P.hybrid_step(fab, plan, cs, STEPS["tiny_x0"], np.full(8, 10))
    with pytest.raises(P.ValidationError):
        P.data_parallel_step(fab, P.ParallelPlan(1, 2), P.columnize(net, 2, (3,)), STEPS["tiny_x0"],
                             STEPS["tiny_y0"])
