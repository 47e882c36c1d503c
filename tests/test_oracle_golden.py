"""Pin the CPU oracle to the reference: golden vectors written by the real
reference (tests/golden/make_golden.py) plus the reference's own known-answer
tests (`pkg/tests/test_kernels.py`) restated. CPU only."""

import numpy as np
import pytest

from conftest import CONFIGS, GOLDEN
import oracle
from oracle import ref_kernels as K
from oracle.ref_engine import OracleFabric, reference_step
from paper_1312_5853_b200.netdef import load_network
from paper_1312_5853_b200.plan import ParallelPlan, init_dense_params

KER = np.load(GOLDEN / "kernels.npz")
STEPS = np.load(GOLDEN / "steps.npz")


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


@pytest.mark.parametrize("gi", range(5))
def test_conv_matches_reference(gi):
    b, c, h, w, n, k, s, p = KER[f"conv{gi}_geom"]
    x, wt, bias, gy = (KER[f"conv{gi}_{t}"] for t in ("x", "w", "b", "gy"))
    assert rel(K.conv2d_forward(x, wt, bias, s, p), KER[f"conv{gi}_y"]) < 1e-13
    gx, gw, gb = K.conv2d_backward(x, wt, gy, s, p)
    assert rel(gx, KER[f"conv{gi}_gx"]) < 1e-13
    assert rel(gw, KER[f"conv{gi}_gw"]) < 1e-13
    assert rel(gb, KER[f"conv{gi}_gb"]) < 1e-13


@pytest.mark.parametrize("gi", range(3))
def test_fc_matches_reference(gi):
    x, w, bias, gy = (KER[f"fc{gi}_{t}"] for t in ("x", "w", "b", "gy"))
    assert rel(K.fc_forward(x, w, bias), KER[f"fc{gi}_y"]) < 1e-13
    for got, key in zip(K.fc_backward(x, w, gy), ("gx", "gw", "gb")):
        assert rel(got, KER[f"fc{gi}_{key}"]) < 1e-13


def test_relu_matches_reference_bit_exact():
    x, g = KER["relu_x"], KER["relu_g"]
    assert np.array_equal(K.relu_forward(x), KER["relu_y"])
    assert np.array_equal(K.relu_backward(x, g), KER["relu_gx"])


@pytest.mark.parametrize("gi", range(4))
def test_maxpool_matches_reference_bit_exact(gi):
    x, (k, s), gy = KER[f"pool{gi}_x"], KER[f"pool{gi}_ks"], KER[f"pool{gi}_gy"]
    y, arg = K.maxpool_forward(x, k, s)
    assert np.array_equal(y, KER[f"pool{gi}_y"])
    assert np.array_equal(arg, KER[f"pool{gi}_arg"])
    assert np.array_equal(K.maxpool_backward(x.shape, k, s, gy, arg), KER[f"pool{gi}_gx"])


@pytest.mark.parametrize("gi", range(3))
def test_softmax_matches_reference(gi):
    loss, grad = K.softmax_xent_scaled(KER[f"sm{gi}_logits"], KER[f"sm{gi}_labels"],
                                       float(KER[f"sm{gi}_scale"]))
    assert abs(loss - float(KER[f"sm{gi}_loss"])) <= 1e-13 * max(1.0, abs(loss))
    assert rel(grad, KER[f"sm{gi}_grad"]) < 1e-13
    assert np.all(np.isfinite(grad))


def test_sgd_matches_reference_bit_exact():
    ps = [KER["sgd_p0"], KER["sgd_p1"]]
    gs = [KER["sgd_g0"], KER["sgd_g1"]]
    vs = [KER["sgd_v0"], KER["sgd_v1"]]
    newp, newv = K.sgd_step(ps, gs, vs)
    for i in range(2):
        assert np.array_equal(newp[i], KER[f"sgd_np{i}"])
        assert np.array_equal(newv[i], KER[f"sgd_nv{i}"])


# --- the reference's own known-answer tests, restated (pkg/tests/test_kernels.py) ---

def test_kat_conv_nine_ones():
    x = np.ones((1, 1, 3, 3))
    assert K.conv2d_forward(x, np.ones((1, 1, 3, 3)), np.zeros(1), 1, 0)[0, 0, 0, 0] == 9.0


def test_kat_maxpool_ties_first_and_overlap_sum():
    y, arg = K.maxpool_forward(np.full((1, 1, 2, 2), 5.0), 2, 2)
    assert arg[0, 0, 0, 0] == 0
    x = np.zeros((1, 1, 5, 5))
    x[0, 0, 2, 2] = 1.0
    y, arg = K.maxpool_forward(x, 3, 2)
    gx = K.maxpool_backward(x.shape, 3, 2, np.ones_like(y), arg)
    assert gx[0, 0, 2, 2] == 4.0


def test_kat_softmax_uniform_is_ln_k():
    loss, grad = K.softmax_xent(np.zeros((3, 7)), [0, 3, 6])
    assert abs(loss - np.log(7)) < 1e-12
    assert np.allclose(grad.sum(axis=1), 0.0, atol=1e-12)
    with pytest.raises(ValueError):
        K.softmax_xent(np.zeros((1, 7)), [7])


def test_kat_sgd_two_step_recurrence():
    p0, g = np.array([1.0, -2.0]), np.array([0.5, 0.25])
    p, v = [p0], [np.zeros(2)]
    for _ in range(2):
        p, v = K.sgd_step(p, [g], v, 0.01, 0.9, 0.0)
    assert np.allclose(v[0], -0.019 * g, rtol=1e-14)
    assert np.allclose(p[0], p0 - 0.029 * g, rtol=1e-14)


# --- step engine vs reference trajectories ---

def _tree(prefix, idxs):
    return {i: {k: STEPS[f"{prefix}_{i}_{k}"] for k in ("w", "b")} for i in idxs}


def test_reference_step_tinynet_trajectory():
    net = load_network(CONFIGS / "tinynet.net")
    params = _tree("tiny_p0", (0, 3, 5, 7))
    vel = None
    for st in range(3):
        loss, params, vel = reference_step(net, params, (STEPS[f"tiny_x{st}"], STEPS[f"tiny_y{st}"]), vel)
        assert abs(loss - float(STEPS[f"tiny_loss{st}"])) < 1e-12
        ref = _tree(f"tiny_p{st + 1}", (0, 3, 5, 7))
        for i in ref:
            for k in ("w", "b"):
                assert rel(params[i][k], ref[i][k]) < 1e-12


def test_init_matches_reference_digest():
    net = load_network(CONFIGS / "alexnet_small64.net")
    p = init_dense_params(net, 3)
    for i, t in p.items():
        for k, v in t.items():
            v = v.astype(np.float32).astype(np.float64)
            dig = STEPS[f"small64_p0_{i}_{k}"]
            assert abs(v.sum() - dig[0]) < 1e-9 and abs(np.sqrt((v ** 2).sum()) - dig[1]) < 1e-9


def test_reference_step_small64_digests():
    net = load_network(CONFIGS / "alexnet_small64.net")
    params = {i: {k: v.astype(np.float32).astype(np.float64) for k, v in t.items()}
              for i, t in init_dense_params(net, 3).items()}
    vel = None
    for st in range(2):
        old = params
        loss, params, vel = reference_step(net, params, (STEPS[f"small64_x{st}"], STEPS[f"small64_y{st}"]), vel)
        assert abs(loss - float(STEPS[f"small64_loss{st}"])) < 1e-11
        for i in params:
            for k in ("w", "b"):
                d = params[i][k] - old[i][k]
                dig = STEPS[f"small64_d{st + 1}_{i}_{k}"]
                assert abs(np.sqrt((d ** 2).sum()) - dig[1]) <= 1e-9 * max(dig[1], 1e-12)


PLANS = {"d2m1": ParallelPlan(2, 1), "d1m2x3": ParallelPlan(1, 2, (3,)),
         "d2m2x3": ParallelPlan(2, 2, (3,)), "d1m4x3": ParallelPlan(1, 4, (3,)),
         "d1m2grp": ParallelPlan(1, 2, ())}


@pytest.mark.parametrize("pname", sorted(PLANS))
def test_oracle_fabric_matches_hybrid_step(pname):
    plan = PLANS[pname]
    net = load_network(CONFIGS / "tinynet.net")
    fab = OracleFabric(net, plan, _tree("tiny_p0", (0, 3, 5, 7)))
    for st in range(2):
        loss = fab.step(STEPS[f"tiny_x{st}"], STEPS[f"tiny_y{st}"])
        assert abs(loss - float(STEPS[f"hyb_{pname}_loss{st}"])) < 1e-12
    for j in range(plan.model_columns):
        for i in (0, 3, 5, 7):
            for k in ("w", "b"):
                ref = STEPS[f"hyb_{pname}_col{j}_{i}_{k}"]
                assert rel(fab.params[j][i][k], ref) < 1e-12


def test_alexnet_reference_step_digest():
    g = np.load(GOLDEN / "alexnet.npz")
    net = load_network(CONFIGS / "alexnet.net")
    params = {i: {k: v.astype(np.float32).astype(np.float64) for k, v in t.items()}
              for i, t in init_dense_params(net, 0).items()}
    x = g["x"].astype(np.float64)
    loss, newp, _ = reference_step(net, params, (x, g["y"]))
    assert abs(loss - float(g["loss"])) < 1e-10
    for i in params:
        for k in ("w", "b"):
            d = newp[i][k] - params[i][k]
            dig = g[f"d_{i}_{k}"]
            assert abs(np.sqrt((d ** 2).sum()) - dig[1]) <= 1e-9 * max(dig[1], 1e-15)


EVAL = np.load(GOLDEN / "eval.npz")
EVAL_CASES = {"tiny_d1m2x3": ("tinynet", (1, 2, (3,))), "tiny_d2m2x3": ("tinynet", (2, 2, (3,))),
              "tiny_d2m1": ("tinynet", (2, 1, ())), "small64_d1m2x6": ("alexnet_small64", (1, 2, (6,)))}


@pytest.mark.parametrize("name", sorted(EVAL_CASES))
def test_oracle_evaluation_errors_match_reference(name):
    """evaluation_errors after one step (`schemes.py:600-645`) vs the reference's count.
    (Dropout-free nets: the forward is deterministic in the oracle.)"""
    from paper_1312_5853_b200.netdef import load_network
    from paper_1312_5853_b200.plan import ParallelPlan, init_dense_params
    from oracle.ref_engine import OracleFabric
    net_name, (d, m, cross) = EVAL_CASES[name]
    net = load_network(CONFIGS / f"{net_name}.net")
    params = {i: {k: v.astype(np.float32).astype(np.float64) for k, v in t.items()}
              for i, t in init_dense_params(net, 3).items()}
    of = OracleFabric(net, ParallelPlan(d, m, cross), params)
    of.step(EVAL[f"{name}_x"].astype(np.float64), EVAL[f"{name}_y"])
    got = of.evaluation_errors(EVAL[f"{name}_tx"], EVAL[f"{name}_ty"])
    assert got == int(EVAL[f"{name}_wrong"])
