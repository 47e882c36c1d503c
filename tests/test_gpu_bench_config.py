"""Parity of the exact configurations bench.py measures.

* AlexNet-227, plan d1m1, batch 256, bf16, every default switch of the timed
  step (CUDA-graph replay as two graphs, fused SGD in the weight-gradient
  epilogues, weight gradients on a side stream, prepared data-gradient
  filters, pool-fused bias gradients, programmatic dependent launch):
    - steps 1 (eager), 2 (captured) and 3 (replayed) are bit-identical to the
      same three steps run eagerly (PC_GRAPH=0): losses and fp32 parameters;
    - step 1 vs the float64 oracle (`oracle/`, the restatement of the
      reference `schemes.py:439-458` pinned by tests/test_oracle_golden.py)
      replaying the device's max-pool decisions (tests/parity.py): loss
      <= 1e-2 relative, every layer's update (weights and biases) <= 0.3
      rel-L2 — the bf16 contract of SURVEY §8 c4.
* The same configuration in the fp32 verification mode, one step, <= 1e-5
  (loss, max-normalised update of every tensor).
* Config #1 of BASELINE.json: alexnet_small64 at its stated batch 32, d1m1,
  bf16 and fp32, two steps vs the oracle.

The batch is the bench's: the first 256 images of rng.permutation(0, 0, 1000)
of the 1000-class synthetic set, Gaussian std 0.01 init (seed 0) rounded to
fp32 so the oracle sees the device's starting point exactly.
"""

import numpy as np
import pytest
import torch

from conftest import CONFIGS
from parity import oracle_replay, rel, rel_l2

pytestmark = pytest.mark.gpu


def f32_params(params):
    return {i: {k: v.astype(np.float32).astype(np.float64) for k, v in t.items()} for i, t in params.items()}


def bench_batch(net, b):
    from paper_1312_5853_b200 import rng
    from paper_1312_5853_b200.data import synthetic_rows
    order = rng.permutation(0, 0, 1000)[:b]
    x, y = synthetic_rows(1000, 1, net.input_shape, 0, order)
    return x.astype(np.float64), y


def run_steps(net, dense, x, y, precision, steps, graph: bool, monkeypatch):
    import paper_1312_5853_b200 as P
    monkeypatch.setenv("PC_GRAPH", "1" if graph else "0")
    plan = P.ParallelPlan(1, 1)
    cs = P.columnize(net, 1)
    fab = P.spawn(1, precision=precision)
    P.setup_workers(fab, plan, cs, dense, P.SgdState())
    out = []
    for s in range(steps):
        res = P.hybrid_step(fab, plan, cs, x, y)
        eng = fab._engines[0]
        snap = {"loss": res.loss, "p32": eng.p32.clone()}
        if s == 0:
            from parity import device_argmax, device_relu_masks
            snap["argmax"] = device_argmax(fab, plan)
            snap["relu"] = device_relu_masks(fab, plan)
            snap["velocity"] = eng.velocity_host()   # zero start: v1 = p1 - p0 = the first update
        out.append(snap)
    run = fab._runner
    return fab, out, run


@pytest.fixture(scope="module")
def alexnet():
    import paper_1312_5853_b200 as P
    net = P.load_network(CONFIGS / "alexnet.net")
    dense = f32_params(P.init_dense_params(net, 0, std=0.01))
    x, y = bench_batch(net, 256)
    return net, dense, x, y


def _oracle_first_step(net, dense, x, y, snap, tie_tol):
    """Oracle step 1 replaying the device's step-1 pool and ReLU decisions."""
    from parity import assert_near_ties, assert_relu_near_ties
    from oracle.ref_engine import OracleFabric
    import paper_1312_5853_b200 as P
    from paper_1312_5853_b200.plan import lists_as_params
    plan = P.ParallelPlan(1, 1)
    trace = {}
    of = OracleFabric(net, plan, dense)
    loss = of.step(x, y, trace=trace, force_argmax=snap["argmax"], force_relu=snap["relu"])
    flips = assert_near_ties(trace, snap["argmax"], of.cs, tie_tol)
    flips += assert_relu_near_ties(trace, snap["relu"], tie_tol)
    return loss, lists_as_params(of.velocity[0], of.cs), flips


def test_alexnet_b256_bf16_graph_replay_bit_identical_and_matches_oracle(alexnet, monkeypatch):
    net, dense, x, y = alexnet
    fab, graph_steps, run = run_steps(net, dense, x, y, "bf16", 3, True, monkeypatch)
    # the timed configuration: graphs captured and replayed, split step, fused SGD, side streams
    assert run.replays >= 1 and len(next(iter(run._graphs.values()))) == 2
    eng = fab._engines[0]
    assert eng.fuse_sgd and run.wg_side is not None and run.wt_side is not None
    _, eager_steps, run_e = run_steps(net, dense, x, y, "bf16", 3, False, monkeypatch)
    assert run_e.replays == 0
    for s, (g, e) in enumerate(zip(graph_steps, eager_steps)):
        assert g["loss"] == e["loss"], (s, g["loss"], e["loss"])
        assert torch.equal(g["p32"], e["p32"]), s
    # step 1 vs the float64 oracle (bf16 contract)
    snap = graph_steps[0]
    oloss, ovel, flips = _oracle_first_step(net, dense, x, y, snap, 2e-2)
    assert abs(snap["loss"] - oloss) / abs(oloss) < 1e-2, (snap["loss"], oloss)
    vel = snap["velocity"]
    worst = {}
    for i in vel:
        for k in ("w", "b"):
            worst[(i, k)] = rel_l2(vel[i][k], ovel[i][k])
    assert max(worst.values()) < 0.3, (worst, flips)
    # the losses of the three steps decrease from ln(1000) like the reference's
    assert abs(graph_steps[0]["loss"] - np.log(1000)) < 1e-2


def test_alexnet_b256_fp32_one_step_matches_oracle(alexnet, monkeypatch):
    net, dense, x, y = alexnet
    _, steps, _ = run_steps(net, dense, x, y, "fp32", 1, True, monkeypatch)
    snap = steps[0]
    oloss, ovel, flips = _oracle_first_step(net, dense, x, y, snap, 1e-5)
    assert abs(snap["loss"] - oloss) / abs(oloss) < 1e-5
    vel = snap["velocity"]
    for i in vel:
        for k in ("w", "b"):
            assert rel(vel[i][k], ovel[i][k]) < 1e-5, (i, k, flips)


def test_alexnet_b256_tf32_one_step_matches_oracle(alexnet, monkeypatch):
    """The bench's `--precision tf32` line (float storage, tcgen05 kind::tf32) at its
    batch 256: one step vs the oracle at the TF32 bounds of test_gpu_tf32.py (loss
    <= 5e-3, update <= 0.1 rel-L2), on the tf32 kernels."""
    from paper_1312_5853_b200._lib import lib
    net, dense, x, y = alexnet
    n0 = lib().dll.pc_tf32_contractions()
    _, steps, _ = run_steps(net, dense, x, y, "tf32", 1, True, monkeypatch)
    assert lib().dll.pc_tf32_contractions() > n0
    snap = steps[0]
    oloss, ovel, flips = _oracle_first_step(net, dense, x, y, snap, 2e-2)
    assert abs(snap["loss"] - oloss) / abs(oloss) < 5e-3, (snap["loss"], oloss)
    vel = snap["velocity"]
    for i in vel:
        for k in ("w", "b"):
            assert rel_l2(vel[i][k], ovel[i][k]) < 0.1, (i, k, flips)


@pytest.mark.parametrize("precision,loss_tol,upd_tol", [("fp32", 1e-5, 1e-5), ("bf16", 1e-2, 0.3)])
def test_small64_config1_b32_two_steps(precision, loss_tol, upd_tol):
    """BASELINE configs[0]: alexnet_small64, gen_synthetic(100, 4, (3, 64, 64), 0), B=32, d1m1.
    Per step: loss, and the velocity (= the momentum update, stored directly in
    fp32) of every tensor vs the oracle. bf16: the oracle is re-synchronised to
    the device's parameters after each step, so step 2 measures the step."""
    import paper_1312_5853_b200 as P
    from oracle.ref_engine import OracleFabric
    from paper_1312_5853_b200 import rng
    from paper_1312_5853_b200.plan import lists_as_params, params_as_lists, split_params
    from parity import assert_near_ties, assert_relu_near_ties, device_argmax, device_relu_masks
    net = P.load_network(CONFIGS / "alexnet_small64.net")
    tr, _ = P.gen_synthetic(100, 4, net.input_shape, seed=0)
    dense = f32_params(P.init_dense_params(net, 0))
    order = rng.permutation(0, 0, tr.size)
    plan = P.ParallelPlan(1, 1)
    cs = P.columnize(net, 1)
    fab = P.spawn(1, precision=precision)
    P.setup_workers(fab, plan, cs, dense, P.SgdState())
    of = OracleFabric(net, plan, dense)
    tie = 2e-2 if precision == "bf16" else 1e-5
    for step in range(2):
        idx = order[step * 32:(step + 1) * 32]
        x, y = tr.images[idx], tr.labels[idx]
        res = P.hybrid_step(fab, plan, cs, x, y)
        forced, relu = device_argmax(fab, plan), device_relu_masks(fab, plan)
        trace = {}
        oloss = of.step(x, y, trace=trace, force_argmax=forced, force_relu=relu)
        assert_near_ties(trace, forced, of.cs, tie)
        assert_relu_near_ties(trace, relu, tie)
        assert abs(res.loss - oloss) / abs(oloss) < loss_tol, (step, res.loss, oloss)
        eng = fab._engines[0]
        got = eng.velocity_host()
        want = lists_as_params(of.velocity[0], cs)
        for i in got:
            for k in ("w", "b"):
                err = rel(got[i][k], want[i][k]) if precision == "fp32" else rel_l2(got[i][k], want[i][k])
                assert err < upd_tol, (step, i, k, err)
        if precision == "bf16":
            of.params = [split_params(eng.params_host(), cs, 0)]
            of.velocity = [[np.array(v, dtype=np.float64) for v in params_as_lists(got, cs)]]
