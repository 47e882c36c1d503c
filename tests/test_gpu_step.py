"""Step-level parity on the B200: the drop-in scheme API vs the reference's
trajectories (golden fixtures written by the reference itself) and vs the
float64 oracle, layer by layer.

fp32 mode bound (north_star): <= 1e-5 relative (max-normalised)
on losses, activations, gradients and updates. bf16 mode: loss <= 1e-2
relative, weight updates <= 0.3 rel-L2. Max-pool decisions: see parity.py
(near-ties may flip end to end; every flip is checked to be a near-tie and
replayed in the oracle).
"""

import numpy as np
import pytest

from conftest import CONFIGS, GOLDEN
from parity import oracle_replay, rel, rel_l2

pytestmark = pytest.mark.gpu

STEPS = np.load(GOLDEN / "steps.npz")
TOL = 1e-5


def tree(prefix, idxs):
    return {i: {k: STEPS[f"{prefix}_{i}_{k}"] for k in ("w", "b")} for i in idxs}


def f32_params(params):
    return {i: {k: v.astype(np.float32).astype(np.float64) for k, v in t.items()} for i, t in params.items()}


def test_library_reports_device():
    from paper_1312_5853_b200._lib import lib
    assert lib().dll.pc_version() == 1
    assert lib().dll.pc_has_tcgen05() == 1


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
    from paper_1312_5853_b200.plan import plan_columnized
    from paper_1312_5853_b200.schemes import column_params
    d, m, cross = PLANS[pname]
    net = P.load_network(CONFIGS / "tinynet.net")
    plan = P.ParallelPlan(d, m, cross)
    cs = plan_columnized(net, plan)
    fab = P.spawn(plan.workers, precision="fp32")
    P.setup_workers(fab, plan, cs, tree("tiny_p0", (0, 3, 5, 7)), P.SgdState())
    for st in range(2):
        res = P.hybrid_step(fab, plan, cs, STEPS[f"tiny_x{st}"], STEPS[f"tiny_y{st}"])
        ref = float(STEPS[f"hyb_{pname}_loss{st}"])
        assert abs(res.loss - ref) / abs(ref) < TOL
        led = STEPS[f"hyb_{pname}_ledger{st}"]
        assert (res.ledger_bytes, res.ledger_messages) == (int(led[0]), int(led[1]))
    for j in range(m):
        got = column_params(fab, j)
        for i in (0, 3, 5, 7):
            for k in ("w", "b"):
                assert rel(got[i][k], STEPS[f"hyb_{pname}_col{j}_{i}_{k}"]) < TOL


def test_small64_layer_by_layer_fp32():
    """Config #1 net, Krizhevsky two-column plan: every layer's forward output,
    every parameter gradient vs the oracle (B=4)."""
    import paper_1312_5853_b200 as P
    from paper_1312_5853_b200.plan import plan_columnized
    net = P.load_network(CONFIGS / "alexnet_small64.net")
    plan = P.ParallelPlan(1, 2, (6,))
    cs = plan_columnized(net, plan)
    dense = f32_params(P.init_dense_params(net, 3))
    x, y = STEPS["small64_x0"], STEPS["small64_y0"]
    fab = P.spawn(2, precision="fp32")
    P.setup_workers(fab, plan, cs, dense, P.SgdState())
    res = P.hybrid_step(fab, plan, cs, x, y)
    _, oloss, trace, _ = oracle_replay(net, plan, dense, x, y, fab)
    assert abs(res.loss - oloss) / abs(oloss) < TOL
    for j in range(2):
        eng = fab._engines[j]
        for i, cl in enumerate(cs.col_layers):
            st = eng.layers[i]
            if st.kind == "softmax" or (st.kind == "relu" and st.relu_fused_fwd):
                continue
            ref_idx = cl.index + 1 if st.relu_after else cl.index   # fused ReLU output
            assert rel(eng.activation_host(i, "out"), trace["fwd"][ref_idx][j]) < TOL, cl.index
        for i, t in eng.grads_host().items():
            for k in ("w", "b"):
                assert rel(t[k], trace["grads"][j][i][k]) < TOL, (j, i, k)


def test_small64_dense_two_steps_fp32_match_reference():
    """Config #1 net (reference CPU default config), dense plan, 2 steps vs the
    reference's own losses and update digests (golden)."""
    import paper_1312_5853_b200 as P
    net = P.load_network(CONFIGS / "alexnet_small64.net")
    plan = P.ParallelPlan(1, 1)
    cs = P.columnize(net, 1)
    dense = f32_params(P.init_dense_params(net, 3))
    fab = P.spawn(1, precision="fp32")
    P.setup_workers(fab, plan, cs, dense, P.SgdState())
    prev = dense
    for st in range(2):
        res = P.hybrid_step(fab, plan, cs, STEPS[f"small64_x{st}"], STEPS[f"small64_y{st}"])
        ref = float(STEPS[f"small64_loss{st}"])
        assert abs(res.loss - ref) / ref < TOL
        cur = fab._engines[0].params_host()
        for i in (13, 15, 17):       # above every pool (conv layers: see the replayed tests)
            for k in ("w", "b"):
                d = cur[i][k] - prev[i][k]
                dig = STEPS[f"small64_d{st + 1}_{i}_{k}"]
                # fp32 storage of p bounds the update's precision at ~6e-8 |p| per element
                assert abs(np.sqrt((d ** 2).sum()) - dig[1]) <= 1e-3 * dig[1], (st, i, k)
        prev = cur


def test_alexnet_b2_fp32_matches_reference():
    """AlexNet-227, B=2, dense plan: loss and every layer's update vs the
    reference's own step (golden digests) and vs the oracle replaying the
    device's pool decisions."""
    import paper_1312_5853_b200 as P
    from paper_1312_5853_b200.plan import lists_as_params
    g = np.load(GOLDEN / "alexnet.npz")
    net = P.load_network(CONFIGS / "alexnet.net")
    plan = P.ParallelPlan(1, 1)
    cs = P.columnize(net, 1)
    dense = f32_params(P.init_dense_params(net, 0))
    x, y = g["x"].astype(np.float64), g["y"]
    fab = P.spawn(1, precision="fp32")
    P.setup_workers(fab, plan, cs, dense, P.SgdState())
    res = P.hybrid_step(fab, plan, cs, x, y)
    assert abs(res.loss - float(g["loss"])) / float(g["loss"]) < TOL
    # first step from zero velocity: the velocity IS the update p1 - p0, in fp32
    vel = fab._engines[0].velocity_host()
    for i in (13, 15, 17):   # above every pool: no tie routing involved -> direct reference digests
        for k in ("w", "b"):
            dig = g[f"d_{i}_{k}"]
            assert abs(np.sqrt((vel[i][k] ** 2).sum()) - dig[1]) <= TOL * dig[1], (i, k)
            assert abs(np.abs(vel[i][k]).max() - dig[2]) <= TOL * dig[2], (i, k)
    of, oloss, _, flips = oracle_replay(net, plan, dense, x, y, fab)
    ovel = lists_as_params(of.velocity[0], cs)
    for i in vel:
        for k in ("w", "b"):
            assert rel(vel[i][k], ovel[i][k]) < TOL, (i, k, flips)


def test_alexnet_krizhevsky_columns_bf16_bounds():
    """AlexNet-227 two-column cross(6) plan in bf16 tensor-core mode vs the
    float64 oracle: loss and update bounds of the bf16 contract."""
    import paper_1312_5853_b200 as P
    from paper_1312_5853_b200.plan import plan_columnized, split_params
    from paper_1312_5853_b200.schemes import column_params
    net = P.load_network(CONFIGS / "alexnet.net")
    plan = P.ParallelPlan(1, 2, (6,))
    cs = plan_columnized(net, plan)
    dense = f32_params(P.init_dense_params(net, 0, std=0.01))
    tr, _ = P.gen_synthetic(4, 1, net.input_shape, seed=1)
    x, y = tr.images, np.array([0, 17, 999, 500])
    fab = P.spawn(2, precision="bf16")
    P.setup_workers(fab, plan, cs, dense, P.SgdState())
    res = P.hybrid_step(fab, plan, cs, x, y)
    of, oloss, _, _ = oracle_replay(net, plan, dense, x, y, fab)
    assert abs(res.loss - oloss) / oloss < 1e-2
    for j in range(2):
        got = column_params(fab, j)
        start = split_params(dense, cs, j)
        for i in got:
            d_got = got[i]["w"] - start[i]["w"]
            d_ref = of.params[j][i]["w"] - start[i]["w"]
            assert rel_l2(d_got, d_ref) < 0.3, (j, i)


def test_bf16_dp_and_hybrid_match_single_worker_bf16():
    """Scheme equivalence on the device in bf16: d2 x m1 and d2 x m2 (cross 3)
    follow the single-worker bf16 trajectory (tinynet, 3 steps)."""
    import paper_1312_5853_b200 as P
    net = P.load_network(CONFIGS / "tinynet.net")
    out = P.run_equivalence(net, [P.ParallelPlan(2, 1), P.ParallelPlan(1, 2, (3,))], steps=3,
                            batch=8, precision="bf16")
    for dv in out:
        assert dv.loss_rel < 2e-2, dv


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


def test_equivalence_fp32_all_small_grids():
    """run_equivalence over every grid up to 4 workers (reference
    `tests/test_trainer.py:220-231`), fp32 mode, 1e-5."""
    import paper_1312_5853_b200 as P
    net = P.load_network(CONFIGS / "tinynet.net")
    plans = [P.ParallelPlan(2, 1), P.ParallelPlan(4, 1), P.ParallelPlan(1, 2, (3,)),
             P.ParallelPlan(2, 2, (3,)), P.ParallelPlan(1, 4, (3,))]
    for dv in P.run_equivalence(net, plans, steps=4, batch=8, precision="fp32"):
        assert dv.worst < 1e-5, dv


def test_alexnet_input_layer_space_to_depth_bf16():
    """The bf16 input layer (11x11/s4 over 3 channels) runs as a 3x3/s1 conv over
    4x4 space-to-depth blocks. Against the float64 oracle on the same
    bf16-rounded operands: forward (bias+ReLU fused, bf16 store) within 2^-7,
    weight and bias gradients (fed the device's own upstream gradient) within
    1e-3; the regrouped weights' structural zeros stay exactly zero after SGD."""
    import torch
    import paper_1312_5853_b200 as P
    from oracle import ref_kernels as O
    net = P.load_network(CONFIGS / "alexnet.net")
    plan = P.ParallelPlan(1, 1)
    cs = P.columnize(net, 1)
    dense = f32_params(P.init_dense_params(net, 0, std=0.01))
    tr, _ = P.gen_synthetic(4, 1, net.input_shape, seed=2)
    x, y = tr.images, np.array([3, 1, 2, 0])
    fab = P.spawn(1, precision="bf16")
    fab.fuse_sgd = False   # gradients are read back below
    P.setup_workers(fab, plan, cs, dense, P.SgdState())
    P.hybrid_step(fab, plan, cs, x, y)
    eng = fab._engines[0]
    st0 = eng.layers[0]
    assert st0.s2d == 4 and st0.geom.k == 3 and st0.geom.stride == 1 and st0.geom.C == 64

    def bf(a):
        return torch.as_tensor(np.asarray(a, np.float32)).bfloat16().double().numpy()

    xb, wb = bf(x), bf(dense[0]["w"])
    want = O.relu_forward(O.conv2d_forward(xb, wb, dense[0]["b"], 4, 0))
    got = eng.activation_host(0, "out")
    assert rel(got, want) < 2.0 ** -7
    ho = st0.out_nhwc
    gy = st0.gout[: 4 * ho[0] * ho[1] * ho[2]].float().cpu().numpy().astype(np.float64)
    gy = gy.reshape(4, *ho).transpose(0, 3, 1, 2)
    _, gw, gb = O.conv2d_backward(xb, wb, gy, 4, 0)
    grads = eng.grads_host()
    assert rel(grads[0]["w"], gw) < 1e-3
    assert rel(grads[0]["b"], gb) < 1e-3
    keep = st0.keep.cpu().numpy().astype(bool)
    wdev = eng.p32[st0.w_off: st0.w_off + keep.size].cpu().numpy()
    assert np.all(wdev[~keep] == 0.0) and np.any(wdev[keep] != 0.0)


def test_fused_sgd_epilogue_matches_separate_update():
    """Fused momentum-SGD (single-replica plans, the default): the weight-gradient
    kernels update p/v in place (FC: TMA epilogue on the fp32 accumulator; conv:
    split-K reduction epilogue) instead of the multi-tensor SGD launch; parameters
    after two steps match the unfused run (same fp32 update arithmetic, up to FMA
    contraction)."""
    import paper_1312_5853_b200 as P
    net = P.load_network(CONFIGS / "alexnet_small64.net")
    plan = P.ParallelPlan(1, 1)
    cs = P.columnize(net, 1)
    dense = f32_params(P.init_dense_params(net, 5))
    tr, _ = P.gen_synthetic(100, 1, net.input_shape, seed=4)
    x, y = tr.images[:16], tr.labels[:16]
    out = []
    for fuse in (False, True):
        fab = P.spawn(1, precision="bf16")
        fab.fuse_sgd = fuse
        P.setup_workers(fab, plan, cs, dense, P.SgdState())
        losses = [P.hybrid_step(fab, plan, cs, x, y).loss for _ in range(2)]
        assert fab._engines[0].fuse_sgd == fuse
        out.append((losses, P.gather_dense_params(fab, plan, cs)))
    (l0, p0), (l1, p1) = out
    assert abs(l0[1] - l1[1]) <= 1e-6 * abs(l0[1])
    for i in p0:
        for k in ("w", "b"):
            assert rel(p1[i][k] - dense[i][k], p0[i][k] - dense[i][k]) < 1e-5, (i, k)


def test_train_device_resident_feed_matches_host_feed_and_oracle():
    """trainer.train (reference `trainer.py:99-154`) with the batch gathered on the
    device from an HBM-resident copy of the dataset gives the
    same trajectory as the host-gathered feed, and both follow the float64
    oracle over the same rng.permutation batch order (fp32 mode, 1e-5)."""
    import paper_1312_5853_b200 as P
    from oracle.ref_engine import OracleFabric
    from paper_1312_5853_b200 import rng
    net = P.load_network(CONFIGS / "tinynet.net")
    train_set, _ = P.gen_synthetic(10, 4, net.input_shape, seed=3)
    plan = P.ParallelPlan(2, 1)
    runs = []
    for dev in (True, False):
        cfg = P.TrainConfig(net=net, plan=plan, epochs=2, batch=8, seed=5, train_data=train_set,
                            precision="fp32", device_data=dev)
        runs.append([r.train_loss for r in P.train(cfg).records])
    assert runs[0] == runs[1]
    of = OracleFabric(net, plan, P.init_dense_params(net, 5))
    want = []
    for epoch in range(2):
        order = rng.permutation(5, epoch, train_set.size)
        for step in range(train_set.size // 8):
            idx = order[step * 8:(step + 1) * 8]
            want.append(of.step(train_set.images[idx], train_set.labels[idx]))
    assert len(want) == len(runs[0])
    for got, ref in zip(runs[0], want):
        assert abs(got - ref) / abs(ref) < 1e-5


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_train_device_resident_feed_single_replica_pipelined_upload(precision):
    """d = 1 (the pipelined-upload path: the batch copy runs on its own stream,
    overlapping the previous step's backward). With the batch gathered on the
    device, the copy must wait for the gather, which queues behind that backward
    (ADVICE r01): the device feed must reproduce the host feed bit for bit, and
    follow the oracle."""
    import paper_1312_5853_b200 as P
    from oracle.ref_engine import OracleFabric
    from paper_1312_5853_b200 import rng
    net = P.load_network(CONFIGS / "alexnet_small64.net")
    train_set, _ = P.gen_synthetic(100, 1, net.input_shape, seed=3)
    plan = P.ParallelPlan(1, 1)
    runs = []
    for dev in (True, False):
        cfg = P.TrainConfig(net=net, plan=plan, epochs=2, batch=16, seed=5, train_data=train_set,
                            precision=precision, device_data=dev)
        runs.append([r.train_loss for r in P.train(cfg).records])
    assert runs[0] == runs[1]
    if precision == "fp32":
        of = OracleFabric(net, plan, P.init_dense_params(net, 5))
        want = []
        for epoch in range(2):
            order = rng.permutation(5, epoch, train_set.size)
            for step in range(train_set.size // 16):
                idx = order[step * 16:(step + 1) * 16]
                want.append(of.step(train_set.images[idx], train_set.labels[idx]))
        # the first two steps at the fp32 bound. The free-running trajectory is chaotic
        # (small64, He init, lr 0.01: the loss climbs 9.8 -> 20 -> 60): the oracle itself,
        # restarted from parameters perturbed by 1e-7, is 4e-2 off by step 12, so later
        # steps are compared between the two device feeds only (bit-identical above)
        for n, (got, ref) in enumerate(zip(runs[0][:2], want[:2])):
            assert abs(got - ref) / abs(ref) < 1e-5, n


def test_sync_step_option_returns_after_the_update():
    """fabric.sync_step = True: hybrid_step returns only after the backward and the
    update have finished (the default returns after the forward);
    both give the same trajectory."""
    import torch
    import paper_1312_5853_b200 as P
    net = P.load_network(CONFIGS / "tinynet.net")
    plan = P.ParallelPlan(1, 1)
    cs = P.columnize(net, 1)
    out = []
    for sync in (False, True):
        fab = P.spawn(1, precision="bf16")
        fab.sync_step = sync
        P.setup_workers(fab, plan, cs, tree("tiny_p0", (0, 3, 5, 7)), P.SgdState())
        losses = [P.hybrid_step(fab, plan, cs, STEPS[f"tiny_x{s % 2}"], STEPS[f"tiny_y{s % 2}"]).loss
                  for s in range(3)]
        if sync:
            assert torch.cuda.current_stream().query()
        out.append((losses, fab._engines[0].p32.clone()))
    assert out[0][0] == out[1][0] and torch.equal(out[0][1], out[1][1])


def test_float64_numpy_batch_matches_float32_batch_bit_for_bit():
    """A parconv caller's float64 images travel raw (PC_FP64 source of the input
    kernel): the step is bit-identical to the float32 upload of the same values."""
    import torch
    import paper_1312_5853_b200 as P
    from paper_1312_5853_b200.data import synthetic_rows
    net = P.load_network(CONFIGS / "alexnet.net")
    plan = P.ParallelPlan(1, 1)
    cs = P.columnize(net, 1)
    x, y = synthetic_rows(1000, 1, net.input_shape, 2, np.arange(16) * 37)
    dense = P.init_dense_params(net, 1, std=0.01)
    out = []
    x64 = torch.from_numpy(x.astype(np.float64))
    # float64 numpy, float64 CPU tensor (pageable, pinned: the host-fed trainer's
    # staging buffer), float32 pinned
    for xb in (x.astype(np.float64), x64, x64.pin_memory(), torch.from_numpy(x).pin_memory()):
        fab = P.spawn(1, precision="bf16")
        P.setup_workers(fab, plan, cs, dense, P.SgdState())
        losses = [P.hybrid_step(fab, plan, cs, xb, y).loss for _ in range(3)]
        out.append((losses, fab._engines[0].p32.clone(), fab._runner.x_dev.dtype))
    assert [o[2] for o in out] == [torch.float64] * 3 + [torch.float32]
    for o in out[1:]:
        assert out[0][0] == o[0] and torch.equal(out[0][1], o[1])


@pytest.mark.parametrize("precision,loss_tol,upd_tol", [("bf16", 1e-2, 0.3), ("tf32", 5e-3, 0.1)])
def test_alexnet_reference_plan_cross_3_6_8_10(precision, loss_tol, upd_tol):
    """The reference's shipped two-column plan (cross at conv2, conv3, conv4, conv5 and the
    FC layers) on AlexNet-227 vs the float64 oracle, per column."""
    import paper_1312_5853_b200 as P
    from paper_1312_5853_b200.data import synthetic_rows
    from paper_1312_5853_b200.plan import plan_columnized, split_params
    from paper_1312_5853_b200.schemes import column_params
    net = P.load_network(CONFIGS / "alexnet.net")
    plan = P.ParallelPlan(1, 2, (3, 6, 8, 10))
    cs = plan_columnized(net, plan)
    dense = {i: {k: v.astype(np.float32).astype(np.float64) for k, v in t.items()}
             for i, t in P.init_dense_params(net, 0, std=0.01).items()}
    x, y = synthetic_rows(1000, 1, net.input_shape, 3, np.arange(8) * 113)
    x = x.astype(np.float64)
    fab = P.spawn(2, precision=precision)
    P.setup_workers(fab, plan, cs, dense, P.SgdState())
    res = P.hybrid_step(fab, plan, cs, x, y)
    of, oloss, _, _ = oracle_replay(net, plan, dense, x, y, fab)
    assert abs(res.loss - oloss) / oloss < loss_tol
    for j in range(2):
        got = column_params(fab, j)
        start = split_params(dense, cs, j)
        for i in got:
            d_got = got[i]["w"] - start[i]["w"]
            d_ref = of.params[j][i]["w"] - start[i]["w"]
            assert rel_l2(d_got, d_ref) < upd_tol, (j, i)
