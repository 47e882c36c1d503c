"""Extension layers on the B200: LRN and dropout kernels through
the C ABI against their float64 definition (oracle/ref_kernels.py,
rng.dropout_keep), and training steps of a net using them against the
oracle under several plans. fp32 verification mode: 1e-5; bf16 with the same
operands: 2^-7 on bf16-stored outputs; dropout masks bit-exact."""

import ctypes as C

import numpy as np
import pytest

from conftest import CONFIGS
from parity import rel

pytestmark = pytest.mark.gpu


def _dev(a, dtype):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32)).to(dtype).cuda()


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("C,size", [(48, 5), (96, 5), (256, 9), (44, 5), (16, 3)])
def test_lrn_kernels_match_definition(prec, C, size):
    """C % 8 == 0 and size <= 9: the 8-channel vector kernels (sliding window sums
    across neighbouring groups and the tensor's channel edges); C = 44: scalar."""
    import torch
    from oracle import ref_kernels as O
    from paper_1312_5853_b200 import _lib as L
    lib = L.lib()
    rs = np.random.RandomState(3)
    B, H, W = 3, 5, 7
    x = np.maximum(rs.randn(B, C, H, W), 0.0) * 3.0
    g = rs.randn(B, C, H, W)
    dt, pc = (torch.float32, L.PC_FP32) if prec == "fp32" else (torch.bfloat16, L.PC_BF16)
    xr = _dev(x, dt).float().cpu().double().numpy()      # the operands the device sees
    gr = _dev(g, dt).float().cpu().double().numpy()
    xd, gd = _dev(xr.transpose(0, 2, 3, 1), dt), _dev(gr.transpose(0, 2, 3, 1), dt)
    y, gx = torch.empty_like(xd), torch.empty_like(xd)
    st = torch.cuda.current_stream().cuda_stream
    args = (size, 2.0, 1e-2, 0.75)
    lib.call("pc_lrn_forward", B * H * W, C, *args, xd.data_ptr(), y.data_ptr(), pc, st)
    lib.call("pc_lrn_backward", B * H * W, C, *args, xd.data_ptr(), gd.data_ptr(), gx.data_ptr(), pc, st)
    want_y = O.lrn_forward(xr, *args)
    want_g = O.lrn_backward(xr, gr, *args)
    got_y = y.float().cpu().double().numpy().transpose(0, 3, 1, 2)
    got_g = gx.float().cpu().double().numpy().transpose(0, 3, 1, 2)
    tol = 1e-5 if prec == "fp32" else 2.0 ** -7
    assert rel(got_y, want_y) < tol
    assert rel(got_g, want_g) < tol


def test_dropout_mask_bit_exact_on_a_column_slice():
    """Column 1 of 2 (channels 24..47 of 48), replica rows 8..11 of the global batch."""
    import torch
    from paper_1312_5853_b200 import _lib as L, rng
    lib = L.lib()
    B, H, W, Cc, m, row0, layer, seed, step, p = 4, 3, 5, 24, 2, 8, 7, 11, 5, 0.4
    rs = np.random.RandomState(4)
    x = rs.randn(B, H, W, Cc).astype(np.float32)
    xd = torch.as_tensor(x).cuda()
    y = torch.empty_like(xd)
    ctr = torch.tensor([step], dtype=torch.int64, device="cuda")
    lib.call("pc_dropout", B, H, W, Cc, m * Cc, Cc, row0, seed, ctr.data_ptr(), layer, rng.dropout_threshold(p), p,
             xd.data_ptr(), y.data_ptr(), L.PC_FP32, torch.cuda.current_stream().cuda_stream)
    b = np.arange(B).reshape(B, 1, 1, 1)
    yy = np.arange(H).reshape(1, H, 1, 1)
    xx = np.arange(W).reshape(1, 1, W, 1)
    cc = np.arange(Cc).reshape(1, 1, 1, Cc)
    idx = (row0 + b) * (m * Cc * H * W) + ((Cc + cc) * H + yy) * W + xx
    keep = rng.dropout_keep(seed, step, layer, idx, p)
    got = y.cpu().numpy()
    assert np.array_equal(got != 0, keep & (x != 0))
    assert np.allclose(got[keep], (x / np.float32(1 - p))[keep], rtol=1e-6, atol=0)


@pytest.mark.parametrize("d,m,cross", [(1, 1, ()), (2, 1, ()), (1, 2, (4,)), (2, 2, (4,))])
def test_lrn_dropout_net_fp32_matches_oracle(d, m, cross):
    """Three training steps (the dropout stream advances per step) of a net with
    LRN and dropout, fp32 verification mode vs the float64 oracle."""
    import paper_1312_5853_b200 as P
    from oracle.ref_engine import OracleFabric
    from paper_1312_5853_b200.plan import plan_columnized
    from paper_1312_5853_b200.schemes import column_params
    net = P.load_network(CONFIGS / "tinynet_lrn_dropout.net")
    plan = P.ParallelPlan(d, m, cross)
    cs = plan_columnized(net, plan)
    dense = {i: {k: v.astype(np.float32).astype(np.float64) for k, v in t.items()}
             for i, t in P.init_dense_params(net, 2).items()}
    rs = np.random.RandomState(6)
    x = rs.randn(8, 3, 16, 16).astype(np.float32).astype(np.float64)
    y = rs.randint(0, 10, 8)
    fab = P.spawn(plan.workers, precision="fp32")
    P.setup_workers(fab, plan, cs, dense, P.SgdState())
    of = OracleFabric(net, plan, dense)
    for _ in range(3):
        got = P.hybrid_step(fab, plan, cs, x, y).loss
        want = of.step(x, y)
        assert abs(got - want) / abs(want) < 1e-5
    for j in range(m):
        params = column_params(fab, j)
        for i in params:
            for k in ("w", "b"):
                start = P.split_params(dense, cs, j)[i][k]
                assert rel(params[i][k] - start, of.params[j][i][k] - start) < 1e-4, (j, i, k)


@pytest.mark.parametrize("plan_args", [(1, 1, ()), (1, 2, (8,))])   # 8: conv3 (LRN shifts the indices)
def test_alexnet_lrn_dropout_bf16_bench_config_matches_oracle(plan_args):
    """The bench's second configuration (configs/alexnet_lrn_dropout.net, bf16, every
    default switch) at batch 16, single column and Krizhevsky's two columns: step 1
    against the float64 oracle replaying the device's pool and ReLU decisions (the
    dropout masks come from the same SplitMix64 stream) — loss <= 1e-2, every layer's
    update <= 0.3 rel-L2 — and steps 2-3 (graph captured, replayed) equal to the
    same steps run eagerly."""
    import torch
    import paper_1312_5853_b200 as P
    from oracle.ref_engine import OracleFabric
    from parity import (assert_near_ties, assert_relu_near_ties, device_argmax, device_relu_masks,
                        rel_l2)
    from paper_1312_5853_b200.data import synthetic_rows
    from paper_1312_5853_b200.plan import plan_columnized
    from paper_1312_5853_b200.schemes import column_params
    net = P.load_network(CONFIGS / "alexnet_lrn_dropout.net")
    plan = P.ParallelPlan(*plan_args)
    cs = plan_columnized(net, plan)
    dense = {i: {k: v.astype(np.float32).astype(np.float64) for k, v in t.items()}
             for i, t in P.init_dense_params(net, 0, std=0.01).items()}
    x, y = synthetic_rows(1000, 1, net.input_shape, 4, np.arange(16) * 61)
    x = x.astype(np.float64)
    runs = []
    for graph in ("1", "0"):
        import os
        old = os.environ.get("PC_GRAPH")
        os.environ["PC_GRAPH"] = graph
        try:
            fab = P.spawn(plan.workers, precision="bf16")
            P.setup_workers(fab, plan, cs, dense, P.SgdState())
            losses, snap = [], None
            for s in range(3):
                losses.append(P.hybrid_step(fab, plan, cs, x, y).loss)
                if s == 0 and graph == "1":
                    forced, relu = device_argmax(fab, plan), device_relu_masks(fab, plan)
                    snap = [column_params(fab, j) for j in range(plan.model_columns)]
            runs.append((losses, [e.p32.clone() for _, e in sorted(fab._engines.items())], snap, forced if snap else None,
                         relu if snap else None))
        finally:
            if old is None:
                os.environ.pop("PC_GRAPH", None)
            else:
                os.environ["PC_GRAPH"] = old
    (lg, pg, snap, forced, relu), (le, pe, _, _, _) = runs
    assert lg == le
    for a, b in zip(pg, pe):
        assert torch.equal(a, b)
    of, trace = OracleFabric(net, plan, dense), {}
    oloss = of.step(x, y, trace=trace, force_argmax=forced, force_relu=relu)
    assert_near_ties(trace, forced, of.cs, 2e-2)
    assert_relu_near_ties(trace, relu, 2e-2)
    assert abs(lg[0] - oloss) / abs(oloss) < 1e-2, (lg[0], oloss)
    for j in range(plan.model_columns):
        start = P.split_params(dense, cs, j)
        for i in snap[j]:
            for k in ("w", "b"):
                err = rel_l2(snap[j][i][k] - start[i][k], of.params[j][i][k] - start[i][k])
                assert err < 0.3, (j, i, k, err)
