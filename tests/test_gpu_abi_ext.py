"""GPU tests of the step-program helpers added to the C ABI this round, called
directly through it: the shared-memory-free bias gradient, the prepared
data-gradient filters (PC_WT_PRESET), the all-ones space-to-depth channel and
the input-layer gradient finish, and the per-thread GEMM grid cap."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _lib():
    from paper_1312_5853_b200 import _lib as L
    return L, L.lib()


@pytest.mark.parametrize("P,N,prec", [(186624, 256, "bf16"), (43264, 384, "bf16"), (256, 4096, "bf16"),
                                      (1000, 24, "fp32"), (7, 8, "bf16")])
def test_bias_grad_matches_column_sums(P, N, prec):
    import torch
    L, lib = _lib()
    dt = torch.bfloat16 if prec == "bf16" else torch.float32
    g = torch.randn(P, N, device="cuda").to(dt)
    ctas = 296
    ws = torch.empty(max(lib.raw("pc_bias_grad_workspace")(P, N, ctas), 16), dtype=torch.uint8, device="cuda")
    out = torch.empty(N, device="cuda")
    lib.call("pc_bias_grad", P, N, g.data_ptr(), L.PC_BF16 if prec == "bf16" else L.PC_FP32, out.data_ptr(),
             ws.data_ptr(), ws.numel(), ctas, torch.cuda.current_stream().cuda_stream)
    want = g.double().sum(0)
    got = out.double()
    assert float((got - want).abs().max() / want.abs().max().clamp_min(1.0)) < 1e-5
    # deterministic: a second call gives the same bits
    out2 = torch.empty_like(out)
    lib.call("pc_bias_grad", P, N, g.data_ptr(), L.PC_BF16 if prec == "bf16" else L.PC_FP32, out2.data_ptr(),
             ws.data_ptr(), ws.numel(), ctas, torch.cuda.current_stream().cuda_stream)
    assert torch.equal(out, out2)


@pytest.mark.parametrize("geom", [(4, 96, 27, 27, 256, 5, 1, 2), (4, 256, 13, 13, 384, 3, 1, 1),
                                  (2, 384, 13, 13, 256, 3, 1, 1)])
def test_prepared_dgrad_weights_give_identical_data_gradient(geom):
    import torch
    L, lib = _lib()
    B, Ci, H, W, N, k, s, p = geom
    Ho = (H + 2 * p - k) // s + 1
    g = L.ConvGeom(B, H, W, Ci, N, k, s, p, Ho, Ho, Ci, 0)
    x = torch.randn(B * H * W * Ci, device="cuda").bfloat16()
    w = (torch.randn(N * k * k * Ci, device="cuda") * 0.05).bfloat16()
    gy = torch.randn(B * Ho * Ho * N, device="cuda").bfloat16()
    wsb = lib.raw("pc_conv2d_backward_workspace")(C.byref(g), L.PC_BF16)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    gx0, gx1 = torch.empty_like(x), torch.empty_like(x)
    lib.call("pc_conv2d_backward", C.byref(g), x.data_ptr(), w.data_ptr(), gy.data_ptr(), gx0.data_ptr(), None,
             None, None, L.PC_BF16, L.PC_WANT_DX, ws.data_ptr(), wsb, st)
    wt = torch.empty_like(w)
    lib.call("pc_conv2d_dgrad_weights", C.byref(g), w.data_ptr(), wt.data_ptr(), L.PC_BF16, st)
    lib.call("pc_conv2d_backward", C.byref(g), x.data_ptr(), wt.data_ptr(), gy.data_ptr(), gx1.data_ptr(), None,
             None, None, L.PC_BF16, L.PC_WANT_DX | L.PC_WT_PRESET, ws.data_ptr(), wsb, st)
    assert torch.equal(gx0, gx1)


def test_space_to_depth_ones_channel_and_bias_from_wgrad():
    """The all-ones padding channel's tap-(0,0) weight gradient equals the bias
    gradient computed by the two-pass column sum."""
    import torch
    L, lib = _lib()
    from paper_1312_5853_b200 import layout
    B, Cin, H, s, kk, N = 4, 3, 227, 4, 11, 96
    x = torch.randn(B, Cin, H, H, device="cuda").bfloat16()
    Hs = layout.s2d_extent(H, kk, s, 0)[0]
    st = torch.cuda.current_stream().cuda_stream
    xs = torch.empty(B * Hs * Hs * 64, device="cuda", dtype=torch.bfloat16)
    lib.call("pc_space_to_depth_ex", B, Cin, H, H, s, 0, 64, x.data_ptr(), L.PC_BF16, 48, xs.data_ptr(), st)
    v = xs.view(B, Hs, Hs, 64).float()
    assert torch.all(v[..., 48] == 1.0) and torch.all(v[..., 49:] == 0.0)
    ref = torch.empty_like(xs)
    lib.call("pc_space_to_depth", B, Cin, H, H, s, 0, 64, x.data_ptr(), L.PC_BF16, ref.data_ptr(), st)
    assert torch.equal(v[..., :48], ref.view(B, Hs, Hs, 64).float()[..., :48])
    k3 = -(-kk // s)
    Ho = Hs - k3 + 1
    g = L.ConvGeom(B, Hs, Hs, 64, N, k3, 1, 0, Ho, Ho, 64, 0)
    gy = torch.randn(B * Ho * Ho * N, device="cuda").bfloat16()
    wsb = lib.raw("pc_conv2d_backward_workspace")(C.byref(g), L.PC_BF16)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    w = torch.zeros(N * k3 * k3 * 64, device="cuda").bfloat16()
    gw = torch.empty(N * k3 * k3 * 64, device="cuda")
    gb_ref, gb = torch.empty(N, device="cuda"), torch.empty(N, device="cuda")
    lib.call("pc_conv2d_backward", C.byref(g), xs.data_ptr(), w.data_ptr(), gy.data_ptr(), None, None,
             gw.data_ptr(), gb_ref.data_ptr(), L.PC_BF16, L.PC_WANT_DW, ws.data_ptr(), wsb, st)
    keep = torch.from_numpy(layout.s2d_keep_mask(N, Cin, kk, s, 64).reshape(-1)).cuda()
    lib.call("pc_s2d_wgrad_finish", N, k3 * k3 * 64, 48, keep.data_ptr(), gw.data_ptr(), gb.data_ptr(), st)
    torch.cuda.synchronize()
    assert float((gb - gb_ref).abs().max() / gb_ref.abs().max()) < 1e-5
    assert torch.all(gw.view(N, k3, k3, 64)[..., 48:] == 0.0)


def test_grid_cap_keeps_results_bit_identical():
    import torch
    L, lib = _lib()
    B, Ci, H, N, k = 8, 256, 13, 384, 3
    g = L.ConvGeom(B, H, H, Ci, N, k, 1, 1, H, H, Ci, 0)
    x = torch.randn(B * H * H * Ci, device="cuda").bfloat16()
    w = (torch.randn(N * k * k * Ci, device="cuda") * 0.05).bfloat16()
    bias = torch.zeros(N, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    outs = []
    for cap in (0, 20, 2):
        y = torch.empty(B * H * H * N, device="cuda", dtype=torch.bfloat16)
        lib.call("pc_set_grid_cap", cap)
        try:
            lib.call("pc_conv2d_forward", C.byref(g), x.data_ptr(), w.data_ptr(), bias.data_ptr(), y.data_ptr(),
                     L.PC_BF16, 1, st)
        finally:
            lib.call("pc_set_grid_cap", 0)
        outs.append(y)
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])


@pytest.mark.parametrize("shape", [(8, 27, 27, 256), (4, 13, 13, 128), (3, 55, 55, 64)])
def test_pool_backward_bias_matches_plain_backward_and_column_sums(shape):
    import torch
    L, lib = _lib()
    B, H, W, Cc = shape
    Ho, Wo = (H - 3) // 2 + 1, (W - 3) // 2 + 1
    st = torch.cuda.current_stream().cuda_stream
    x = torch.randn(B * H * W * Cc, device="cuda").relu().bfloat16()
    y = torch.empty(B * Ho * Wo * Cc, device="cuda", dtype=torch.bfloat16)
    arg = torch.empty(B * Ho * Wo * Cc, device="cuda", dtype=torch.uint8)
    lib.call("pc_maxpool_forward", B, H, W, Cc, 3, 2, x.data_ptr(), y.data_ptr(), arg.data_ptr(), L.PC_BF16, st)
    gy = torch.randn(B * Ho * Wo * Cc, device="cuda").bfloat16()
    gx0, gx1 = torch.empty_like(x), torch.empty_like(x)
    lib.call("pc_maxpool_backward", B, H, W, Cc, 3, 2, gy.data_ptr(), arg.data_ptr(), None, gx0.data_ptr(),
             L.PC_BF16, st)
    ws = torch.empty(lib.raw("pc_maxpool_backward_bias_workspace")(Cc), dtype=torch.uint8, device="cuda")
    gb = torch.empty(Cc, device="cuda")
    lib.call("pc_maxpool_backward_bias", B, H, W, Cc, 3, 2, gy.data_ptr(), arg.data_ptr(), None, gx1.data_ptr(),
             L.PC_BF16, gb.data_ptr(), ws.data_ptr(), ws.numel(), st)
    assert torch.equal(gx0, gx1)
    want = gx0.view(-1, Cc).double().sum(0)
    assert float((gb.double() - want).abs().max() / want.abs().max()) < 1e-5
