"""Kernel-level parity on the B200 through the C ABI (the reference's unit
tests, `pkg/tests/test_kernels.py`, re-expressed with device tolerances).

fp32 mode: every op vs the reference's golden outputs, <= 1e-5 relative
(max-normalised). bf16 mode: each op fed bf16-rounded operands vs the float64
oracle on the same rounded operands, <= 1e-5 before the output rounding,
i.e. <= 2^-8 relative on bf16-stored outputs. Max-pool argmax
and label handling are bit-exact in both modes.
"""

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import ref_kernels as O

pytestmark = pytest.mark.gpu

KER = np.load(GOLDEN / "kernels.npz")
FP32_TOL = 1e-5
BF16_OUT_TOL = 2.0 ** -7   # bf16 storage of the result (8-bit mantissa) plus accumulation


@pytest.fixture(autouse=True)
def fp32_mode():
    from paper_1312_5853_b200 import kernels as K
    K.set_precision("fp32")
    yield
    K.set_precision("fp32")


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def bf16(a):
    import torch
    return torch.as_tensor(np.asarray(a, np.float32)).bfloat16().float().numpy().astype(np.float64)


@pytest.mark.parametrize("gi", range(5))
def test_conv_fp32(gi):
    from paper_1312_5853_b200 import kernels as K
    b, c, h, w, n, k, s, p = KER[f"conv{gi}_geom"]
    cp = K.ConvParams(KER[f"conv{gi}_w"], KER[f"conv{gi}_b"], int(s), int(p))
    assert rel(K.conv2d_forward(KER[f"conv{gi}_x"], cp), KER[f"conv{gi}_y"]) < FP32_TOL
    gx, gw, gb = K.conv2d_backward(KER[f"conv{gi}_x"], cp, KER[f"conv{gi}_gy"])
    assert rel(gx, KER[f"conv{gi}_gx"]) < FP32_TOL
    assert rel(gw, KER[f"conv{gi}_gw"]) < FP32_TOL
    assert rel(gb, KER[f"conv{gi}_gb"]) < FP32_TOL


@pytest.mark.parametrize("gi", range(3))
def test_fc_fp32(gi):
    from paper_1312_5853_b200 import kernels as K
    x, w, bias, gy = (KER[f"fc{gi}_{t}"] for t in ("x", "w", "b", "gy"))
    assert rel(K.fc_forward(x, w, bias), KER[f"fc{gi}_y"]) < FP32_TOL
    for got, key in zip(K.fc_backward(x, w, gy), ("gx", "gw", "gb")):
        assert rel(got, KER[f"fc{gi}_{key}"]) < FP32_TOL


def test_relu_bit_exact():
    from paper_1312_5853_b200 import kernels as K
    assert np.array_equal(K.relu_forward(KER["relu_x"]), KER["relu_y"])
    assert np.array_equal(K.relu_backward(KER["relu_x"], KER["relu_g"]), KER["relu_gx"])


@pytest.mark.parametrize("gi", range(4))
def test_maxpool_argmax_bit_exact(gi):
    from paper_1312_5853_b200 import kernels as K
    x, (k, s), gy = KER[f"pool{gi}_x"], KER[f"pool{gi}_ks"], KER[f"pool{gi}_gy"]
    y, arg = K.maxpool_forward(x, int(k), int(s))
    assert np.array_equal(y, KER[f"pool{gi}_y"])
    assert np.array_equal(arg, KER[f"pool{gi}_arg"])
    gx = K.maxpool_backward(x, int(k), int(s), gy, arg)
    assert rel(gx, KER[f"pool{gi}_gx"]) < 1e-6


def test_maxpool_ties_and_overlap_kats():
    from paper_1312_5853_b200 import kernels as K
    _, arg = K.maxpool_forward(np.full((1, 1, 2, 2), 5.0), 2, 2)
    assert arg[0, 0, 0, 0] == 0
    x = np.zeros((1, 1, 5, 5))
    x[0, 0, 2, 2] = 1.0
    y, arg = K.maxpool_forward(x, 3, 2)
    assert K.maxpool_backward(x, 3, 2, np.ones_like(y), arg)[0, 0, 2, 2] == 4.0


@pytest.mark.parametrize("gi", range(3))
def test_softmax_fp32(gi):
    from paper_1312_5853_b200 import kernels as K
    loss, grad = K.softmax_xent_scaled(KER[f"sm{gi}_logits"], KER[f"sm{gi}_labels"], float(KER[f"sm{gi}_scale"]))
    assert abs(loss - float(KER[f"sm{gi}_loss"])) <= 1e-5 * max(1.0, abs(float(KER[f"sm{gi}_loss"])))
    assert rel(grad, KER[f"sm{gi}_grad"]) < FP32_TOL
    assert np.all(np.isfinite(grad))


def test_softmax_label_errors_and_uniform():
    from paper_1312_5853_b200 import kernels as K
    from paper_1312_5853_b200.errors import ValidationError
    loss, grad = K.softmax_xent(np.zeros((3, 7)), [0, 3, 6])
    assert abs(loss - np.log(7)) < 1e-6
    assert np.allclose(grad.sum(axis=1), 0.0, atol=1e-7)
    with pytest.raises(ValidationError):
        K.softmax_xent(np.zeros((2, 7)), [1, 7])
    with pytest.raises(ValidationError):
        K.softmax_xent(np.zeros((2, 7)), [-1, 0])


def test_sgd_matches_reference():
    from paper_1312_5853_b200 import kernels as K
    st = K.SgdState(0.01, 0.9, 0.0005, [KER["sgd_v0"], KER["sgd_v1"]])
    newp, newst = K.sgd_step([KER["sgd_p0"], KER["sgd_p1"]], [KER["sgd_g0"], KER["sgd_g1"]], st)
    for i in range(2):
        assert rel(newp[i], KER[f"sgd_np{i}"]) < 1e-6
        assert rel(newst.velocity[i], KER[f"sgd_nv{i}"]) < 1e-6


def test_sgd_two_step_recurrence():
    from paper_1312_5853_b200 import kernels as K
    p0, g = np.array([1.0, -2.0]), np.array([0.5, 0.25])
    st = K.SgdState(0.01, 0.9, 0.0, [np.zeros(2)])
    p = [p0]
    for _ in range(2):
        p, st = K.sgd_step(p, [g], st)
    assert np.allclose(st.velocity[0], -0.019 * g, rtol=1e-6)
    assert np.allclose(p[0], p0 - 0.029 * g, rtol=1e-6)


# ---------------------------------------------------------------- bf16 mode

@pytest.mark.parametrize("geom", [(2, 8, 9, 9, 16, 3, 1, 1), (2, 16, 13, 13, 32, 3, 1, 1),
                                  (2, 3, 23, 23, 8, 11, 4, 0), (1, 32, 27, 27, 64, 5, 1, 2),
                                  (4, 64, 13, 13, 96, 3, 1, 1)])
def test_conv_bf16_same_operands(geom):
    from paper_1312_5853_b200 import kernels as K
    b, c, h, w, n, k, s, p = geom
    rs = np.random.RandomState(7)
    x = bf16(rs.randn(b, c, h, w))
    wt = bf16(rs.randn(n, c, k, k) * 0.2)
    bias = rs.randn(n).astype(np.float32).astype(np.float64) * 0.1
    K.set_precision("bf16")
    cp = K.ConvParams(wt, bias, s, p)
    y = K.conv2d_forward(x, cp)
    yr = O.conv2d_forward(x, wt, bias, s, p)
    assert rel(y, yr) < BF16_OUT_TOL
    gy = bf16(rs.randn(*yr.shape))
    gx, gw, gb = K.conv2d_backward(x, cp, gy)
    rgx, rgw, rgb = O.conv2d_backward(x, wt, gy, s, p)
    assert rel(gx, rgx) < BF16_OUT_TOL
    assert rel(gw, rgw) < 1e-5        # fp32 weight gradients from bf16 operands
    assert rel(gb, rgb) < 1e-5


@pytest.mark.parametrize("shape", [(8, 64, 32), (32, 512, 96), (256, 1024, 1000)])
def test_fc_bf16_same_operands(shape):
    from paper_1312_5853_b200 import kernels as K
    b, d, u = shape
    rs = np.random.RandomState(3)
    x, w = bf16(rs.randn(b, d)), bf16(rs.randn(d, u) * 0.05)
    bias = rs.randn(u).astype(np.float32).astype(np.float64)
    gy = bf16(rs.randn(b, u))
    K.set_precision("bf16")
    assert rel(K.fc_forward(x, w, bias), O.fc_forward(x, w, bias)) < BF16_OUT_TOL
    gx, gw, gb = K.fc_backward(x, w, gy)
    rgx, rgw, rgb = O.fc_backward(x, w, gy)
    assert rel(gx, rgx) < BF16_OUT_TOL
    assert rel(gw, rgw) < 1e-5
    assert rel(gb, rgb) < 1e-5


def test_maxpool_bf16_argmax_bit_exact():
    from paper_1312_5853_b200 import kernels as K
    rs = np.random.RandomState(5)
    x = bf16(np.round(rs.randn(2, 16, 13, 13) * 4) / 4)   # many ties
    K.set_precision("bf16")
    y, arg = K.maxpool_forward(x, 3, 2)
    ry, rarg = O.maxpool_forward(x, 3, 2)
    assert np.array_equal(arg, rarg)
    assert np.array_equal(y, ry)


@pytest.mark.parametrize("case", ["relu_ties", "mixed_sign", "nan_and_negzero"])
def test_maxpool_bf16_simd_fast_path_bit_exact(case):
    """The bf16 3x3/s2 pool compares raw bit patterns (16-bit SIMD) when a window
    holds only non-negative, non-NaN values (ReLU outputs) and falls back to float
    comparison otherwise; both must give np.argmax's first maximum bit-exactly,
    including zero ties, NaN (first NaN wins) and -0 == +0."""
    from paper_1312_5853_b200 import kernels as K
    rs = np.random.RandomState(11)
    x = np.round(rs.randn(3, 24, 15, 15) * 3) / 4
    if case == "relu_ties":
        x = np.maximum(x, 0.0)                      # many exact zeros and value ties
    elif case == "nan_and_negzero":
        x = np.maximum(x, 0.0)
        x[0, :8, 2, 3] = np.nan
        x[1, 5, 4, 4] = np.nan
        x[1, 5, 4, 5] = np.nan
        x[2, :, 0:3, 0:3] = -0.0
        x[2, :4, 1, 1] = 0.0
    x = bf16(x)
    K.set_precision("bf16")
    y, arg = K.maxpool_forward(x, 3, 2)
    ry, rarg = O.maxpool_forward(x, 3, 2)
    assert np.array_equal(arg, rarg)
    assert np.array_equal(np.isnan(y), np.isnan(ry))
    assert np.array_equal(np.nan_to_num(y, nan=7.0), np.nan_to_num(ry, nan=7.0))


# ------------------------------------------- tensor-core path coverage (bf16)

def _tc_counts():
    import ctypes
    from paper_1312_5853_b200._lib import lib
    a, b = ctypes.c_ulonglong(0), ctypes.c_ulonglong(0)
    lib().dll.pc_contraction_counts(ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


@pytest.mark.parametrize("geom", [(2, 96, 27, 27, 256, 5, 1, 2), (2, 256, 13, 13, 384, 3, 1, 1),
                                  (2, 384, 13, 13, 256, 3, 1, 1), (1, 8, 67, 67, 96, 11, 4, 0),
                                  (3, 16, 10, 10, 24, 3, 1, 1),
                                  # halo (shifted-window) operand: N <= 128, stride 1
                                  (2, 64, 57, 57, 96, 3, 1, 0), (3, 96, 13, 13, 64, 3, 1, 1),
                                  (2, 128, 31, 31, 96, 5, 1, 2),
                                  # M = 19008 = 74 * 256 + 64: the last CTA pair's second CTA
                                  # has no rows (its im2col start pixel would lie past the batch)
                                  (297, 64, 8, 8, 128, 3, 1, 1),
                                  # the space-to-depth input layer at a batch whose pair tiles fill
                                  # the machine: resident-filter halo forward with two sub-tiles
                                  (8, 64, 57, 57, 96, 3, 1, 0)])
def test_conv_bf16_alexnet_shapes_on_tensor_cores(geom):
    from paper_1312_5853_b200 import kernels as K
    b, c, h, w, n, k, s, p = geom
    rs = np.random.RandomState(11)
    x = bf16(rs.randn(b, c, h, w))
    wt = bf16(rs.randn(n, c, k, k) * (2.0 / (c * k * k)) ** 0.5)
    bias = rs.randn(n).astype(np.float32).astype(np.float64) * 0.1
    K.set_precision("bf16")
    tc0, simt0 = _tc_counts()
    cp = K.ConvParams(wt, bias, s, p)
    y = K.conv2d_forward(x, cp)
    yr = O.conv2d_forward(x, wt, bias, s, p)
    assert rel(y, yr) < BF16_OUT_TOL
    gy = bf16(rs.randn(*yr.shape))
    gx, gw, gb = K.conv2d_backward(x, cp, gy)
    rgx, rgw, rgb = O.conv2d_backward(x, wt, gy, s, p)
    assert rel(gx, rgx) < BF16_OUT_TOL
    assert rel(gw, rgw) < 1e-5
    assert rel(gb, rgb) < 1e-5
    tc1, simt1 = _tc_counts()
    assert simt1 == simt0 and tc1 - tc0 >= 3      # fwd, dgrad, wgrad all on tcgen05


@pytest.mark.parametrize("shape", [(256, 9216, 4096), (200, 4096, 1000), (64, 512, 128)])
def test_fc_bf16_on_tensor_cores(shape):
    from paper_1312_5853_b200 import kernels as K
    b, d, u = shape
    rs = np.random.RandomState(13)
    x, w = bf16(rs.randn(b, d)), bf16(rs.randn(d, u) * d ** -0.5)
    bias = rs.randn(u).astype(np.float32).astype(np.float64)
    gy = bf16(rs.randn(b, u))
    K.set_precision("bf16")
    tc0, simt0 = _tc_counts()
    assert rel(K.fc_forward(x, w, bias), O.fc_forward(x, w, bias)) < BF16_OUT_TOL
    gx, gw, gb = K.fc_backward(x, w, gy)
    rgx, rgw, rgb = O.fc_backward(x, w, gy)
    assert rel(gx, rgx) < BF16_OUT_TOL
    assert rel(gw, rgw) < 1e-5
    tc1, simt1 = _tc_counts()
    assert simt1 == simt0 and tc1 - tc0 == 3


@pytest.mark.parametrize("shape", [(2, 16, 13, 13), (1, 32, 27, 27), (2, 8, 11, 15), (1, 24, 7, 9)])
@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_maxpool_k3s2_vectorised_backward(shape, prec):
    """The 2x2-block k=3/s=2 backward (C % 8 == 0) against the oracle's scatter."""
    from paper_1312_5853_b200 import kernels as K
    rs = np.random.RandomState(17)
    x = bf16(np.round(rs.randn(*shape) * 3) / 3)     # quantised: plenty of ties
    K.set_precision(prec)
    y, arg = K.maxpool_forward(x, 3, 2)
    ry, rarg = O.maxpool_forward(x, 3, 2)
    assert np.array_equal(arg, rarg)
    gy = bf16(rs.randn(*ry.shape))
    gx = K.maxpool_backward(x, 3, 2, gy, arg)
    rgx = O.maxpool_backward(x.shape, 3, 2, gy, rarg)
    assert rel(gx, rgx) < (1e-6 if prec == "fp32" else BF16_OUT_TOL)


@pytest.mark.parametrize("case", [(3, 3, 227, 227, 4, 0), (2, 3, 227, 227, 4, 2), (2, 3, 35, 29, 4, 1),
                                  (2, 3, 64, 64, 2, 1)])
@pytest.mark.parametrize("src", ["bf16", "fp32"])
def test_space_to_depth_bit_exact(case, src):
    """pc_space_to_depth (input layer regrouping, SURVEY §8 a): dst[b][Y][X][(dy*s+dx)*C+c] =
    x[b][c][Y*s+dy-p][X*s+dx-p], zero outside the image and in the padding channels;
    bit-exact for both source precisions (the bf16 AlexNet case takes the row-staged kernel)."""
    import ctypes
    import torch
    from paper_1312_5853_b200._lib import lib, PC_BF16, PC_FP32
    b, c, h, w, s, p = case
    rs = np.random.RandomState(5)
    x = torch.as_tensor(rs.randn(b, c, h, w).astype(np.float32))
    if src == "bf16":
        x = x.bfloat16()
    hs, ws = (h + 2 * p + s - 1) // s, (w + 2 * p + s - 1) // s
    xd = x.cuda()
    out = torch.full((b, hs, ws, 64), 7.0, dtype=torch.bfloat16, device="cuda")
    lib().call("pc_space_to_depth", b, c, h, w, s, p, 64, xd.data_ptr(), PC_BF16 if src == "bf16" else PC_FP32,
               out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    got = out.float().cpu().numpy()
    xp = np.zeros((b, c, hs * s, ws * s), np.float32)
    xf = x.float().numpy()
    xp[:, :, p:p + h, p:p + w] = xf[:, :, : hs * s - p, : ws * s - p]
    want = np.zeros((b, hs, ws, 64), np.float32)
    blk = xp.reshape(b, c, hs, s, ws, s).transpose(0, 2, 4, 3, 5, 1).reshape(b, hs, ws, s * s * c)
    want[..., : s * s * c] = torch.as_tensor(blk).bfloat16().float().numpy()
    assert np.array_equal(got, want)


@pytest.mark.parametrize("case", [(3, 3, 227, 227, 4, 0), (2, 3, 64, 64, 2, 1)])
def test_space_to_depth_float64_source_and_float32_output(case):
    """The float64 source (a parconv caller's images, PC_FP64) gives exactly the float32
    source's result; the float32-output variant (tf32 mode) holds the unrounded values;
    the all-ones padding channel is written by both."""
    import torch
    from paper_1312_5853_b200._lib import lib, PC_FP32, PC_FP64
    b, c, h, w, s, p = case
    rs = np.random.RandomState(7)
    x64 = rs.randn(b, c, h, w).astype(np.float32).astype(np.float64)   # float32-exact, like the reference's
    hs, ws = (h + 2 * p + s - 1) // s, (w + 2 * p + s - 1) // s
    st = torch.cuda.current_stream().cuda_stream
    ones = c * s * s
    res = {}
    for name, arr, pc in (("f32", torch.as_tensor(x64.astype(np.float32)), PC_FP32),
                          ("f64", torch.as_tensor(x64), PC_FP64)):
        xd = arr.cuda()
        o16 = torch.empty((b, hs, ws, 64), dtype=torch.bfloat16, device="cuda")
        o32 = torch.empty((b, hs, ws, 64), dtype=torch.float32, device="cuda")
        lib().call("pc_space_to_depth_ex", b, c, h, w, s, p, 64, xd.data_ptr(), pc, ones, o16.data_ptr(), st)
        lib().call("pc_space_to_depth_f32", b, c, h, w, s, p, 64, xd.data_ptr(), pc, ones, o32.data_ptr(), st)
        res[name] = (o16.cpu(), o32.cpu())
    assert torch.equal(res["f32"][0], res["f64"][0]) and torch.equal(res["f32"][1], res["f64"][1])
    o32 = res["f64"][1].numpy()
    assert np.all(o32[..., ones] == 1.0) and np.all(o32[..., ones + 1:] == 0.0)
    xp = np.zeros((b, c, hs * s, ws * s), np.float32)
    xp[:, :, p:p + h, p:p + w] = x64.astype(np.float32)[:, :, : hs * s - p, : ws * s - p]
    blk = xp.reshape(b, c, hs, s, ws, s).transpose(0, 2, 4, 3, 5, 1).reshape(b, hs, ws, s * s * c)
    assert np.array_equal(o32[..., :ones], blk)
