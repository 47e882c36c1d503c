"""Kernel-level drop-ins for `pkg/src/parconv/kernels.py`: same names, same
NCHW numpy arguments, same errors, computed on the B200 through the C ABI.

These are the unit-parity entry points (the reference's tests call kernels
one at a time on host arrays). Each call uploads its operands, runs the
device kernel in the module precision (``set_precision``; "fp32" =
verification mode by default, "bf16" = tensor-core mode, "tf32" = float
storage with tf32 tensor-core contractions) and returns
float64 numpy arrays. Like the reference they are pure: inputs are never
aliased or modified. The training step itself never goes through this
module — it keeps everything resident (``engine.py``).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .errors import ShapeError, ValidationError
from .netdef import conv_output_size

_PREC = {"fp32": L.PC_FP32, "bf16": L.PC_BF16, "tf32": L.PC_TF32}
_state = {"prec": L.PC_FP32}


def set_precision(name: str) -> None:
    if name not in _PREC:
        raise ValidationError(f"unknown precision {name!r}")
    _state["prec"] = _PREC[name]


def _storage() -> int:
    """Storage precision of the module precision (tf32 keeps float32 tensors)."""
    return L.PC_FP32 if _state["prec"] == L.PC_TF32 else _state["prec"]


def tensor(values) -> np.ndarray:
    return np.ascontiguousarray(values, dtype=np.float64)


def _require(cond, msg):
    if not cond:
        raise ShapeError(msg)


def _dev():
    if not torch.cuda.is_available():
        raise ValidationError("paper_1312_5853_b200.kernels needs a CUDA device")
    return torch.device("cuda", torch.cuda.current_device())


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _up(a: np.ndarray, prec: int) -> torch.Tensor:
    t = torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32)).to(_dev())
    return t.to(torch.bfloat16) if prec == L.PC_BF16 else t


def _down(t: torch.Tensor, shape) -> np.ndarray:
    return t.float().cpu().numpy().astype(np.float64).reshape(shape)


def _nhwc(a):
    return np.ascontiguousarray(np.transpose(a, (0, 2, 3, 1)))


def _nchw(a):
    return np.ascontiguousarray(np.transpose(a, (0, 3, 1, 2)))


@dataclass
class ConvParams:
    weights: np.ndarray
    bias: np.ndarray
    stride: int = 1
    pad: int = 0

    def __post_init__(self):
        self.weights, self.bias = tensor(self.weights), tensor(self.bias)
        if self.weights.ndim != 4:
            raise ShapeError(f"conv weights must be 4-d, got {self.weights.shape}")
        if self.bias.shape != (self.weights.shape[0],):
            raise ShapeError(f"conv bias shape {self.bias.shape} does not match "
                             f"{self.weights.shape[0]} output channels")
        if min(self.weights.shape) < 1:
            raise ValidationError("conv extents must all be >= 1")
        if self.stride < 1:
            raise ValidationError(f"conv stride must be >= 1, got {self.stride}")
        if self.pad < 0:
            raise ValidationError(f"conv pad must be >= 0, got {self.pad}")

    @property
    def out_channels(self):
        return self.weights.shape[0]

    @property
    def in_channels(self):
        return self.weights.shape[1]


def _conv_setup(x, p: ConvParams, prec):
    _require(x.ndim == 4, f"conv input must be 4-d, got {x.shape}")
    _require(x.shape[1] == p.in_channels,
             f"conv input has {x.shape[1]} channels, weights expect {p.in_channels}")
    b, c, h, w = x.shape
    n, _, k, _ = p.weights.shape
    ho, wo = conv_output_size(h, k, p.stride, p.pad), conv_output_size(w, k, p.stride, p.pad)
    cp = c if prec != L.PC_BF16 or c % 8 == 0 else (c + 7) // 8 * 8
    xn = np.zeros((b, h, w, cp))
    xn[..., :c] = _nhwc(x)
    wd = np.zeros((n, k, k, cp))
    wd[..., :c] = p.weights.transpose(0, 2, 3, 1)
    g = L.ConvGeom(b, h, w, cp, n, k, p.stride, p.pad, ho, wo, cp, 0)
    return g, xn, wd, ho, wo, cp


def conv2d_forward(x: np.ndarray, p: ConvParams) -> np.ndarray:
    prec = _state["prec"]
    g, xn, wd, ho, wo, _ = _conv_setup(x, p, prec)
    xd, wdd = _up(xn, prec), _up(wd, prec)
    bd = torch.as_tensor(p.bias.astype(np.float32)).to(_dev())
    y = torch.empty(max(x.shape[0] * ho * wo * p.out_channels, 1), dtype=xd.dtype, device=_dev())
    L.lib().call("pc_conv2d_forward", C.byref(g), xd.data_ptr(), wdd.data_ptr(), bd.data_ptr(),
                 y.data_ptr(), prec, 0, _stream())
    return _nchw(_down(y[: x.shape[0] * ho * wo * p.out_channels], (x.shape[0], ho, wo, p.out_channels)))


def conv2d_backward(x: np.ndarray, p: ConvParams, grad_out: np.ndarray):
    prec = _state["prec"]
    g, xn, wd, ho, wo, cp = _conv_setup(x, p, prec)
    b, c, h, w = x.shape
    n = p.out_channels
    _require(grad_out.shape == (b, n, ho, wo),
             f"conv grad_out shape {grad_out.shape} does not match forward output {(b, n, ho, wo)}")
    xd, wdd, gy = _up(xn, prec), _up(wd, prec), _up(_nhwc(grad_out), prec)
    gx = torch.empty(max(b * h * w * cp, 1), dtype=xd.dtype, device=_dev())
    gw = torch.empty(n * p.weights.shape[2] ** 2 * cp, dtype=torch.float32, device=_dev())
    gb = torch.empty(n, dtype=torch.float32, device=_dev())
    lib = L.lib()
    wsb = lib.raw("pc_conv2d_backward_workspace")(C.byref(g), prec)
    ws = torch.empty(max(int(wsb), 16), dtype=torch.uint8, device=_dev())
    lib.call("pc_conv2d_backward", C.byref(g), xd.data_ptr(), wdd.data_ptr(), gy.data_ptr(), gx.data_ptr(),
             None, gw.data_ptr(), gb.data_ptr(), prec, L.PC_WANT_DX | L.PC_WANT_DW, ws.data_ptr(),
             int(wsb), _stream())
    k = p.weights.shape[2]
    gxn = _nchw(_down(gx[: b * h * w * cp], (b, h, w, cp)))[:, :c]
    gwn = _down(gw, (n, k, k, cp))[..., :c].transpose(0, 3, 1, 2)
    return np.ascontiguousarray(gxn), np.ascontiguousarray(gwn), _down(gb, (n,))


def fc_forward(x: np.ndarray, weights: np.ndarray, bias: np.ndarray) -> np.ndarray:
    _require(x.ndim == 2 and weights.ndim == 2, "fc expects 2-d input and weights")
    _require(x.shape[1] == weights.shape[0],
             f"fc inner dimensions disagree: input {x.shape} vs weights {weights.shape}")
    _require(bias.shape == (weights.shape[1],), f"fc bias shape {bias.shape} invalid")
    prec = _state["prec"]
    b, d = x.shape
    u = weights.shape[1]
    xd, wdd = _up(x, prec), _up(np.ascontiguousarray(weights.T), prec)
    bd = torch.as_tensor(np.asarray(bias, np.float32)).to(_dev())
    y = torch.empty(max(b * u, 1), dtype=xd.dtype, device=_dev())
    m = L.Mat(xd.data_ptr(), d, d, 0)
    L.lib().call("pc_fc_forward", b, d, u, C.byref(m), wdd.data_ptr(), bd.data_ptr(), y.data_ptr(), prec,
                 0, _stream())
    return _down(y[: b * u], (b, u))


def fc_backward(x: np.ndarray, weights: np.ndarray, grad_out: np.ndarray):
    _require(grad_out.shape == (x.shape[0], weights.shape[1]),
             f"fc grad_out shape {grad_out.shape} does not match output {(x.shape[0], weights.shape[1])}")
    prec = _state["prec"]
    b, d = x.shape
    u = weights.shape[1]
    xd, wdd, gy = _up(x, prec), _up(np.ascontiguousarray(weights.T), prec), _up(grad_out, prec)
    gx = torch.empty(max(b * d, 1), dtype=xd.dtype, device=_dev())
    gw = torch.empty(u * d, dtype=torch.float32, device=_dev())
    gb = torch.empty(u, dtype=torch.float32, device=_dev())
    lib = L.lib()
    wsb = int(lib.raw("pc_fc_backward_workspace")(b, d, u, prec))
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device=_dev())
    xm, gm = L.Mat(xd.data_ptr(), d, d, 0), L.Mat(gx.data_ptr(), d, d, 0)
    lib.call("pc_fc_backward", b, d, u, C.byref(xm), wdd.data_ptr(), gy.data_ptr(), C.byref(gm), None,
             gw.data_ptr(), gb.data_ptr(), prec, L.PC_WANT_DX | L.PC_WANT_DW, ws.data_ptr(), wsb, _stream())
    return _down(gx[: b * d], (b, d)), _down(gw, (u, d)).T.copy(), _down(gb, (u,))


def relu_forward(x: np.ndarray) -> np.ndarray:
    prec = _storage()
    xd = _up(x, prec)
    y = torch.empty_like(xd)
    L.lib().call("pc_relu_forward", xd.numel(), xd.data_ptr(), y.data_ptr(), prec, _stream())
    return _down(y, x.shape)


def relu_backward(x: np.ndarray, grad_out: np.ndarray) -> np.ndarray:
    _require(x.shape == grad_out.shape, "relu grad_out shape mismatch")
    prec = _storage()
    xd, gd = _up(x, prec), _up(grad_out, prec)
    gx = torch.empty_like(xd)
    L.lib().call("pc_relu_backward", xd.numel(), xd.data_ptr(), gd.data_ptr(), gx.data_ptr(), prec,
                 _stream())
    return _down(gx, x.shape)


def maxpool_forward(x: np.ndarray, k: int, stride: int):
    _require(x.ndim == 4, f"maxpool input must be 4-d, got {x.shape}")
    prec = _storage()
    b, c, h, w = x.shape
    ho, wo = conv_output_size(h, k, stride, 0), conv_output_size(w, k, stride, 0)
    xd = _up(_nhwc(x), prec)
    y = torch.empty(max(b * ho * wo * c, 1), dtype=xd.dtype, device=_dev())
    arg = torch.empty(max(b * ho * wo * c, 1), dtype=torch.uint8, device=_dev())
    L.lib().call("pc_maxpool_forward", b, h, w, c, k, stride, xd.data_ptr(), y.data_ptr(), arg.data_ptr(),
                 prec, _stream())
    n = b * ho * wo * c
    yo = _nchw(_down(y[:n], (b, ho, wo, c)))
    ao = _nchw(arg[:n].cpu().numpy().reshape(b, ho, wo, c)).astype(np.int64)
    return yo, ao


def maxpool_backward(x: np.ndarray, k: int, stride: int, grad_out: np.ndarray, argmax=None) -> np.ndarray:
    if argmax is None:
        _, argmax = maxpool_forward(x, k, stride)
    prec = _storage()
    b, c, h, w = x.shape
    ho, wo = conv_output_size(h, k, stride, 0), conv_output_size(w, k, stride, 0)
    _require(grad_out.shape == (b, c, ho, wo), "maxpool grad_out shape mismatch")
    gy = _up(_nhwc(grad_out), prec)
    ad = torch.as_tensor(_nhwc(np.asarray(argmax)).astype(np.uint8)).to(_dev())
    gx = torch.empty(max(b * h * w * c, 1), dtype=gy.dtype, device=_dev())
    L.lib().call("pc_maxpool_backward", b, h, w, c, k, stride, gy.data_ptr(), ad.data_ptr(), None,
                 gx.data_ptr(), prec, _stream())
    return _nchw(_down(gx[: b * h * w * c], (b, h, w, c)))


def softmax_xent_scaled(logits: np.ndarray, labels, scale: float):
    _require(logits.ndim == 2, f"logits must be 2-d, got {logits.shape}")
    labels = np.asarray(labels, dtype=np.int64)
    _require(labels.shape == (logits.shape[0],), "labels length must equal batch size")
    k = logits.shape[1]
    if labels.size and (labels.min() < 0 or labels.max() >= k):
        raise ValidationError(f"labels must lie in [0, {k})")
    prec = _storage()
    b = logits.shape[0]
    zd = _up(logits, prec)
    yd = torch.as_tensor(labels.astype(np.int32)).to(_dev())
    grad = torch.empty_like(zd)
    rows = torch.empty(max(b, 1), dtype=torch.float64, device=_dev())
    tot = torch.empty(1, dtype=torch.float64, device=_dev())
    bad = torch.zeros(1, dtype=torch.int32, device=_dev())
    lib = L.lib()
    lib.call("pc_softmax_xent", b, k, zd.data_ptr(), yd.data_ptr(), float(scale), grad.data_ptr(),
             rows.data_ptr(), bad.data_ptr(), prec, _stream())
    lib.call("pc_sum_f64", b, rows.data_ptr(), tot.data_ptr(), _stream())
    return float(tot.cpu().item()), _down(grad, logits.shape)


def softmax_xent(logits: np.ndarray, labels):
    labels = np.asarray(labels, dtype=np.int64)
    _require(logits.shape[0] >= 1, "softmax_xent needs at least one row")
    return softmax_xent_scaled(logits, labels, 1.0 / logits.shape[0])


@dataclass
class SgdState:
    learning_rate: float = 0.01
    momentum: float = 0.9
    weight_decay: float = 0.0005
    velocity: list = field(default_factory=list)

    def __post_init__(self):
        if self.learning_rate < 0:
            raise ValidationError("learning_rate must be non-negative")
        if not 0.0 <= self.momentum < 1.0:
            raise ValidationError("momentum must lie in [0, 1)")
        if self.weight_decay < 0:
            raise ValidationError("weight_decay must be non-negative")

    @classmethod
    def zeros(cls, params, **hyper):
        st = cls(**hyper)
        st.velocity = [np.zeros_like(p) for p in params]
        return st


def sgd_step(params, grads, state: SgdState):
    """v <- mu v - lr (g + wd p); p <- p + v, one multi-tensor launch."""
    if len(params) != len(grads) or len(params) != len(state.velocity):
        raise ShapeError("sgd_step: params, grads and velocity counts differ")
    for p, g, v in zip(params, grads, state.velocity):
        if np.shape(p) != np.shape(g) or np.shape(p) != np.shape(v):
            raise ShapeError(f"sgd_step shape mismatch: param {np.shape(p)}, grad {np.shape(g)}, "
                             f"velocity {np.shape(v)}")
    dev = _dev()
    ps = [torch.as_tensor(np.asarray(p, np.float32).ravel().copy()).to(dev) for p in params]
    vs = [torch.as_tensor(np.asarray(v, np.float32).ravel().copy()).to(dev) for v in state.velocity]
    gs = [torch.as_tensor(np.asarray(g, np.float32).ravel().copy()).to(dev) for g in grads]
    tab = (L.SgdTensor * max(len(ps), 1))()
    for i, (p, v, g) in enumerate(zip(ps, vs, gs)):
        tab[i] = L.SgdTensor(p.data_ptr(), v.data_ptr(), g.data_ptr(), None, p.numel())
    td = torch.frombuffer(bytearray(bytes(tab)), dtype=torch.uint8).to(dev)
    mx = max([p.numel() for p in ps], default=0)
    L.lib().call("pc_sgd_step", len(ps), td.data_ptr(), mx, state.learning_rate, state.momentum,
                 state.weight_decay, _stream())
    new_p = [p.cpu().numpy().astype(np.float64).reshape(np.shape(o)) for p, o in zip(ps, params)]
    new_v = [v.cpu().numpy().astype(np.float64).reshape(np.shape(o)) for v, o in zip(vs, params)]
    return new_p, SgdState(state.learning_rate, state.momentum, state.weight_decay, new_v)
