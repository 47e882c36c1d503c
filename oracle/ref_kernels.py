"""TEST INFRASTRUCTURE ONLY — float64 restatement of the reference kernels.

Each function cites the reference code it restates
(`/root/reference/pkg/src/parconv/kernels.py`). Layout is NCHW, as in the
reference. Contractions use BLAS matmul (the reference uses single-threaded
einsum); results agree with the reference to ~1e-13 relative, which the
golden tests check.
"""

from __future__ import annotations

import numpy as np


def out_extent(n: int, k: int, s: int, p: int) -> int:
    """`kernels.py:72-83` (geometry must tile exactly)."""
    span = n + 2 * p - k
    if span < 0 or span % s:
        raise ValueError(f"geometry does not tile: n={n} k={k} s={s} p={p}")
    return span // s + 1


def _patches(x: np.ndarray, k: int, s: int, p: int):
    """im2col as in `kernels.py:86-101`: (B, Ho*Wo, C*k*k), K order (c, i, j)."""
    b, c, h, w = x.shape
    ho, wo = out_extent(h, k, s, p), out_extent(w, k, s, p)
    xp = np.pad(x, ((0, 0), (0, 0), (p, p), (p, p))) if p else x
    cols = np.empty((b, ho, wo, c, k, k), dtype=np.float64)
    for i in range(k):
        for j in range(k):
            cols[:, :, :, :, i, j] = xp[:, :, i:i + s * ho:s, j:j + s * wo:s].transpose(0, 2, 3, 1)
    return cols.reshape(b, ho * wo, c * k * k), ho, wo


def conv2d_forward(x, w, bias, stride, pad):
    """`kernels.py:104-116`: out[b,n,y,x] = bias[n] + sum_{c,i,j} in * w."""
    n, c, k, _ = w.shape
    cols, ho, wo = _patches(np.asarray(x, np.float64), k, stride, pad)
    out = cols @ w.reshape(n, -1).T + bias
    return np.ascontiguousarray(out.transpose(0, 2, 1).reshape(x.shape[0], n, ho, wo))


def conv2d_backward(x, w, grad_out, stride, pad):
    """`kernels.py:119-152`: (grad_x, grad_w, grad_b)."""
    n, c, k, _ = w.shape
    b, _, h, wd = x.shape
    cols, ho, wo = _patches(np.asarray(x, np.float64), k, stride, pad)
    go = grad_out.reshape(b, n, ho * wo)
    gb = go.sum(axis=(0, 2))
    gw = np.einsum("bnp,bpk->nk", go, cols, optimize=True).reshape(w.shape)
    gcols = (go.transpose(0, 2, 1) @ w.reshape(n, -1)).reshape(b, ho, wo, c, k, k)
    gx = np.zeros((b, c, h + 2 * pad, wd + 2 * pad))
    for i in range(k):
        for j in range(k):
            gx[:, :, i:i + stride * ho:stride, j:j + stride * wo:stride] += \
                gcols[:, :, :, :, i, j].transpose(0, 3, 1, 2)
    if pad:
        gx = gx[:, :, pad:pad + h, pad:pad + wd]
    return np.ascontiguousarray(gx), gw, gb


def fc_forward(x, w, bias):
    """`kernels.py:160-168`: W stored (D, U)."""
    return x @ w + bias


def fc_backward(x, w, grad_out):
    """`kernels.py:171-182`."""
    return grad_out @ w.T, x.T @ grad_out, grad_out.sum(axis=0)


def relu_forward(x):
    """`kernels.py:190-191`."""
    return np.maximum(x, 0.0)


def relu_backward(x, grad_out):
    """`kernels.py:194-197`: subgradient 0 at x == 0 (and NaN)."""
    return np.where(x > 0.0, grad_out, 0.0)


def maxpool_forward(x, k, stride):
    """`kernels.py:200-220`: window max + argmax as the local window index
    (row-major in the k*k window, first maximum wins)."""
    b, c, h, w = x.shape
    ho, wo = out_extent(h, k, stride, 0), out_extent(w, k, stride, 0)
    win = np.empty((b, c, ho, wo, k * k))
    for i in range(k):
        for j in range(k):
            win[..., i * k + j] = x[:, :, i:i + stride * ho:stride, j:j + stride * wo:stride]
    arg = np.argmax(win, axis=-1)
    return np.take_along_axis(win, arg[..., None], axis=-1)[..., 0], arg


def maxpool_backward(x_shape, k, stride, grad_out, argmax):
    """`kernels.py:223-244`: route each upstream value to its argmax; windows
    that overlap accumulate."""
    b, c, h, w = x_shape
    _, _, ho, wo = grad_out.shape
    gx = np.zeros(x_shape)
    iy, ix = np.divmod(argmax, k)
    rows = np.arange(ho)[:, None] * stride + iy
    cols = np.arange(wo)[None, :] * stride + ix
    flat = ((np.arange(b * c).reshape(b, c, 1, 1) * h + rows) * w + cols).ravel()
    np.add.at(gx.reshape(-1), flat, grad_out.ravel())
    return gx


def softmax_xent_scaled(logits, labels, scale):
    """`kernels.py:252-276`: loss = -scale * sum_b log softmax[b, y_b]."""
    labels = np.asarray(labels, dtype=np.int64)
    kk = logits.shape[1]
    if labels.size and (labels.min() < 0 or labels.max() >= kk):
        raise ValueError(f"labels must lie in [0, {kk})")
    z = logits - logits.max(axis=1, keepdims=True)
    e = np.exp(z)
    s = e.sum(axis=1, keepdims=True)
    rows = np.arange(logits.shape[0])
    loss = -float((z - np.log(s))[rows, labels].sum()) * scale
    g = e / s
    g[rows, labels] -= 1.0
    return loss, g * scale


def softmax_xent(logits, labels):
    """`kernels.py:279-283`."""
    return softmax_xent_scaled(logits, labels, 1.0 / logits.shape[0])


def sgd_step(params, grads, velocity, lr=0.01, momentum=0.9, weight_decay=0.0005):
    """`kernels.py:319-341`: v <- mu v - lr (g + wd p); p <- p + v."""
    new_v = [momentum * v - lr * (g + weight_decay * p) for p, g, v in zip(params, grads, velocity)]
    return [p + v for p, v in zip(params, new_v)], new_v


# --- extensions beyond the reference: the reference has no LRN or
# dropout (`netdef.py:219-220`). These float64 definitions ARE the
# specification the device kernels are checked against ("parity unpinned" with
# respect to the reference itself; pinned by finite differences in tests/).

def _lrn_scale(x, size, k, alpha):
    """S[b,c] = k + alpha * sum_{|c'-c| <= size//2} x[b,c']^2 (channels clipped at the edges)."""
    h = size // 2
    sq = np.asarray(x, np.float64) ** 2
    c = x.shape[1]
    csum = np.concatenate([np.zeros_like(sq[:, :1]), np.cumsum(sq, axis=1)], axis=1)
    lo = np.clip(np.arange(c) - h, 0, c)
    hi = np.clip(np.arange(c) + h + 1, 0, c)
    win = np.take(csum, hi, axis=1) - np.take(csum, lo, axis=1)
    return k + alpha * win


def lrn_forward(x, size=5, k=2.0, alpha=1e-4, beta=0.75):
    """Krizhevsky local response normalisation across channels (NCHW)."""
    x = np.asarray(x, np.float64)
    return x * _lrn_scale(x, size, k, alpha) ** (-beta)


def lrn_backward(x, grad_out, size=5, k=2.0, alpha=1e-4, beta=0.75):
    """gx_c = g_c S_c^-b - 2 a b x_c sum_{c': |c-c'| <= size//2} g_c' x_c' S_c'^(-b-1)."""
    x = np.asarray(x, np.float64)
    g = np.asarray(grad_out, np.float64)
    s = _lrn_scale(x, size, k, alpha)
    t = g * x * s ** (-beta - 1.0)
    h = size // 2
    c = x.shape[1]
    tsum = np.concatenate([np.zeros_like(t[:, :1]), np.cumsum(t, axis=1)], axis=1)
    lo = np.clip(np.arange(c) - h, 0, c)
    hi = np.clip(np.arange(c) + h + 1, 0, c)
    win = np.take(tsum, hi, axis=1) - np.take(tsum, lo, axis=1)
    return g * s ** (-beta) - 2.0 * alpha * beta * x * win


def dropout_forward(x, keep, p):
    return np.asarray(x, np.float64) * keep / (1.0 - p)


def dropout_backward(grad_out, keep, p):
    return np.asarray(grad_out, np.float64) * keep / (1.0 - p)
