"""Host-side conversions between the reference's parameter layout and the
device layout (numpy; run at setup / gather time only, never per step).

Reference layouts (`kernels.py:37-69`, `:160-168`, `schemes.py:160-182`):
  conv w: [N][C][kh][kw];  FC w: [D][U] with D the NCHW flatten of the
  (cross-concatenated) input, concatenation along channels/units in
  ascending column order.
Device layouts (include/pc_b200.h):
  conv w: [N][kh][kw][Cp] (C zero-padded to Cp for the bf16 input layer);
  FC w: [U][D'] where D' is the flatten order of the channel-blocked NHWC
  input: D' = k*(HW*Cs) + (h*W + w)*Cs + c for source column k, versus the
  reference's D = (k*Cs + c)*HW + h*W + w.
"""

from __future__ import annotations

import math

import numpy as np


def fc_row_perm(in_shape: tuple, m: int, cross: bool) -> np.ndarray | None:
    """perm[d'] = reference row d for an FC fed by `in_shape` (per-sample, after
    concatenation when cross). None when the two orders coincide."""
    if len(in_shape) != 3:
        return None
    c_full, h, w = in_shape
    blocks = m if cross else 1
    cs = c_full // blocks
    hw = h * w
    k = np.arange(blocks).reshape(blocks, 1, 1)
    p = np.arange(hw).reshape(1, hw, 1)
    c = np.arange(cs).reshape(1, 1, cs)
    perm = ((k * cs + c) * hw + p).reshape(-1)
    return None if np.array_equal(perm, np.arange(perm.size)) else perm


def conv_to_device(w: np.ndarray, cp: int) -> np.ndarray:
    n, c, kh, kw = w.shape
    out = np.zeros((n, kh, kw, cp), dtype=np.float32)
    out[..., :c] = w.transpose(0, 2, 3, 1)
    return out


def conv_from_device(wd: np.ndarray, c: int) -> np.ndarray:
    return np.ascontiguousarray(wd[..., :c].transpose(0, 3, 1, 2), dtype=np.float64)


def fc_to_device(w: np.ndarray, perm) -> np.ndarray:
    src = w if perm is None else w[perm]
    return np.ascontiguousarray(src.T, dtype=np.float32)


def fc_from_device(wd: np.ndarray, perm) -> np.ndarray:
    w = wd.T.astype(np.float64)
    if perm is None:
        return np.ascontiguousarray(w)
    out = np.empty_like(w)
    out[perm] = w
    return out


def device_weight_shape(cl, cp: int) -> tuple:
    if len(cl.weight_shape) == 4:
        n, _, kh, kw = cl.weight_shape
        return (n, kh, kw, cp)
    d, u = cl.weight_shape
    return (u, d)


def numel(shape) -> int:
    return int(math.prod(shape))


def s2d_extent(n: int, k: int, s: int, p: int) -> tuple:
    """(blocked extent, blocked kernel) of a k x k / stride-s / pad-p input conv
    rewritten as a stride-1 conv over s x s space-to-depth blocks."""
    return -(-(n + 2 * p) // s), -(-k // s)


def conv_to_device_s2d(w: np.ndarray, s: int, cs: int) -> np.ndarray:
    """[N][C][k][k] -> [N][k'][k'][cs] with channel (dy*s + dx)*C + c of block tap
    (I, J) = w[n][c][I*s+dy][J*s+dx] (zero where the tap falls beyond k, and for
    channels >= s*s*C)."""
    n, c, k, _ = w.shape
    kb = -(-k // s)
    wp = np.zeros((n, c, kb * s, kb * s), dtype=np.float64)
    wp[:, :, :k, :k] = w
    r = wp.reshape(n, c, kb, s, kb, s).transpose(0, 2, 4, 3, 5, 1).reshape(n, kb, kb, s * s * c)
    out = np.zeros((n, kb, kb, cs), dtype=np.float32)
    out[..., : s * s * c] = r
    return out


def conv_from_device_s2d(wd: np.ndarray, c: int, k: int, s: int) -> np.ndarray:
    n, kb = wd.shape[0], wd.shape[1]
    r = wd[..., : s * s * c].reshape(n, kb, kb, s, s, c).transpose(0, 5, 1, 3, 2, 4)
    return np.ascontiguousarray(r.reshape(n, c, kb * s, kb * s)[:, :, :k, :k], dtype=np.float64)


def s2d_keep_mask(n: int, c: int, k: int, s: int, cs: int) -> np.ndarray:
    """uint8 [N][k'][k'][cs]: 1 where the regrouped weight is a real filter tap."""
    return (conv_to_device_s2d(np.ones((n, c, k, k)), s, cs) != 0).astype(np.uint8)
