"""Per-worker device engine: the B200 restatement of `schemes.column_fwd_bwd`
(`pkg/src/parconv/schemes.py:342-419`) plus the worker's slice of the
data-parallel leg and the SGD update (`schemes.py:540-558`).

Layout in HBM (one worker = one column of one replica):
  * activations NHWC in the storage precision (bf16 in production, fp32 in
    the verification mode); a cross layer's input is a channel-blocked
    concatenation buffer [m][B][H][W][C/m] that the column exchange fills;
  * parameters, velocity and gradients are single flat fp32 buffers in the
    reference's canonical order (ascending layer, weights then bias; device
    weight layouts from ``layout.py``), so the data-parallel all-reduce is
    one contiguous buffer and the optimizer is one launch; a flat bf16
    shadow of the parameters feeds the tensor cores and is rewritten by the
    same SGD launch.
Fusions: conv/FC + ReLU forward (epilogue), ReLU backward folded into the
consumer's data-grad epilogue (conv/FC dgrad mask) or the max-pool gather
backward, softmax loss + gradient in one kernel.
Every call goes through the C ABI (``_lib``); nothing here computes on the
host.
"""

from __future__ import annotations

import ctypes as C
import os
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from . import layout
from .errors import ValidationError
from . import rng
from .netdef import FC, LRN, ColumnizedSpec, Conv, Dropout, MaxPool, ReLU, SoftmaxXent

ALIGN = 32  # elements; every flat-buffer slice starts 128-byte aligned in fp32
PROFILE: list | None = None  # set to a list to record per-call CUDA events


def _wg_ctas() -> dict:
    """PC_WG_CTAS: grid caps of the side-stream conv weight gradients, "N" for all
    layers or "layer:N,layer:N" (e.g. "3:100"); empty = uncapped."""
    out = {}
    for part in filter(None, os.environ.get("PC_WG_CTAS", "").split(",")):
        k, _, v = part.rpartition(":")
        out[int(k) if k else -1] = int(v)
    return out


WG_CTAS = _wg_ctas()


def torch_dtype(prec: int):
    return torch.bfloat16 if prec == L.PC_BF16 else torch.float32


@dataclass
class LayerState:
    cl: object
    kind: str
    inp: torch.Tensor | None = None      # input activation (concat buffer when cross)
    in_nhwc: tuple | None = None         # (H, W, C_full) or (D,) per sample
    in_blocks: int = 1
    out: torch.Tensor | None = None
    out_nhwc: tuple | None = None
    argmax: torch.Tensor | None = None
    gin: torch.Tensor | None = None      # gradient w.r.t. inp (same layout)
    gout: torch.Tensor | None = None     # gradient w.r.t. out
    rs: torch.Tensor | None = None       # cross layers: reduce-scatter target (own slice)
    relu_fused_fwd: bool = False         # ReLU computed by the producer's epilogue
    relu_after: bool = False             # conv/FC: next layer is a fused ReLU
    skip_bwd: bool = False               # ReLU: backward folded into consumer
    mask_dx: bool = False                # consumer applies the ReLU mask (= inp > 0)
    w_off: int = -1
    b_off: int = -1
    w_shape: tuple = ()
    cp: int = 0                          # padded input channels (conv)
    perm: np.ndarray | None = None       # FC row permutation (reference <-> device)
    geom: object = None
    row_loss: torch.Tensor | None = None
    col: int = 0                         # explicit-im2col input conv: padded K (0 = implicit GEMM)
    s2d: int = 0                         # space-to-depth input conv: block size (= reference stride)
    drop: tuple = ()                     # dropout: (H, W, C, C_dense, c_off, threshold) of this column's slice
    keep: torch.Tensor | None = None     # s2d: uint8 mask of real filter taps in the device weights
    wt: torch.Tensor | None = None       # conv: filters prepared for the data gradient (pc_conv2d_dgrad_weights)
    bias_by_pool: bool = False           # conv: bias gradient reduced by the pool backward that writes its gy
    pool_bias: int = -1                  # pool: position of the conv whose bias gradient it reduces


class ColumnEngine:
    """One worker's buffers and step program on one device."""

    def __init__(self, cs: ColumnizedSpec, wid: int, replica: int, column: int, shard: int,
                 prec: int, device: torch.device, hyper: tuple, cprec: int | None = None):
        self.cs, self.m = cs, cs.columns
        self.wid, self.replica, self.column = wid, replica, column
        # prec: storage precision of activations (PC_FP32 / PC_BF16); cprec: the
        # contractions' (PC_TF32 = float storage, tf32 tensor-core math)
        self.B, self.prec, self.device = shard, prec, device
        self.cprec = prec if cprec is None else cprec
        self.lr, self.mom, self.wd = (float(h) for h in hyper)
        self.dtype = torch_dtype(prec)
        self.lib = L.lib()
        self.layers: list[LayerState] = []
        self._build_activations()
        self._build_params()
        self._build_grads()
        self.labels = torch.zeros(max(shard, 1), dtype=torch.int32, device=device)
        # dropout stream (rng.dropout_state): seed, device step counter (advanced in the step program)
        self.dropout_seed = 0
        self.training = True
        self.step_ctr = torch.zeros(1, dtype=torch.int64, device=device)
        self.has_dropout = any(st.kind == "dropout" for st in self.layers)
        self.bad_label = torch.zeros(1, dtype=torch.int32, device=device)
        self.loss = torch.zeros(1, dtype=torch.float64, device=device)
        self.loss_ticket = torch.zeros(1, dtype=torch.int32, device=device)   # pc_softmax_xent_loss
        self.bias_side = None                # enable_bias_side
        self.wt_ready = False                # the step program prepared st.wt this step

    # ------------------------------------------------------------------ setup
    def _new(self, n, dtype=None):
        return torch.empty(max(int(n), 1), dtype=dtype or self.dtype, device=self.device)

    def _build_activations(self):
        cs, B, m = self.cs, self.B, self.m
        c, h, w = cs.base.input_shape
        first = cs.col_layers[0]
        self.in_c = c
        self.in_cp = c
        # bf16 input conv with channels too narrow for 128-byte im2col rows (AlexNet:
        # 3). Strided (AlexNet 11x11/s4): space-to-depth the image into s x s blocks
        # (s*s*C <= 64 channels, padded to 64) and run the layer as a stride-1
        # ceil(k/s)^2 implicit-GEMM conv on the tensor cores. Stride 1: materialise
        # its columns once per step (pc_im2col) and run it as a dense GEMM over
        # pixels; col_kp = padded K (reference (c, i, j) order).
        self.col_kp = 0
        self.s2d = 0
        self.s2d_ones = -1
        lay0 = first.layer if isinstance(first.layer, Conv) else None
        tc = self.prec == L.PC_BF16 or self.cprec == L.PC_TF32    # a tensor-core input layer
        if tc and lay0 is not None and c % 64 and lay0.stride > 1 and c * lay0.stride ** 2 <= 64:
            self.s2d = lay0.stride
            self.s2d_hw = (layout.s2d_extent(h, lay0.kernel, lay0.stride, lay0.pad)[0],
                           layout.s2d_extent(w, lay0.kernel, lay0.stride, lay0.pad)[0])
            self.in_cp = 64
            self.x = self._new(B * self.s2d_hw[0] * self.s2d_hw[1] * 64)
            # padding channel held at 1.0: its weight gradient at tap (0, 0) is the
            # layer's bias gradient (pc_s2d_wgrad_finish); its weights stay 0
            self.s2d_ones = c * lay0.stride ** 2 if c * lay0.stride ** 2 < 64 and \
                os.environ.get("PC_S2D_ONES", "1") != "0" else -1
        elif (self.prec == L.PC_BF16 or self.cprec == L.PC_TF32) and lay0 is not None and c % 32:
            # tf32: the tensor-core im2col path needs 32-channel (128-byte) rows too
            k0 = lay0.kernel
            q = 8 if self.prec == L.PC_BF16 else 32
            self.col_kp = (c * k0 * k0 + q - 1) // q * q
            ho0, wo0 = first.out_shape[1], first.out_shape[2]
            self.x = self._new(B * ho0 * wo0 * self.col_kp)
        else:
            self.x = self._new(B * h * w * self.in_cp)
        prev_out, prev_shape = self.x, (self.s2d_hw + (64,)) if self.s2d else (h, w, self.in_cp)
        n = len(cs.col_layers)
        for i, cl in enumerate(cs.col_layers):
            layer = cl.layer
            kind = {Conv: "conv", FC: "fc", ReLU: "relu", MaxPool: "pool", SoftmaxXent: "softmax", LRN: "lrn",
                    Dropout: "dropout"}[type(layer)]
            st = LayerState(cl, kind)
            per = math.prod(prev_shape)
            if cl.cross:
                st.inp = self._new(m * B * per)
                st.in_blocks = m
                st.in_nhwc = (prev_shape[:-1] + (prev_shape[-1] * m,)) if len(prev_shape) == 3 \
                    else (prev_shape[0] * m,)
                st.rs = self._new(B * per)
            else:
                st.inp, st.in_nhwc = prev_out, prev_shape
            if kind == "conv":
                hh, ww, cc = st.in_nhwc
                kk, ss, pp = layer.kernel, layer.stride, layer.pad
                if i == 0 and self.s2d:
                    st.s2d = self.s2d
                    kk, ss, pp = -(-layer.kernel // self.s2d), 1, 0
                ho = (hh + 2 * pp - kk) // ss + 1
                wo = (ww + 2 * pp - kk) // ss + 1
                nout = cl.out_shape[0]
                assert (ho, wo) == tuple(cl.out_shape[1:]), (ho, wo, cl.out_shape)
                if i == 0 and self.col_kp:
                    st.col = self.col_kp
                elif cc % 8 and self.prec == L.PC_BF16:
                    raise ValidationError(f"layer {cl.index}: bf16 conv needs C % 8 == 0 (C={cc})")
                st.cp = cc
                cs_blk = cc // st.in_blocks
                st.geom = L.ConvGeom(B, hh, ww, cc, nout, kk, ss, pp, ho, wo, cs_blk, B * hh * ww * cs_blk)
                st.out_nhwc = (ho, wo, nout)
                st.out = self._new(B * ho * wo * nout)
            elif kind == "fc":
                st.out_nhwc = (cl.out_shape[0],)
                st.out = self._new(B * cl.out_shape[0])
                st.perm = layout.fc_row_perm(cl.in_shape, m, cl.cross)
            elif kind in ("lrn", "dropout"):
                st.out_nhwc = st.in_nhwc
                st.out = self._new(B * per)
                if kind == "dropout":
                    hh, ww, cc = st.in_nhwc if len(st.in_nhwc) == 3 else (1, 1, st.in_nhwc[0])
                    split = self._split_before(i)
                    st.drop = (hh, ww, cc, cc * (m if split else 1), cc * self.column if split else 0,
                               rng.dropout_threshold(layer.p))
            elif kind == "relu":
                prev = self.layers[-1] if self.layers else None
                st.out_nhwc = st.in_nhwc
                if prev is not None and prev.kind in ("conv", "fc") and not cl.cross:
                    st.relu_fused_fwd = True
                    prev.relu_after = True
                    st.out = st.inp
                else:
                    st.out = self._new(B * per)
            elif kind == "pool":
                hh, ww, cc = st.in_nhwc
                ho = (hh - layer.kernel) // layer.stride + 1
                wo = (ww - layer.kernel) // layer.stride + 1
                st.out_nhwc = (ho, wo, cc)
                st.out = self._new(B * ho * wo * cc)
                st.argmax = self._new(B * ho * wo * cc, torch.uint8)
            else:
                st.out_nhwc = (layer.classes,)
                st.out = self._new(B * layer.classes)          # gradient of the logits
                st.row_loss = self._new(B, torch.float64)
            self.layers.append(st)
            prev_out, prev_shape = st.out, st.out_nhwc
        # backward wiring (reverse order so ReLU aliases resolve)
        for i in range(n - 1, -1, -1):
            st = self.layers[i]
            nxt = self.layers[i + 1] if i + 1 < n else None
            if nxt is not None:
                st.gout = nxt.rs if nxt.cl.cross else nxt.gin
            if st.kind == "relu":
                st.skip_bwd = nxt is not None and nxt.kind in ("conv", "fc", "pool")
            if i == 0:
                continue
            if st.kind == "softmax":
                st.gin = st.out
            elif st.kind == "relu" and st.skip_bwd:
                st.gin = st.gout
            else:
                st.gin = self._new(st.inp.numel())
        for i in range(1, n):
            st, prv = self.layers[i], self.layers[i - 1]
            st.mask_dx = st.kind in ("conv", "fc", "pool") and prv.kind == "relu" and prv.skip_bwd
        # ReLU -> max-pool -> conv/FC: the ReLU mask at a pixel that receives pool
        # gradient is (its value > 0) = (the window maximum > 0), so the consumer's
        # data-gradient epilogue masks by its own input (the pooled maximum) and the
        # pool backward routes without reading the full-resolution activation —
        # exact (masks are 0/1 and every contribution to a pixel shares its value).
        # conv -> ReLU -> 3x3/s2 max-pool (bf16): the pool backward writes the conv's
        # upstream gradient and reduces its bias gradient on the way (pc_maxpool_backward_bias)
        if self.prec == L.PC_BF16 and os.environ.get("PC_POOL_BIAS", "1") != "0":
            for i in range(2, n):
                st, rl, cv = self.layers[i], self.layers[i - 1], self.layers[i - 2]
                if st.kind == "pool" and rl.kind == "relu" and rl.skip_bwd and cv.kind == "conv" and \
                        not cv.col and not cv.s2d and st.cl.layer.kernel == 3 and st.cl.layer.stride == 2:
                    c = st.in_nhwc[2]
                    if c % 8 == 0 and 256 % (c // 8) == 0:
                        st.pool_bias, cv.bias_by_pool = i - 2, True
        if any(st.pool_bias >= 0 for st in self.layers):
            cmax = max(st.in_nhwc[2] for st in self.layers if st.pool_bias >= 0)
            self.pool_ws = torch.empty(self.lib.raw("pc_maxpool_backward_bias_workspace")(cmax), dtype=torch.uint8,
                                       device=self.device)
        if os.environ.get("PC_POOL_MASK_FOLD", "1") != "0":
            for i in range(1, n - 1):
                st, nxt = self.layers[i], self.layers[i + 1]
                if st.kind == "pool" and st.mask_dx and nxt.kind in ("conv", "fc") and not nxt.mask_dx \
                        and not (nxt.kind == "conv" and nxt.col):
                    st.mask_dx, nxt.mask_dx = False, True

    def param_region(self, i: int) -> tuple:
        """[lo, hi) of layer position i's weights + bias in the flat buffers (up to the
        next parameter layer, alignment padding included)."""
        st = self.layers[i]
        nxt = [t.w_off for t in self.layers[i + 1:] if t.w_off >= 0]
        return st.w_off, (nxt[0] if nxt else self.n_flat)

    def _split_before(self, i: int) -> bool:
        """Is the activation entering layer position i split across columns?"""
        rep = True
        for cl in self.cs.col_layers[:i]:
            if cl.cross:
                rep = True
            if isinstance(cl.layer, (Conv, FC)):
                rep = cl.shared
        if self.cs.col_layers[i].cross:
            rep = True
        return self.m > 1 and not rep

    def _build_params(self):
        off = 0
        for st in self.layers:
            if st.kind not in ("conv", "fc"):
                continue
            if st.col:
                st.w_shape = (st.cl.weight_shape[0], st.col)
            elif st.s2d:
                n_, c_, k_, _ = st.cl.weight_shape
                keep = layout.s2d_keep_mask(n_, c_, k_, st.s2d, st.cp)
                st.w_shape = keep.shape
                st.keep = torch.from_numpy(keep.reshape(-1)).to(self.device)
            else:
                st.w_shape = layout.device_weight_shape(st.cl, st.cp)
            st.w_off = off
            off += -(-layout.numel(st.w_shape) // ALIGN) * ALIGN
            st.b_off = off
            off += -(-st.cl.bias_shape[0] // ALIGN) * ALIGN
        self.n_flat = max(off, ALIGN)
        self.p32 = torch.zeros(self.n_flat, dtype=torch.float32, device=self.device)
        self.v32 = torch.zeros_like(self.p32)
        self.plow = torch.zeros(self.n_flat, dtype=torch.bfloat16, device=self.device) \
            if self.prec == L.PC_BF16 else None
        tab = L.SgdTensor(self.p32.data_ptr(), self.v32.data_ptr(), 0,
                          self.plow.data_ptr() if self.plow is not None else None, self.n_flat)
        self._sgd_host = tab
        self._sgd_dev = torch.frombuffer(bytearray(bytes(tab)), dtype=torch.uint8).to(self.device)

    def _build_grads(self):
        self.g32 = torch.zeros(self.n_flat, dtype=torch.float32, device=self.device)
        self.set_grad_source(self.g32)
        ws = 0
        for st in self.layers:
            if st.kind == "conv" and st.col:
                g = st.geom
                ws = max(ws, self.lib.raw("pc_fc_backward_workspace")(self.B * g.Ho * g.Wo, st.col, g.N, self.cprec))
            elif st.kind == "conv":
                ws = max(ws, self.lib.raw("pc_conv2d_backward_workspace")(C.byref(st.geom), self.cprec))
            elif st.kind == "fc":
                d = math.prod(st.in_nhwc)
                ws = max(ws, self.lib.raw("pc_fc_backward_workspace")(self.B, d, st.cl.out_shape[0], self.cprec),
                         self.lib.raw("pc_fc_forward_workspace")(self.B, d, st.cl.out_shape[0], self.cprec))
        self.ws_bytes = int(ws)
        self.ws = torch.empty(max(self.ws_bytes, 16), dtype=torch.uint8, device=self.device)

    def set_grad_source(self, g: torch.Tensor):
        """Point the SGD launch at a (possibly reduced, shared) gradient buffer."""
        self._sgd_host.g = g.data_ptr()
        self._sgd_dev.copy_(torch.frombuffer(bytearray(bytes(self._sgd_host)), dtype=torch.uint8))
        self._sgd_regions = None

    def sgd_split_table(self, first: int):
        """Two SGD launch tables over the flat buffers: parameters of layer positions
        >= ``first`` (the FC head: final once the backward has passed it, so their
        update can run on a side stream beside the convolutions' backward) and the
        rest. Returns ((n, max_numel, device table), same) or None."""
        groups = ([], [])
        for i, st in enumerate(self.layers):
            if st.w_off < 0:
                continue
            lo, hi = self.param_region(i)
            groups[0 if i >= first else 1].append((lo, hi - lo))
        if not groups[0] or not groups[1]:
            return None
        merged = []
        for regs in groups:  # adjacent regions -> one descriptor (one long grid-stride range)
            m = []
            for o, n in sorted(regs):
                if m and m[-1][0] + m[-1][1] == o:
                    m[-1] = (m[-1][0], m[-1][1] + n)
                else:
                    m.append((o, n))
            merged.append(m)
        out = []
        for regs in merged:
            tabs = [L.SgdTensor(self.p32[o:].data_ptr(), self.v32[o:].data_ptr(), self.g32[o:].data_ptr(),
                                self.plow[o:].data_ptr() if self.plow is not None else None, n) for o, n in regs]
            arr = (L.SgdTensor * len(tabs))(*tabs)
            out.append((len(tabs), max(n for _, n in regs),
                        torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8).to(self.device)))
        return tuple(out)

    def sgd_table(self, tab, ctas_per_sm: int = 0, stream=None):
        """ctas_per_sm > 0: background launch (pc_sgd_step_ex) for a side stream."""
        n, mx, dev = tab
        self.lib.call("pc_sgd_step_ex", n, dev.data_ptr(), mx, self.lr, self.mom, self.wd, ctas_per_sm,
                      self.stream if stream is None else stream)

    def enable_bias_side(self, stream, ctas: int):
        """Single-replica plans: bias gradients of conv / FC layers run on ``stream``
        (pc_bias_grad: no shared memory, ``ctas`` CTAs) beside the data/weight-gradient
        GEMMs; the step program joins the stream before the update."""
        self.bias_side, self.bias_ctas = stream, int(ctas)
        ws = 16
        for st in self.layers:
            if st.kind in ("conv", "fc") and not st.col and not st.s2d:
                n = st.cl.out_shape[0]
                if n % 8 == 0:
                    ws = max(ws, self.lib.raw("pc_bias_grad_workspace")(self._bias_rows(st), n, self.bias_ctas))
        self.bias_ws = torch.empty(int(ws), dtype=torch.uint8, device=self.device)

    def _bias_rows(self, st) -> int:
        return self.B * st.geom.Ho * st.geom.Wo if st.kind == "conv" else self.B

    def _bias_fork(self, st) -> bool:
        """Launch layer st's bias gradient on the side stream (True) or leave it to
        the gradient kernels (False)."""
        side = getattr(self, "bias_side", None)
        n = st.cl.out_shape[0]
        if side is None or n % 8 or st.col or st.s2d:
            return False
        self._fork(side)
        self.lib.call("pc_bias_grad", self._bias_rows(st), n, st.gout.data_ptr(), self.prec,
                      self.g32[st.b_off:].data_ptr(), self.bias_ws.data_ptr(), self.bias_ws.numel(), self.bias_ctas,
                      side.cuda_stream)
        return True

    def enable_dgrad_weights(self):
        """bf16: per conv layer with a data gradient, a buffer for its filters in the
        data-gradient layout, filled by prepare_dgrad_weights (on a side stream at the
        start of the step) instead of by a transpose inside every backward call."""
        if self.prec != L.PC_BF16:
            return False
        for i, st in enumerate(self.layers):
            g = st.geom
            tc = g is not None and g.C % 8 == 0 and g.cs % 8 == 0 and g.N % 8 == 0 and \
                (g.C == g.cs or g.cstride % 8 == 0)   # the tensor-core data gradient (conv_tc_shape)
            if st.kind == "conv" and i > 0 and not st.col and not st.s2d and tc:
                st.wt = torch.empty(layout.numel(st.w_shape), dtype=torch.bfloat16, device=self.device)
        return any(st.wt is not None for st in self.layers)

    def prepare_dgrad_weights(self, stream):
        for st in self.layers:
            if st.wt is not None:
                self.lib.call("pc_conv2d_dgrad_weights", C.byref(st.geom), self._w_lowp(st), st.wt.data_ptr(),
                              self.prec, stream)

    def enable_wgrad_side(self, stream):
        """Single replica, fused update: each conv layer's weight gradient (+ bias and
        fused momentum update) runs on ``stream``, forked after its data gradient, so the
        persistent weight-gradient kernels fill the SMs the data-gradient chain leaves
        idle in its last wave (and vice versa); joined before the final update."""
        self.wg_side = stream
        self.ws_wg = torch.empty(max(self.ws_bytes, 16), dtype=torch.uint8, device=self.device)

    def enable_fc_side(self, stream, side_ctas: int, main_ctas: int, span: int):
        """Single replica, fused update: every FC layer's weight gradient + momentum
        update (HBM-bound: the FC6 update alone moves 680 MB) runs on ``stream`` with
        its GEMM grid capped at ``side_ctas`` CTAs, while the data-gradient chain keeps
        the main stream; the main-stream GEMMs are capped at ``main_ctas`` from the
        first fork through the next ``span`` conv layers, so the two chains run on
        disjoint SM sets instead of queueing behind each other's persistent grids."""
        self.fc_side, self.fc_side_ctas, self.fc_main_ctas, self.fc_span = stream, side_ctas, main_ctas, span
        self.ws_side = torch.empty(max(self.ws_bytes, 16), dtype=torch.uint8, device=self.device)
        self._main_cap_left = 0

    def _main_cap(self, st):
        """Grid cap of this main-stream layer's GEMMs while the FC side chain runs."""
        if getattr(self, "_main_cap_left", 0) <= 0 or st.kind not in ("conv", "fc"):
            return False
        self.lib.call("pc_set_grid_cap", self.fc_main_ctas)
        if st.kind == "conv":
            self._main_cap_left -= 1
        return True

    def _fork(self, side):
        """side waits for the current stream (and is remembered for join_side)."""
        side.wait_stream(torch.cuda.current_stream(self.device))
        self._forked = getattr(self, "_forked", [])
        if all(f is not side for f in self._forked):
            self._forked.append(side)

    def join_side(self):
        # only streams forked in this step program (joining an unforked stream during a
        # CUDA-graph capture would depend on work outside the capture)
        for side in getattr(self, "_forked", []):
            torch.cuda.current_stream(self.device).wait_stream(side)
        self._forked = []
        if getattr(self, "fc_side", None) is not None:
            self._main_cap_left = 0
            self.lib.call("pc_set_grid_cap", 0)

    def configure_fused_sgd(self, on: bool):
        """Single-replica plans (no gradient reduction between backward and update):
        the bf16 weight-gradient kernels of conv/FC layers apply the momentum-SGD
        update in their epilogue (pc_*_backward_ex) and never store the weight
        gradient; one SGD launch then covers only the remaining regions (biases and
        the masked input layer). ``grads_host`` is then valid for those regions only."""
        self.fuse_sgd = bool(on) and self.prec == L.PC_BF16
        self._fuse = {}
        if not self.fuse_sgd:
            self._sgd_regions = None
            return
        rest = []
        for st in self.layers:
            if st.w_off < 0:
                continue
            nw = layout.numel(st.w_shape)
            if st.kind in ("conv", "fc") and not st.s2d and not st.col:
                self._fuse[id(st)] = L.SgdFuse(self.p32[st.w_off:].data_ptr(), self.v32[st.w_off:].data_ptr(),
                                               self.plow[st.w_off:].data_ptr(), self.lr, self.mom, self.wd)
            else:
                rest.append((st.w_off, nw))
            rest.append((st.b_off, st.cl.bias_shape[0]))
        tabs = [L.SgdTensor(self.p32[o:].data_ptr(), self.v32[o:].data_ptr(), self.g32[o:].data_ptr(),
                            self.plow[o:].data_ptr(), n) for o, n in rest]
        arr = (L.SgdTensor * len(tabs))(*tabs)
        self.sgd_numel_fused = sum(n for _, n in rest)
        self._sgd_regions = (len(tabs), max(n for _, n in rest),
                             torch.frombuffer(bytearray(bytes(arr)), dtype=torch.uint8).to(self.device))

    # ------------------------------------------------------ parameter transfer
    def _w_lowp(self, st):
        src = self.plow if self.plow is not None else self.p32
        return src[st.w_off:].data_ptr()

    def load_params(self, col_params: dict, velocity: dict | None = None):
        """col_params: reference-layout column ParamSet (float64 numpy)."""
        hp = np.zeros(self.n_flat, dtype=np.float32)
        hv = np.zeros(self.n_flat, dtype=np.float32)
        for st in self.layers:
            if st.w_off < 0:
                continue
            idx = st.cl.index
            for buf, tree in ((hp, col_params), (hv, velocity)):
                if tree is None:
                    continue
                w = tree[idx]["w"]
                if st.col:
                    dw = np.zeros(st.w_shape, dtype=np.float32)
                    dw[:, : w[0].size] = w.reshape(w.shape[0], -1)
                elif st.s2d:
                    dw = layout.conv_to_device_s2d(w, st.s2d, st.cp)
                elif st.kind == "conv":
                    dw = layout.conv_to_device(w, st.cp)
                else:
                    dw = layout.fc_to_device(w, st.perm)
                buf[st.w_off:st.w_off + dw.size] = dw.ravel()
                b = np.asarray(tree[idx]["b"], dtype=np.float32)
                buf[st.b_off:st.b_off + b.size] = b
        self.p32.copy_(torch.from_numpy(hp))
        self.v32.copy_(torch.from_numpy(hv))
        if self.plow is not None:
            self.plow.copy_(self.p32)

    def _unflatten(self, flat: np.ndarray) -> dict:
        out = {}
        for st in self.layers:
            if st.w_off < 0:
                continue
            n = layout.numel(st.w_shape)
            wd = flat[st.w_off:st.w_off + n].reshape(st.w_shape)
            if st.col:
                w = wd[:, : math.prod(st.cl.weight_shape[1:])].reshape(st.cl.weight_shape).astype(np.float64)
            elif st.s2d:
                w = layout.conv_from_device_s2d(wd, st.cl.weight_shape[1], st.cl.weight_shape[2], st.s2d)
            elif st.kind == "conv":
                w = layout.conv_from_device(wd, st.cl.weight_shape[1])
            else:
                w = layout.fc_from_device(wd, st.perm)
            nb = st.cl.bias_shape[0]
            out[st.cl.index] = {"w": w, "b": flat[st.b_off:st.b_off + nb].astype(np.float64)}
        return out

    def params_host(self) -> dict:
        return self._unflatten(self.p32.cpu().numpy())

    def velocity_host(self) -> dict:
        return self._unflatten(self.v32.cpu().numpy())

    def grads_host(self, g: torch.Tensor | None = None) -> dict:
        if g is None and getattr(self, "fuse_sgd", False):
            raise RuntimeError("weight gradients were consumed by the fused update; "
                               "set fabric.fuse_sgd = False before setup_workers to read them")
        return self._unflatten((self.g32 if g is None else g).cpu().numpy())

    def activation_host(self, i: int, which: str = "out") -> np.ndarray:
        """Layer i's forward output (or input gradient) back in the reference's
        NCHW float64 layout, for layer-by-layer parity tests."""
        st = self.layers[i]
        t = getattr(st, which)
        shape = st.out_nhwc if which == "out" else st.in_nhwc
        blocks = 1 if which == "out" else st.in_blocks
        a = t[: self.B * math.prod(shape)].float().cpu().numpy().astype(np.float64)
        if blocks > 1:
            per = (shape[:-1] + (shape[-1] // blocks,))
            a = a.reshape((blocks, self.B) + per)
            a = np.concatenate(list(a), axis=-1)
        else:
            a = a.reshape((self.B,) + tuple(shape))
        if a.ndim == 4:
            a = a.transpose(0, 3, 1, 2)
            if st.kind == "conv" and which == "gin" and self.in_cp != self.in_c and i == 0:
                a = a[:, : self.in_c]
        return np.ascontiguousarray(a)

    def pool_argmax_host(self) -> dict:
        """{layer index: int64 NCHW local-window argmax} of the last forward pass."""
        out = {}
        for st in self.layers:
            if st.kind == "pool":
                ho, wo, c = st.out_nhwc
                a = st.argmax[: self.B * ho * wo * c].cpu().numpy().reshape(self.B, ho, wo, c)
                out[st.cl.index] = np.ascontiguousarray(a.transpose(0, 3, 1, 2)).astype(np.int64)
        return out

    # ------------------------------------------------------------ step program
    @property
    def stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    def _call(self, st, name: str, *args, tag: str = ""):
        """C-ABI call of one layer pass; with ``PROFILE`` set, bracketed by CUDA
        events on the launching stream (bench.py's per-kernel roofline)."""
        return self._pcall(st.cl.index, st.kind, name, *args, tag=tag)

    def _pcall(self, idx: int, kind: str, name: str, *args, tag: str = ""):
        if PROFILE is None:
            return self.lib.call(name, *args)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        self.lib.call(name, *args)
        b.record()
        PROFILE.append((self.wid, idx, kind, name + tag, a, b))

    def _split_backward(self, st, name: str, flags: int, call):
        """Under ``PROFILE``, issue a backward pass as its data-gradient and its
        weight-gradient halves (separately timed); otherwise one call."""
        if PROFILE is None or not (flags & L.PC_WANT_DX) or not (flags & L.PC_WANT_DW):
            return call(flags, "")
        call(flags & ~L.PC_WANT_DW, "[dx]")
        call(flags & ~(L.PC_WANT_DX | L.PC_MASK_DX), "[dw]")

    def load_batch(self, x_nchw: torch.Tensor, labels_i32: torch.Tensor):
        """x_nchw: device (B, C, H, W) slice of the global batch: float32, or bf16
        for the explicit-im2col input layer (the bf16 rounding the device would
        apply anyway, done by the caller's input pipeline)."""
        c, h, w = self.cs.base.input_shape
        src_prec = {torch.bfloat16: L.PC_BF16, torch.float64: L.PC_FP64}.get(x_nchw.dtype, L.PC_FP32)
        self.x_src_es = x_nchw.element_size()
        if self.s2d:
            lay = self.cs.col_layers[0].layer
            self._pcall(-1, "input", "pc_space_to_depth_ex" if self.prec == L.PC_BF16 else "pc_space_to_depth_f32",
                        self.B, c, h, w, lay.stride, lay.pad, 64, x_nchw.data_ptr(), src_prec, self.s2d_ones,
                        self.x.data_ptr(), self.stream)
        elif self.col_kp:
            lay = self.cs.col_layers[0].layer
            self._pcall(-1, "input", "pc_im2col_ex", self.B, c, h, w, lay.kernel, lay.stride, lay.pad, self.col_kp,
                          x_nchw.data_ptr(), L.PC_BF16 if x_nchw.dtype == torch.bfloat16 else L.PC_FP32,
                          self.x.data_ptr(), self.prec, self.stream)
        else:
            self._pcall(-1, "input", "pc_nchw_to_nhwc", self.B, c, h, w, self.in_cp, x_nchw.data_ptr(),
                          self.x.data_ptr(), self.prec, self.stream)
        self.labels[: self.B].copy_(labels_i32, non_blocking=True)

    def forward(self, i: int, loss_scale: float):
        st, lib, s = self.layers[i], self.lib, self.stream
        if st.kind == "conv" and st.col:
            g = st.geom
            mat = L.Mat(st.inp.data_ptr(), st.col, st.col, 0)
            self._call(st, "pc_fc_forward", self.B * g.Ho * g.Wo, st.col, g.N, C.byref(mat), self._w_lowp(st),
                       self.p32[st.b_off:].data_ptr(), st.out.data_ptr(), self.cprec,
                       L.PC_RELU if st.relu_after else 0, s)
        elif st.kind == "conv":
            flags = L.PC_RELU if st.relu_after else 0
            if st.s2d and st.cp - self.in_c * st.s2d ** 2 >= 16 and os.environ.get("PC_ZERO_TAIL", "1") != "0":
                flags |= L.PC_ZERO_TAIL16   # channels >= 48 of the 64 are structural zeros (and the ones channel)
            self._call(st, "pc_conv2d_forward", C.byref(st.geom), st.inp.data_ptr(), self._w_lowp(st),
                     self.p32[st.b_off:].data_ptr(), st.out.data_ptr(), self.cprec, flags, s)
        elif st.kind == "fc":
            d = math.prod(st.in_nhwc)
            mat = self._in_mat(st)
            flags = L.PC_RELU if st.relu_after else 0
            self._call(st, "pc_fc_forward_ex", self.B, d, st.cl.out_shape[0], C.byref(mat), self._w_lowp(st),
                       self.p32[st.b_off:].data_ptr(), st.out.data_ptr(), self.cprec, flags, self.ws.data_ptr(),
                       self.ws_bytes, s)
        elif st.kind == "relu":
            if not st.relu_fused_fwd:
                self._call(st, "pc_relu_forward", self.B * math.prod(st.in_nhwc), st.inp.data_ptr(),
                         st.out.data_ptr(), self.prec, s)
        elif st.kind == "lrn":
            lay = st.cl.layer
            hh, ww, cc = st.in_nhwc
            self._call(st, "pc_lrn_forward", self.B * hh * ww, cc, lay.size, lay.k, lay.alpha, lay.beta,
                       st.inp.data_ptr(), st.out.data_ptr(), self.prec, s)
        elif st.kind == "dropout":
            if self.training:
                self._dropout(st, st.inp, st.out)
            else:
                st.out[: st.inp.numel()].copy_(st.inp)
        elif st.kind == "pool":
            hh, ww, cc = st.in_nhwc
            self._call(st, "pc_maxpool_forward", self.B, hh, ww, cc, st.cl.layer.kernel, st.cl.layer.stride,
                     st.inp.data_ptr(), st.out.data_ptr(), st.argmax.data_ptr(), self.prec, s)
        else:
            k = st.cl.layer.classes
            # loss + gradient + the step loss's fixed-order sum in one launch
            self._call(st, "pc_softmax_xent_loss", self.B, k, st.inp.data_ptr(), self.labels.data_ptr(),
                       float(loss_scale), st.out.data_ptr(), st.row_loss.data_ptr(), self.bad_label.data_ptr(),
                       self.loss.data_ptr(), self.loss_ticket.data_ptr(), self.prec, s)

    def _dropout(self, st, src, dst):
        hh, ww, cc, cdense, coff, thresh = st.drop
        self._call(st, "pc_dropout", self.B, hh, ww, cc, cdense, coff, self.replica * self.B, self.dropout_seed,
                   self.step_ctr.data_ptr(), st.cl.index, thresh, st.cl.layer.p, src.data_ptr(), dst.data_ptr(),
                   self.prec, self.stream)

    def _in_mat(self, st) -> L.Mat:
        d = math.prod(st.in_nhwc)
        ds = d // st.in_blocks
        return L.Mat(st.inp.data_ptr(), ds, ds, self.B * ds)

    def backward(self, i: int):
        capped = self._main_cap(self.layers[i])
        try:
            self._backward(i)
        finally:
            if capped:
                self.lib.call("pc_set_grid_cap", 0)

    def _backward(self, i: int):
        st, lib, s = self.layers[i], self.lib, self.stream
        want_dx = i > 0
        if st.kind == "conv" and st.col:      # input layer: weight / bias gradients only
            g = st.geom
            mat = L.Mat(st.inp.data_ptr(), st.col, st.col, 0)
            self._call(st, "pc_fc_backward", self.B * g.Ho * g.Wo, st.col, g.N, C.byref(mat), self._w_lowp(st),
                       st.gout.data_ptr(), C.byref(mat), None, self.g32[st.w_off:].data_ptr(),
                       self.g32[st.b_off:].data_ptr(), self.cprec, L.PC_WANT_DW, self.ws.data_ptr(),
                       self.ws_bytes, s)
        elif st.kind == "conv":
            flags = L.PC_WANT_DW | (L.PC_WANT_DX if want_dx else 0) | (L.PC_MASK_DX if st.mask_dx else 0)
            upd = self._fuse.get(id(st)) if getattr(self, "_fuse", None) else None
            no_gb = (st.s2d and self.s2d_ones >= 0) or st.bias_by_pool or self._bias_fork(st)
            w_ptr = self._w_lowp(st)
            if want_dx and st.wt is not None and self.wt_ready:
                flags |= L.PC_WT_PRESET
                w_ptr = st.wt.data_ptr()
            wg = getattr(self, "wg_side", None)
            if wg is not None and upd is not None and PROFILE is None and (not want_dx or flags & L.PC_WT_PRESET):
                # data gradient here (it reads the prepared filters, not the ones the fused
                # update rewrites); weight gradient + bias + update on the side stream
                gb = None if no_gb else self.g32[st.b_off:].data_ptr()
                if want_dx:
                    self.lib.call("pc_conv2d_backward_ex", C.byref(st.geom), st.inp.data_ptr(), w_ptr,
                                  st.gout.data_ptr(), st.gin.data_ptr(), st.inp.data_ptr() if st.mask_dx else None,
                                  None, None, self.cprec, flags & ~L.PC_WANT_DW, None, 0, None, s)
                self._fork(wg)
                cap = WG_CTAS.get(st.cl.index, WG_CTAS.get(-1, 0))
                if cap:
                    self.lib.call("pc_set_grid_cap", cap)
                try:
                    self.lib.call("pc_conv2d_backward_ex", C.byref(st.geom), st.inp.data_ptr(), w_ptr,
                                  st.gout.data_ptr(), None, None, self.g32[st.w_off:].data_ptr(), gb, self.cprec,
                                  L.PC_WANT_DW, self.ws_wg.data_ptr(), self.ws_bytes, C.byref(upd), wg.cuda_stream)
                finally:
                    if cap:
                        self.lib.call("pc_set_grid_cap", 0)
                if st.keep is not None:   # (not reached: the input layer's update is not fused)
                    raise RuntimeError("weight-gradient side stream: masked layer")
                return
            self._split_backward(st, "pc_conv2d_backward_ex", flags, lambda f, tag: self._call(
                st, "pc_conv2d_backward_ex", C.byref(st.geom), st.inp.data_ptr(), w_ptr,
                st.gout.data_ptr(), st.gin.data_ptr() if want_dx else None,
                st.inp.data_ptr() if st.mask_dx else None,
                self.g32[st.w_off:].data_ptr(), None if no_gb else self.g32[st.b_off:].data_ptr(), self.cprec, f,
                self.ws.data_ptr(), self.ws_bytes, C.byref(upd) if upd is not None else None, s, tag=tag))
        elif st.kind == "fc":
            d = math.prod(st.in_nhwc)
            u = st.cl.out_shape[0]
            xm = self._in_mat(st)
            gm = L.Mat(st.gin.data_ptr() if want_dx else st.inp.data_ptr(), xm.ld, xm.cb, xm.bstride)
            flags = L.PC_WANT_DW | (L.PC_WANT_DX if want_dx else 0) | (L.PC_MASK_DX if st.mask_dx else 0)
            upd = self._fuse.get(id(st)) if getattr(self, "_fuse", None) else None
            no_gb = self._bias_fork(st)

            def fc_call(f, tag, stream=s, ws=self.ws):
                self._call(st, "pc_fc_backward_ex", self.B, d, u, C.byref(xm), self._w_lowp(st), st.gout.data_ptr(),
                           C.byref(gm), st.inp.data_ptr() if st.mask_dx else None,
                           self.g32[st.w_off:].data_ptr(), None if no_gb else self.g32[st.b_off:].data_ptr(),
                           self.cprec, f, ws.data_ptr(), self.ws_bytes, C.byref(upd) if upd is not None else None,
                           stream, tag=tag)

            side = getattr(self, "fc_side", None)
            if side is not None and upd is not None and PROFILE is None:
                # data gradient here; weight gradient + fused update on the side chain, forked
                # after the data gradient (which reads the pre-update weights)
                if want_dx:
                    fc_call(flags & ~L.PC_WANT_DW, "")
                self._fork(side)
                self.lib.call("pc_set_grid_cap", self.fc_side_ctas)
                try:
                    fc_call(flags & ~(L.PC_WANT_DX | L.PC_MASK_DX), "", stream=side.cuda_stream, ws=self.ws_side)
                finally:
                    self.lib.call("pc_set_grid_cap", 0)
                self._main_cap_left = self.fc_span
            else:
                self._split_backward(st, "pc_fc_backward_ex", flags, fc_call)
        elif st.kind == "relu":
            if not st.skip_bwd and want_dx:
                self._call(st, "pc_relu_backward", self.B * math.prod(st.in_nhwc), st.inp.data_ptr(),
                         st.gout.data_ptr(), st.gin.data_ptr(), self.prec, s)
        elif st.kind == "lrn":
            if want_dx:
                lay = st.cl.layer
                hh, ww, cc = st.in_nhwc
                self._call(st, "pc_lrn_backward", self.B * hh * ww, cc, lay.size, lay.k, lay.alpha, lay.beta,
                           st.inp.data_ptr(), st.gout.data_ptr(), st.gin.data_ptr(), self.prec, s)
        elif st.kind == "dropout":
            if want_dx:
                self._dropout(st, st.gout, st.gin)
        elif st.kind == "pool":
            if want_dx:
                hh, ww, cc = st.in_nhwc
                if st.pool_bias >= 0:
                    cv = self.layers[st.pool_bias]
                    self._call(st, "pc_maxpool_backward_bias", self.B, hh, ww, cc, st.cl.layer.kernel,
                               st.cl.layer.stride, st.gout.data_ptr(), st.argmax.data_ptr(),
                               st.inp.data_ptr() if st.mask_dx else None, st.gin.data_ptr(), self.prec,
                               self.g32[cv.b_off:].data_ptr(), self.pool_ws.data_ptr(), self.pool_ws.numel(), s)
                else:
                    self._call(st, "pc_maxpool_backward", self.B, hh, ww, cc, st.cl.layer.kernel,
                               st.cl.layer.stride, st.gout.data_ptr(), st.argmax.data_ptr(),
                               st.inp.data_ptr() if st.mask_dx else None, st.gin.data_ptr(), self.prec, s)
        if st.keep is not None and self.s2d_ones >= 0:
            self._call(st, "pc_s2d_wgrad_finish", st.w_shape[0], st.keep.numel() // st.w_shape[0], self.s2d_ones,
                          st.keep.data_ptr(), self.g32[st.w_off:].data_ptr(), self.g32[st.b_off:].data_ptr(), s)
        elif st.keep is not None:
            self.lib.call("pc_mask_f32", st.keep.numel(), st.keep.data_ptr(), self.g32[st.w_off:].data_ptr(),
                          s)
        if st.cl.cross and st.cl.shared and want_dx and self.m > 1:
            n = st.gin.numel()
            self._call(st, "pc_scale", n, st.gin.data_ptr(), st.gin.data_ptr(), 1.0 / self.m, self.prec, s)

    def sgd_numel(self) -> int:
        """Elements the final pc_sgd_step launch updates (bench.py's byte count)."""
        if getattr(self, "_sgd_regions", None) is not None:
            return int(self.sgd_numel_fused)
        return int(self.n_flat)

    def sgd(self):
        if self.has_dropout:  # next step draws fresh masks
            self.lib.call("pc_counter_add", self.step_ctr.data_ptr(), 1, self.stream)
        if getattr(self, "_sgd_regions", None) is not None:
            n, mx, tab = self._sgd_regions
            self._pcall(-1, "sgd", "pc_sgd_step", n, tab.data_ptr(), mx, self.lr, self.mom, self.wd, self.stream)
            return
        self._pcall(-1, "sgd", "pc_sgd_step", 1, self._sgd_dev.data_ptr(), self.n_flat, self.lr, self.mom, self.wd,
                      self.stream)

    @property
    def n_layers(self) -> int:
        return len(self.layers)
