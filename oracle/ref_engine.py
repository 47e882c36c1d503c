"""TEST INFRASTRUCTURE ONLY — float64 restatement of the reference step engine.

Restates `/root/reference/pkg/src/parconv/schemes.py`:

* ``column_fwd_bwd`` (`schemes.py:342-419`) for all m columns of one replica
  at once: at a cross layer the columns' slices are concatenated along axis 1
  in ascending column order (`schemes.py:296-305`); on the way back the
  full-width gradient of every column is split into m channel pieces and
  column k receives the ascending-order sum of everyone's piece k
  (`schemes.py:307-318`), shared layers pre-dividing by m (`:412-414`).
* ``OracleFabric.step`` = ``hybrid_step`` (`schemes.py:500-569`): contiguous
  replica shards, loss scale 1/B_global, per-column gradient sum over the
  replicas in ascending worker order (`fabric.py:146-156`), SGD at the
  column root, parameters broadcast to every replica.
* ``reference_step`` (`schemes.py:439-458`).

The optional ``trace`` dict records every layer's forward output and every
layer's input gradient, per column, for layer-by-layer parity tests.
"""

from __future__ import annotations

import numpy as np

from paper_1312_5853_b200.netdef import FC, LRN, Conv, Dropout, MaxPool, ReLU, SoftmaxXent, columnize
from paper_1312_5853_b200 import rng
from paper_1312_5853_b200.plan import (
    params_as_lists,
    lists_as_params,
    split_params,
    merge_params,
    plan_columnized,
)

from . import ref_kernels as K


def dropout_index(cs, cl, batch_rows, row0, column):
    """Dense-activation element indices (NCHW flatten, global batch row-major) of
    column ``column``'s slice of dropout layer ``cl``'s input for global sample
    rows row0 .. row0 + batch_rows - 1 (the mask contract of rng.dropout_state)."""
    m = cs.columns
    split = column_split_before(cs, cl.index)
    shape = cl.in_shape
    per = int(np.prod(shape))
    cols = m if split else 1
    dense = per * cols
    j = column if split else 0
    rows = (row0 + np.arange(batch_rows, dtype=np.int64)).reshape(-1, *([1] * len(shape)))
    if len(shape) == 3:
        c, h, w = shape
        cc = (j * c + np.arange(c)).reshape(c, 1, 1)
        f = (cc * h + np.arange(h).reshape(1, h, 1)) * w + np.arange(w).reshape(1, 1, w)
    else:
        f = j * shape[0] + np.arange(shape[0])
    return rows * dense + f


def column_split_before(cs, index):
    """True when the activation entering layer ``index`` is split across columns
    (a non-shared conv/fc upstream, no cross point since), False when replicated."""
    rep = True
    for cl in cs.col_layers:
        if cl.index == index:
            return cs.columns > 1 and not rep
        if cl.cross:
            rep = True
        if isinstance(cl.layer, (Conv, FC)):
            rep = cl.shared
    raise ValueError(index)


def column_fwd_bwd(cs, col_params, x, labels, loss_scale, trace=None, force_argmax=None, dropout=None,
                   force_relu=None):
    """All m columns of one replica; returns (per-column losses, per-column grads).

    ``dropout`` = (seed, step, row0): the training step's dropout stream and the
    replica's first global sample row (rng.dropout_state); None: no dropout
    layers may be present.

    ``force_argmax`` ({layer: [per-column argmax]}) replays another engine's
    max-pool decisions ("teacher forcing"): where a window holds a near-tie
    that float32 and float64 rank differently, the checker then measures the
    arithmetic of the rest of the step instead of the tie's routing.
    ``force_relu`` ({layer: [per-column bool mask]}) does the same for ReLU
    decisions at pre-activations within rounding of zero: the backward passes
    the gradient where the forced mask is set."""
    m = cs.columns
    acts = [np.asarray(x, dtype=np.float64)] * m
    caches = []
    losses = [0.0] * m
    glog = [None] * m
    for cl in cs.col_layers:
        if cl.cross:
            full = np.concatenate(acts, axis=1)
            acts = [full] * m
        cache = [{"in": a} for a in acts]
        outs = []
        for j in range(m):
            a, p, L = acts[j], col_params[j].get(cl.index), cl.layer
            if isinstance(L, Conv):
                o = K.conv2d_forward(a, p["w"], p["b"], L.stride, L.pad)
            elif isinstance(L, FC):
                cache[j]["flat"] = a.reshape(a.shape[0], -1)
                o = K.fc_forward(cache[j]["flat"], p["w"], p["b"])
            elif isinstance(L, ReLU):
                o = K.relu_forward(a)
            elif isinstance(L, LRN):
                o = K.lrn_forward(a, L.size, L.k, L.alpha, L.beta)
            elif isinstance(L, Dropout):
                seed, step, row0 = dropout
                idx = dropout_index(cs, cl, a.shape[0], row0, j)
                cache[j]["keep"] = rng.dropout_keep(seed, step, cl.index, idx, L.p)
                o = K.dropout_forward(a, cache[j]["keep"], L.p)
            elif isinstance(L, MaxPool):
                o, cache[j]["arg"] = K.maxpool_forward(a, L.kernel, L.stride)
                if force_argmax is not None and cl.index in force_argmax:
                    cache[j]["arg"] = np.asarray(force_argmax[cl.index][j], dtype=np.int64)
            else:
                losses[j], glog[j] = K.softmax_xent_scaled(a.reshape(a.shape[0], -1), labels, loss_scale)
                o = glog[j]
            outs.append(o)
        if trace is not None:
            trace.setdefault("fwd", {})[cl.index] = outs
            if any("arg" in c for c in cache):
                trace.setdefault("argmax", {})[cl.index] = [c["arg"] for c in cache]
        caches.append(cache)
        acts = outs

    grads = [dict() for _ in range(m)]
    g = [None] * m
    for pos in range(len(cs.col_layers) - 1, -1, -1):
        cl, cache, L = cs.col_layers[pos], caches[pos], cs.col_layers[pos].layer
        gin = []
        for j in range(m):
            c = cache[j]
            if isinstance(L, SoftmaxXent):
                gi = glog[j].reshape(c["in"].shape)
            elif isinstance(L, Conv):
                p = col_params[j][cl.index]
                gi, gw, gb = K.conv2d_backward(c["in"], p["w"], g[j], L.stride, L.pad)
                grads[j][cl.index] = {"w": gw, "b": gb}
            elif isinstance(L, FC):
                gi, gw, gb = K.fc_backward(c["flat"], col_params[j][cl.index]["w"], g[j])
                grads[j][cl.index] = {"w": gw, "b": gb}
                gi = gi.reshape(c["in"].shape)
            elif isinstance(L, ReLU):
                if force_relu is not None and cl.index in force_relu:
                    gi = np.where(np.asarray(force_relu[cl.index][j], dtype=bool), g[j], 0.0)
                else:
                    gi = K.relu_backward(c["in"], g[j])
            elif isinstance(L, LRN):
                gi = K.lrn_backward(c["in"], g[j], L.size, L.k, L.alpha, L.beta)
            elif isinstance(L, Dropout):
                gi = K.dropout_backward(g[j], c["keep"], L.p)
            else:
                gi = K.maxpool_backward(c["in"].shape, L.kernel, L.stride, g[j], c["arg"])
            gin.append(gi)
        if trace is not None:
            trace.setdefault("bwd", {})[cl.index] = gin
        if cl.cross:
            contrib = [gi / m for gi in gin] if cl.shared else gin
            width = contrib[0].shape[1] // m
            new = []
            for k in range(m):
                acc = None
                for src in range(m):
                    piece = contrib[src][:, k * width:(k + 1) * width]
                    acc = np.array(piece, copy=True) if acc is None else acc + piece
                new.append(acc)
            g = new
        else:
            g = gin
    return losses, grads


def reference_step(net, params, batch, velocity=None, lr=0.01, momentum=0.9, weight_decay=0.0005,
                   dropout_seed=0, step=0):
    """Dense single-worker step; returns (loss, new_params, new_velocity)."""
    cs = columnize(net, 1)
    x, y = batch
    losses, grads = column_fwd_bwd(cs, [params], x, y, 1.0 / x.shape[0], dropout=(dropout_seed, step, 0))
    plist = params_as_lists(params, cs)
    vlist = velocity if velocity is not None else [np.zeros_like(p) for p in plist]
    newp, newv = K.sgd_step(plist, params_as_lists(grads[0], cs), vlist, lr, momentum, weight_decay)
    return losses[0], lists_as_params(newp, cs), newv


class OracleFabric:
    """Sequential simulation of a d x m plan (state per column; replicas are
    bit-identical after every step, as in the reference's broadcast)."""

    def __init__(self, net, plan, dense_params, lr=0.01, momentum=0.9, weight_decay=0.0005):
        self.net, self.plan = net, plan
        self.cs = plan_columnized(net, plan)
        m = plan.model_columns
        self.params = [split_params(dense_params, self.cs, j) for j in range(m)]
        self.velocity = [[np.zeros_like(p) for p in params_as_lists(self.params[j], self.cs)]
                         for j in range(m)]
        self.hyper = (lr, momentum, weight_decay)
        self.dropout_seed, self.steps = 0, 0   # dropout stream (rng.dropout_state): seed, step counter

    def step(self, x, y, trace=None, force_argmax=None, force_relu=None):
        """force_argmax / force_relu: {layer: [replica][column] arrays} (see column_fwd_bwd)."""
        d, m = self.plan.data_shards, self.plan.model_columns
        b = x.shape[0]
        if b % d:
            raise ValueError(f"batch size {b} not divisible by {d} data shards")
        shard, scale = b // d, 1.0 / b
        labels = np.asarray(y, dtype=np.int64)
        per_replica = []
        total = 0.0
        for r in range(d):
            lo, hi = r * shard, (r + 1) * shard
            fa = None if force_argmax is None else {k: v[r] for k, v in force_argmax.items()}
            fr = None if force_relu is None else {k: v[r] for k, v in force_relu.items()}
            losses, grads = column_fwd_bwd(self.cs, self.params, x[lo:hi], labels[lo:hi], scale,
                                           trace=trace if r == 0 else None, force_argmax=fa,
                                           dropout=(self.dropout_seed, self.steps, lo), force_relu=fr)
            per_replica.append(grads)
            total += losses[0]
        for j in range(m):
            summed = None
            for r in range(d):
                gl = params_as_lists(per_replica[r][j], self.cs)
                summed = [np.array(g, copy=True) for g in gl] if summed is None else \
                    [a + g for a, g in zip(summed, gl)]
            if trace is not None:
                trace.setdefault("grads", {})[j] = lists_as_params(summed, self.cs)
            newp, newv = K.sgd_step(params_as_lists(self.params[j], self.cs), summed,
                                    self.velocity[j], *self.hyper)
            self.params[j] = lists_as_params(newp, self.cs)
            self.velocity[j] = newv
        self.steps += 1
        return total

    def evaluation_errors(self, x, labels):
        """`schemes.py:600-645`: misclassifications of replica 0's columns (forward
        only, the head's logits, argmax ties -> lowest class)."""
        x = np.asarray(x, dtype=np.float64)
        if x.shape[0] == 0:
            return 0
        trace = {}
        head = [cl.index for cl in self.cs.col_layers if isinstance(cl.layer, FC)][-1]
        column_fwd_bwd(self.cs, self.params, x, np.zeros(x.shape[0], dtype=np.int64), 1.0, trace=trace,
                       dropout=None if not any(isinstance(cl.layer, Dropout) for cl in self.cs.col_layers)
                       else (self.dropout_seed, self.steps, 0))
        logits = trace["fwd"][head][0].reshape(x.shape[0], -1)
        return int(np.count_nonzero(np.argmax(logits, axis=1) != np.asarray(labels, dtype=np.int64)))

    def dense_params(self):
        return merge_params(self.params, self.cs)
