"""Parallel plans, dense parameter sets and the communication closed forms.

Host logic around the step (reference `pkg/src/parconv/schemes.py:68-269`
and `:653-733`):

* ``ParallelPlan(d, m, cross)``: worker (i, j) = replica i, column j,
  flat id i*m + j.
* ``init_dense_params``: He-normal std sqrt(2/fan_in) per layer from the
  INIT substream, drawn in the dense layout, biases zero (`schemes.py:128-153`).
* ``split_params`` / ``merge_params``: column slices of conv filters (and of
  input channels for grouped layers) and of FC units; the head is copied.
* ``pack_tree`` canonical order: ascending layer, weights then bias.
* ``comm_phases`` / ``comm_volume``: the reference's logical ledger, which
  the device fabric books per step so ``fabric.ledger`` equals the closed
  form exactly.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import rng
from .errors import ValidationError
from .netdef import WIRE_ELEMENT_SIZE, ColumnizedSpec, Conv, NetworkSpec, columnize

ParamSet = dict  # layer index -> {"w": ndarray, "b": ndarray}


@dataclass(frozen=True)
class ParallelPlan:
    data_shards: int = 1
    model_columns: int = 1
    cross_layers: tuple = ()

    def __post_init__(self):
        if self.data_shards < 1 or self.model_columns < 1:
            raise ValidationError("data_shards and model_columns must be >= 1")

    @property
    def workers(self) -> int:
        return self.data_shards * self.model_columns

    def worker_of(self, replica: int, column: int) -> int:
        return replica * self.model_columns + column

    def describe(self) -> str:
        return f"d{self.data_shards}xm{self.model_columns}"


def parse_plan(text: str) -> ParallelPlan:
    vals = {"data_shards": 1, "model_columns": 1, "cross_layers": ()}
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        parts = line.split(None, 1)
        key, rest = parts[0].lower(), (parts[1].strip() if len(parts) > 1 else "")
        if key not in vals:
            raise ValidationError(f"line {lineno}: unknown plan key {key!r}")
        try:
            if key == "cross_layers":
                vals[key] = tuple(int(t) for t in rest.replace(",", " ").split())
            else:
                vals[key] = int(rest)
        except ValueError:
            raise ValidationError(f"line {lineno}: bad integer in {line!r}") from None
    return ParallelPlan(vals["data_shards"], vals["model_columns"], vals["cross_layers"])


def load_plan(path) -> ParallelPlan:
    return parse_plan(Path(path).read_text(encoding="utf-8"))


def plan_columnized(net: NetworkSpec, plan: ParallelPlan) -> ColumnizedSpec:
    return columnize(net, plan.model_columns, plan.cross_layers)


# ---------------------------------------------------------------------------
# Dense parameters and column slices
# ---------------------------------------------------------------------------


def init_dense_params(net: NetworkSpec, seed: int, std: float | None = None) -> ParamSet:
    stream = rng.derive(seed, rng.DOMAIN_INIT)
    params: ParamSet = {}
    for cl in columnize(net, 1).param_layers():
        if std is not None:
            scale = std
        elif isinstance(cl.layer, Conv):
            scale = math.sqrt(2.0 / (cl.in_shape[0] * cl.layer.kernel ** 2))
        else:
            scale = math.sqrt(2.0 / cl.weight_shape[0])
        params[cl.index] = {"w": stream.gauss_array(cl.weight_shape, std=scale),
                            "b": np.zeros(cl.bias_shape, dtype=np.float64)}
    return params


def dense_layers(cs: ColumnizedSpec) -> dict:
    return {cl.index: cl for cl in columnize(cs.base, 1).param_layers()}


def split_params(dense: ParamSet, cs: ColumnizedSpec, column: int) -> ParamSet:
    out: ParamSet = {}
    for cl in cs.param_layers():
        w, b = dense[cl.index]["w"], dense[cl.index]["b"]
        if cl.shared:
            out[cl.index] = {"w": w.copy(), "b": b.copy()}
            continue
        if isinstance(cl.layer, Conv):
            oc, ic = cl.weight_shape[0], cl.weight_shape[1]
            rows = slice(column * oc, (column + 1) * oc)
            ws = w[rows]
            if ic != w.shape[1]:        # grouped conv: own input-channel slice only
                ws = ws[:, column * ic:(column + 1) * ic]
            bs = b[rows]
        else:
            u = cl.weight_shape[1]
            ws, bs = w[:, column * u:(column + 1) * u], b[column * u:(column + 1) * u]
        out[cl.index] = {"w": np.ascontiguousarray(ws), "b": np.ascontiguousarray(bs)}
    return out


def merge_params(per_column: list, cs: ColumnizedSpec) -> ParamSet:
    m = cs.columns
    if len(per_column) != m:
        raise ValidationError(f"merge_params needs {m} column sets, got {len(per_column)}")
    dl = dense_layers(cs)
    out: ParamSet = {}
    for cl in cs.param_layers():
        i = cl.index
        if cl.shared:
            first = per_column[0][i]
            if any(not np.array_equal(pc[i]["w"], first["w"]) for pc in per_column[1:]):
                raise ValidationError(f"layer {i}: replicated head copies diverged across columns")
            out[i] = {"w": first["w"].copy(), "b": first["b"].copy()}
            continue
        if not cl.cross and cl.in_shape != dl[i].in_shape:
            raise ValidationError(
                f"layer {i} consumes a column slice (grouped); no dense equivalent exists")
        axis = 0 if isinstance(cl.layer, Conv) else 1
        w = np.concatenate([pc[i]["w"] for pc in per_column], axis=axis)
        b = np.concatenate([pc[i]["b"] for pc in per_column])
        out[i] = {"w": np.ascontiguousarray(w, dtype=np.float64), "b": b.astype(np.float64)}
    return out


def pack_tree(tree: ParamSet, cs: ColumnizedSpec) -> np.ndarray:
    parts = [tree[cl.index][k].ravel() for cl in cs.param_layers() for k in ("w", "b")]
    return np.concatenate(parts) if parts else np.zeros(0)


def unpack_tree(flat: np.ndarray, cs: ColumnizedSpec) -> ParamSet:
    if flat.size != cs.column_param_count:
        raise ValidationError(f"packed parameter vector has {flat.size} elements, "
                              f"expected {cs.column_param_count}")
    out: ParamSet = {}
    pos = 0
    for cl in cs.param_layers():
        entry = {}
        for key, shape in (("w", cl.weight_shape), ("b", cl.bias_shape)):
            n = math.prod(shape)
            entry[key] = flat[pos:pos + n].reshape(shape).copy()
            pos += n
        out[cl.index] = entry
    return out


def params_as_lists(params: ParamSet, cs: ColumnizedSpec) -> list:
    return [params[cl.index][k] for cl in cs.param_layers() for k in ("w", "b")]


def lists_as_params(values: list, cs: ColumnizedSpec) -> ParamSet:
    it = iter(values)
    return {cl.index: {"w": next(it), "b": next(it)} for cl in cs.param_layers()}


# ---------------------------------------------------------------------------
# Logical communication closed forms
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class CommPhase:
    label: str
    total_bytes: int
    total_messages: int
    max_node_bytes: int
    max_node_messages: int


def comm_phases(plan: ParallelPlan, cs: ColumnizedSpec, batch: int,
                wire: int = WIRE_ELEMENT_SIZE) -> list:
    d, m = plan.data_shards, plan.model_columns
    if batch % d:
        raise ValidationError(f"batch size {batch} not divisible by {d} data shards")
    shard = batch // d
    crosses = [cl for cl in cs.col_layers if cl.cross]

    def cross_phase(cl, leg):
        pair = shard * (math.prod(cl.in_shape) // m) * wire
        return CommPhase(f"cross{cl.index}-{leg}", d * m * (m - 1) * pair, d * m * (m - 1),
                         (m - 1) * pair, m - 1)

    phases = [cross_phase(cl, "fwd") for cl in crosses]
    phases += [cross_phase(cl, "bwd") for cl in reversed(crosses)]
    if d > 1:
        col = cs.column_param_count * wire
        phases += [CommPhase(lbl, m * (d - 1) * col, m * (d - 1), (d - 1) * col, d - 1)
                   for lbl in ("grad-reduce", "param-broadcast")]
    return phases


@dataclass(frozen=True)
class CommVolume:
    bytes: int
    messages: int


def comm_volume(plan: ParallelPlan, net: NetworkSpec, batch: int,
                wire: int = WIRE_ELEMENT_SIZE) -> CommVolume:
    phases = comm_phases(plan, plan_columnized(net, plan), batch, wire)
    return CommVolume(sum(p.total_bytes for p in phases), sum(p.total_messages for p in phases))
