"""The three schemes on B200: drop-in ``setup_workers`` / ``hybrid_step`` /
``data_parallel_step`` / ``model_parallel_step`` / ``gather_dense_params`` /
``evaluation_errors`` / ``reference_step`` with the reference's signatures
and error behaviour (`pkg/src/parconv/schemes.py:439-645`).

One call of ``hybrid_step`` = one synchronous update of the whole plan:
contiguous replica shards of the global batch (`schemes.py:516-527`), loss
scale 1/B_global, the column engines of every local replica run layer by
layer with the column exchange at cross layers, gradients are summed over
replicas and every replica applies the identical SGD update (the
reference's reduce-to-root + root SGD + broadcast, with the broadcast
replaced by bit-identical local updates; the ledger still books it).
"""

from __future__ import annotations

import gc
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .engine import ColumnEngine
from .errors import ValidationError
from .fabric import (Fabric, LocalExchange, LocalReducer, NcclExchange, NcclReducer, book_step)
from .netdef import FC, ColumnizedSpec, NetworkSpec, columnize, column_footprint_elements
from .plan import (  # noqa: F401  (re-exported API)
    CommPhase, CommVolume, ParallelPlan, ParamSet, comm_phases, comm_volume, init_dense_params,
    lists_as_params, load_plan, merge_params, pack_tree, params_as_lists, parse_plan, plan_columnized,
    split_params, unpack_tree)


@dataclass
class StepResult:
    loss: float
    ledger_bytes: int = 0
    ledger_messages: int = 0
    params: dict | None = None
    sgd: object = None
    sim_seconds: float | None = None


# ----------------------------------------------------------------------------
# Worker setup
# ----------------------------------------------------------------------------


def setup_workers(fabric: Fabric, plan: ParallelPlan, cs: ColumnizedSpec, dense_params: dict, sgd,
                  meter: bool = True, _velocity: dict | None = None) -> None:
    if fabric.n != plan.workers:
        raise ValidationError(f"plan grid {plan.describe()} needs {plan.workers} workers, "
                              f"fabric has {fabric.n}")
    fabric.torch_device          # the device path: raises ValidationError when no CUDA device is visible
    m = plan.model_columns
    fabric._engines.clear()
    fabric._runner = None
    fabric._plan, fabric._cs = plan, cs
    fabric._hyper = (sgd.learning_rate, sgd.momentum, sgd.weight_decay)
    for wid in range(fabric.n):
        replica, column = divmod(wid, m)
        st = fabric._local[wid]
        dict.clear(st)
        st.update(replica=replica, column=column, hyper=fabric._hyper, holds_velocity=replica == 0)
        if wid in fabric.local_wids:
            # like the reference (schemes.py:486-489) the column velocity starts at
            # zero; reference_step passes its SgdState velocity through _velocity
            vel = split_params(_velocity, cs, column) if _velocity is not None else None
            st.update(host_params=split_params(dense_params, cs, column), host_velocity=vel)
        if meter:
            elems = cs.column_param_count * (2 if replica == 0 else 1)
            st["resident_bytes"] = elems * fabric.device.wire_element_size
            fabric.meter.alloc(wid, st["resident_bytes"])
            fabric.meter_assert(wid)


_COPY_POOL = None


def _parallel_copy(dst: np.ndarray, src: np.ndarray, parts: int = 8) -> None:
    """dst[...] = src in `parts` row slices on a thread pool (numpy releases the GIL
    for large same-dtype copies): a 317 MB float64 batch in a fraction of one
    thread's time."""
    global _COPY_POOL
    n = src.shape[0]
    if n < parts or src.nbytes < (16 << 20):
        np.copyto(dst, src)
        return
    if _COPY_POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _COPY_POOL = ThreadPoolExecutor(max_workers=parts, thread_name_prefix="pc-copy")
    bounds = [(i * n // parts, (i + 1) * n // parts) for i in range(parts)]
    list(_COPY_POOL.map(lambda b: np.copyto(dst[b[0]:b[1]], src[b[0]:b[1]]), bounds))


def _parallel_take(dst: np.ndarray, src: np.ndarray, idx: np.ndarray, parts: int = 8) -> None:
    """dst[...] = src[idx] (rows) in `parts` slices on the copy pool: the host-fed
    trainer's batch gather straight into pinned staging memory."""
    global _COPY_POOL
    n = len(idx)
    if n < parts or dst.nbytes < (16 << 20):
        np.take(src, idx, axis=0, out=dst)
        return
    if _COPY_POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _COPY_POOL = ThreadPoolExecutor(max_workers=parts, thread_name_prefix="pc-copy")
    bounds = [(i * n // parts, (i + 1) * n // parts) for i in range(parts)]
    list(_COPY_POOL.map(lambda b: np.take(src, idx[b[0]:b[1]], axis=0, out=dst[b[0]:b[1]]), bounds))


class _Runner:
    """Engines of this process for one (plan, shard) plus the exchange wiring."""

    def __init__(self, fabric: Fabric, plan: ParallelPlan, cs: ColumnizedSpec, shard: int):
        self.fabric, self.plan, self.cs, self.shard = fabric, plan, cs, shard
        d, m = plan.data_shards, plan.model_columns
        dev = fabric.torch_device
        self.engines = {}
        with torch.cuda.device(dev):
            for wid in fabric.local_wids:
                replica, column = divmod(wid, m)
                old = fabric._engines.get(wid)
                eng = ColumnEngine(cs, wid, replica, column, shard, fabric.prec, dev, fabric._hyper, fabric.cprec)
                eng.dropout_seed = int(getattr(fabric, "dropout_seed", 0))
                if old is not None:
                    eng.p32.copy_(old.p32)
                    eng.v32.copy_(old.v32)
                    eng.step_ctr.copy_(old.step_ctr)
                    if eng.plow is not None:
                        eng.plow.copy_(old.plow)
                else:
                    st = fabric._local[wid]
                    eng.load_params(dict.__getitem__(st, "host_params"), dict.get(st, "host_velocity"))
                self.engines[wid] = eng
        # single-replica plans fuse the weight updates into the gradient kernels (the FC
        # weight gradient's epilogue updates p/v in place, the split-K reductions of the
        # convolutions do the same), so those gradients never reach HBM. Off with
        # fabric.fuse_sgd = False or PC_FUSE_SGD=0 (e.g. to read gradients back).
        fuse = d == 1 and getattr(fabric, "fuse_sgd", os.environ.get("PC_FUSE_SGD", "1") == "1")
        for eng in self.engines.values():
            eng.configure_fused_sgd(fuse)
        fabric._engines.update(self.engines)
        if fabric.dist:
            col_g, rep_g = fabric.groups(d, m)
            self.exchange = NcclExchange(col_g) if m > 1 else None
            self.reducer = NcclReducer(rep_g) if d > 1 else None
        else:
            self.exchange = LocalExchange(dev) if m > 1 else None
            self.reducer = LocalReducer(dev) if d > 1 else None
        self.replicas = {}
        self.columns = {}
        for wid, eng in sorted(self.engines.items()):
            self.replicas.setdefault(eng.replica, []).append(eng)
            self.columns.setdefault(eng.column, []).append(eng)
        self.x_dev = None
        self.y_dev = None
        self.fwd_done = None
        self._fwd_single = True
        split = len(self.replicas) == 1 and os.environ.get("PC_SPLIT_STEP", "1") != "0" and not fabric.dist
        self.copy_stream = torch.cuda.Stream(device=dev) if split else None
        self.loss_stream = torch.cuda.Stream(device=dev) if split else None
        self.loss_host = torch.zeros(2, dtype=torch.float64).pin_memory() if split else None
        self._graphs, self._seen = {}, set()
        self.graph_launches, self.replays = 0, 0
        # single replica, unfused SGD: the FC head's update runs on a side stream as soon
        # as the backward has passed the first FC layer, overlapping the conv backward
        self.head_pos = next((i for i, cl in enumerate(cs.col_layers) if isinstance(cl.layer, FC)), None)
        self.split_sgd = {}
        if d == 1 and self.head_pos is not None and os.environ.get("PC_SGD_OVERLAP", "1") != "0":
            for wid, eng in self.engines.items():
                if not getattr(eng, "fuse_sgd", False) and not eng.has_dropout:
                    tabs = eng.sgd_split_table(self.head_pos)
                    if tabs is not None:
                        self.split_sgd[wid] = tabs
        self.side = torch.cuda.Stream(device=dev) if self.split_sgd else None
        # opt-in (PC_BIAS_SIDE=1), single replica: bias gradients on their own side
        # stream beside the GEMMs (with d > 1 the bucketed all-reduce needs each
        # layer's bias at once). Measured on AlexNet b256: no gain — the reduction
        # competes with the operand-bound GEMMs for L2 bandwidth — so off by default.
        # FC weight gradients + fused updates on a side stream, on a separate SM set
        # (PC_FC_SIDE_CTAS CTAs; 0 = off) beside the data-gradient chain
        self.fc_side = None
        side_ctas = int(os.environ.get("PC_FC_SIDE_CTAS", "0"))
        if fuse and side_ctas > 0:
            sms = torch.cuda.get_device_properties(dev).multi_processor_count
            side_ctas = min(side_ctas, sms - 2) & ~1
            self.fc_side = torch.cuda.Stream(device=dev)
            for eng in self.engines.values():
                if getattr(eng, "fuse_sgd", False):
                    eng.enable_fc_side(self.fc_side, side_ctas, (sms - side_ctas) & ~1,
                                       int(os.environ.get("PC_FC_SIDE_SPAN", "2")))
        # conv weight gradients (+ fused updates) on a side stream beside the data-gradient
        # chain (PC_WGRAD_SIDE=0 off): their persistent kernels fill the SMs the chain's
        # last waves leave idle; needs the prepared data-gradient filters below
        self.wg_side = None
        if fuse and os.environ.get("PC_WGRAD_SIDE", "1") != "0" and os.environ.get("PC_WT_PREP", "1") != "0":
            self.wg_side = torch.cuda.Stream(device=dev)
            fc_too = os.environ.get("PC_FC_WG_SIDE", "1") != "0" and self.fc_side is None
            for eng in self.engines.values():
                if getattr(eng, "fuse_sgd", False):
                    eng.enable_wgrad_side(self.wg_side)
                    if fc_too:   # FC weight gradients + updates on the same stream (PC_FC_WG_CTAS: grid cap)
                        eng.enable_fc_side(self.wg_side, int(os.environ.get("PC_FC_WG_CTAS", "0")), 0, 0)
        # conv filters in the data-gradient layout, prepared on a side stream at the
        # start of every step (beside the forward) instead of inside each backward
        self.wt_side = None
        if os.environ.get("PC_WT_PREP", "1") != "0":
            if any([eng.enable_dgrad_weights() for eng in self.engines.values()]):
                self.wt_side = torch.cuda.Stream(device=dev)
        self.bias_side = None
        if d == 1 and os.environ.get("PC_BIAS_SIDE", "0") != "0":
            self.bias_side = torch.cuda.Stream(device=dev)
            ctas = torch.cuda.get_device_properties(dev).multi_processor_count * \
                int(os.environ.get("PC_BIAS_CTAS_PER_SM", "2"))
            for eng in self.engines.values():
                eng.enable_bias_side(self.bias_side, ctas)
        # background CTAs per SM for the side-stream update: few enough that each
        # backward GEMM still finds room for its one persistent CTA per SM
        self.sgd_bg_ctas = int(os.environ.get("PC_SGD_BG_CTAS", "2"))

    def upload(self, batch_x, batch_y):
        """Host -> device copy of the global batch (float32 NCHW, int32 labels).
        numpy input is staged through pinned memory; a pinned float32 CPU
        tensor is copied directly; a CUDA tensor is used in place."""
        dev = self.fabric.torch_device
        # a bf16 host batch (an input pipeline that stores images in bf16) is copied as
        # bf16 when every engine's input layer is the explicit-im2col GEMM, which rounds
        # to bf16 first anyway (identical results, half the host->device bytes)
        keep_bf16 = isinstance(batch_x, torch.Tensor) and batch_x.dtype == torch.bfloat16 and \
            all((e.col_kp or e.s2d) and e.prec == L.PC_BF16 for e in self.engines.values())
        # a float64 numpy batch (what a parconv caller passes: Dataset.images) for a
        # space-to-depth input layer travels as raw float64 — a multi-threaded copy into
        # pinned memory, no host-side conversion pass — and the input kernel rounds it
        # to float32 on the device (the value the float32 path uploads)
        raw64 = (isinstance(batch_x, np.ndarray) and batch_x.dtype == np.float64 or
                 isinstance(batch_x, torch.Tensor) and not batch_x.is_cuda and batch_x.dtype == torch.float64) and \
            all(e.s2d and e.in_c == 3 for e in self.engines.values())
        pinned64 = raw64 and isinstance(batch_x, torch.Tensor) and batch_x.is_pinned() and batch_x.is_contiguous()
        xdt = torch.bfloat16 if keep_bf16 else torch.float64 if raw64 else torch.float32
        if isinstance(batch_x, torch.Tensor) and batch_x.is_cuda and batch_x.dtype == xdt:
            xs = batch_x.contiguous()
        else:
            xs = None
            if raw64:
                x = None
            elif isinstance(batch_x, torch.Tensor):
                x = batch_x if batch_x.dtype == xdt else batch_x.to(xdt)
            else:
                x = torch.as_tensor(np.ascontiguousarray(batch_x, dtype=np.float32))
        y = torch.as_tensor(np.asarray(batch_y, dtype=np.int32)) if not isinstance(batch_y, torch.Tensor) \
            else batch_y.to(torch.int32)
        shape = tuple(xs.shape if xs is not None else batch_x.shape if raw64 else x.shape)
        if self.x_dev is None or tuple(self.x_dev.shape) != shape or self.x_dev.dtype != xdt:
            self.x_host = torch.empty(shape, dtype=xdt).pin_memory()
            self.y_host = torch.empty(tuple(y.shape), dtype=torch.int32).pin_memory()
            self.x_dev = torch.empty(shape, dtype=xdt, device=dev)
            self.y_dev = torch.empty(tuple(y.shape), dtype=torch.int32, device=dev)
        # host -> device on a copy stream that waits only until the previous step's
        # forward has consumed the input buffers: the upload overlaps that step's backward
        cs = self.copy_stream if self.copy_stream is not None else torch.cuda.current_stream()
        if self.copy_stream is not None:
            if self.fwd_done is None or (xs is not None) or y.is_cuda:
                # a device-resident source (e.g. the trainer's on-device batch gather) is
                # produced on the current stream, behind the previous step's backward:
                # the copy must wait for that producer, not only for the forward
                cs.wait_stream(torch.cuda.current_stream())
            else:
                cs.wait_event(self.fwd_done)
            if xs is not None:
                xs.record_stream(cs)
            if y.is_cuda:
                y.record_stream(cs)
        if raw64 and not pinned64:
            _parallel_copy(self.x_host.numpy(), batch_x.numpy() if isinstance(batch_x, torch.Tensor) else batch_x)
        with torch.cuda.stream(cs):
            if xs is not None:
                self.x_dev.copy_(xs)
            elif pinned64:
                self.x_dev.copy_(batch_x, non_blocking=True)
            elif raw64:
                self.x_dev.copy_(self.x_host, non_blocking=True)
            elif x.is_pinned():
                self.x_dev.copy_(x, non_blocking=True)
            else:
                self.x_host.copy_(x)
                self.x_dev.copy_(self.x_host, non_blocking=True)
            if y.is_cuda:
                self.y_dev.copy_(y)
            else:
                self.y_host.copy_(y)
                self.y_dev.copy_(self.y_host, non_blocking=True)

    def program(self, loss_scale: float, eager: bool = False):
        """The device step (no host synchronisation inside).

        The first call for a given (loss scale, batch buffer) runs eagerly (it
        is a real update, and it warms every kernel's launch attributes); the
        second captures the same launch sequence into a CUDA graph, and every
        call from then on replays it, so the ~60 launches of a step cost one
        host call. Under torchrun the NCCL collectives are captured too
        (``PC_GRAPH_DIST=0``: eager); a failed capture falls back to eager launches."""
        self.fwd_done = None
        if self.copy_stream is not None:   # this step's batch upload (pipelined, see upload())
            torch.cuda.current_stream().wait_stream(self.copy_stream)
        if eager or not self._graph_enabled():
            self._launch(loss_scale, "fwd")
            self._mark_fwd_done()
            return self._launch(loss_scale, "bwd")
        key = (float(loss_scale), self.x_dev.data_ptr(), self.x_dev.dtype)
        g = self._graphs.get(key)
        if g is None:
            if key not in self._seen:
                self._seen.add(key)
                self._launch(loss_scale, "fwd")
                self._mark_fwd_done()
                return self._launch(loss_scale, "bwd")
            # free garbage first: a collection during capture can release blocks that
            # other streams used, and the allocator's event calls would invalidate it
            gc.collect()
            torch.cuda.synchronize(self.fabric.torch_device)
            l0 = L.lib().dll.pc_launch_count()
            # two graphs (forward + loss, backward + update) when the plan allows it, so the
            # loss can be read back while the backward runs
            parts = ("fwd", "bwd") if self._split_ok() else ("all",)
            g = []
            try:
                for part in parts:
                    gp = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(gp, capture_error_mode="thread_local"):
                        self._launch(loss_scale, part)
                    g.append(gp)
            except RuntimeError as err:
                # a capture records and executes nothing: this step (and every later one)
                # runs eagerly; under torchrun the collectives stay in the same order
                # whether a rank replays a graph or launches eagerly
                import warnings
                warnings.warn(f"CUDA-graph capture of the step failed ({err}); running eagerly")
                self._graph_broken = True
                torch.cuda.synchronize(self.fabric.torch_device)
                if self.fabric.dist and hasattr(self.reducer, "works"):
                    self.reducer.works = []
                self._launch(loss_scale, "fwd")
                self._mark_fwd_done()
                return self._launch(loss_scale, "bwd")
            self.graph_launches = int(L.lib().dll.pc_launch_count() - l0)
            self._graphs[key] = g
        g[0].replay()
        if len(g) > 1:
            self._mark_fwd_done()
            g[1].replay()
        self.replays += 1

    def _mark_fwd_done(self):
        """Event after the forward (loss, label flag and the input buffers consumed)."""
        if self._split_ok():
            self.fwd_done = torch.cuda.Event()
            self.fwd_done.record()

    def _graph_enabled(self) -> bool:
        """CUDA-graph replay: single process always; under torchrun too (the NCCL
        collectives are captured with the kernels; PC_GRAPH_DIST=0 keeps them eager)."""
        if os.environ.get("PC_GRAPH", "1") == "0" or getattr(self, "_graph_broken", False):
            return False
        return not self.fabric.dist or os.environ.get("PC_GRAPH_DIST", "1") == "1"

    def _split_ok(self) -> bool:
        """One local replica: the forward (and so the loss) is complete before any
        backward work, so the step can be two graphs with the loss read in between."""
        return len(self.replicas) == 1 and os.environ.get("PC_SPLIT_STEP", "1") != "0"

    def _launch(self, loss_scale: float, part: str = "all"):
        if part in ("all", "fwd"):
            self._launch_fwd(loss_scale)
        if part in ("all", "bwd"):
            self._launch_bwd()

    def _launch_fwd(self, loss_scale: float):
        shard = self.shard
        for eng in self.engines.values():
            lo = eng.replica * shard
            eng.load_batch(self.x_dev[lo:lo + shard], self.y_dev[lo:lo + shard])
        n = len(self.cs.col_layers)
        if self.wt_side is not None:   # fork: data-gradient filters, joined before the backward
            self.wt_side.wait_stream(torch.cuda.current_stream())
            for eng in self.engines.values():
                eng.prepare_dgrad_weights(self.wt_side.cuda_stream)
                eng.wt_ready = True
        single = len(self.replicas) == 1
        for engines in self.replicas.values():
            for i in range(n):
                if self.cs.col_layers[i].cross and self.exchange is not None:
                    self.exchange.all_gather(i, engines)
                for e in engines:
                    e.forward(i, loss_scale)
            if self.wt_side is not None:
                torch.cuda.current_stream().wait_stream(self.wt_side)
            if not single:   # several local replicas: each replica's backward follows its forward
                self._backward_replica(engines)
        self._fwd_single = single

    def _launch_bwd(self):
        if self._fwd_single:
            for engines in self.replicas.values():
                self._backward_replica(engines)
        self._finish()

    def _backward_replica(self, engines):
        n = len(self.cs.col_layers)
        overlap = self.reducer is not None and hasattr(self.reducer, "layer_done")
        for i in range(n - 1, -1, -1):
            for e in engines:
                e.backward(i)
                if overlap and e.layers[i].w_off >= 0:
                    self.reducer.layer_done(e, *e.param_region(i))
                if i == self.head_pos and e.wid in self.split_sgd:   # fork: head update on the side stream
                    self.side.wait_stream(torch.cuda.current_stream())
                    if e.bias_side is not None:   # the head's bias gradients
                        self.side.wait_stream(e.bias_side)
                    with torch.cuda.stream(self.side):
                        e.sgd_table(self.split_sgd[e.wid][0], ctas_per_sm=self.sgd_bg_ctas)
            if self.cs.col_layers[i].cross and self.exchange is not None and i > 0:
                self.exchange.reduce_scatter(i, engines)

    def _finish(self):
        if self.reducer is not None:
            self.reducer.reduce(self.columns)
        for eng in self.engines.values():
            eng.join_side()
        for eng in self.engines.values():
            if eng.wid in self.split_sgd:
                eng.sgd_table(self.split_sgd[eng.wid][1])
            else:
                eng.sgd()
        if self.side is not None:   # join
            torch.cuda.current_stream().wait_stream(self.side)

    def loss(self) -> float:
        """Sum over replicas of column 0's loss, accumulated on the host in ascending
        replica order like the reference (`schemes.py:562-564`); raises on bad labels.
        With a split step the read waits only for the forward (fwd_done), on its own
        stream: the backward keeps running while the caller gets the loss."""
        parts = [e.loss.reshape(()) for e in sorted(self.engines.values(), key=lambda e: e.replica)
                 if e.column == 0]

        def flag():
            return torch.stack([e.bad_label.reshape(()) for e in self.engines.values()]).sum().double()

        if getattr(self, "fwd_done", None) is not None and not self.fabric.dist:
            # after the forward only, on the loss stream: the losses (f64) and label flags
            # (i32) go straight to pinned host memory by device-to-host copies (no kernels)
            ls = self.loss_stream
            ls.wait_event(self.fwd_done)
            engines = list(self.engines.values())
            if self.loss_host.numel() != len(parts) or getattr(self, "flag_host", None) is None:
                self.loss_host = torch.zeros(len(parts), dtype=torch.float64).pin_memory()
                self.flag_host = torch.zeros(len(engines), dtype=torch.int32).pin_memory()
            lib = L.lib()
            for i, t in enumerate(parts):
                lib.call("pc_copy_async", self.loss_host.data_ptr() + 8 * i, t.data_ptr(), 8, ls.cuda_stream)
            for j, e in enumerate(engines):
                lib.call("pc_copy_async", self.flag_host.data_ptr() + 4 * j, e.bad_label.data_ptr(), 4, ls.cuda_stream)
            ls.synchronize()
            return self._check_loss(np.append(self.loss_host.numpy(), float(self.flag_host.numpy().sum())))
        if self.fabric.dist:
            m = self.plan.model_columns
            mine = parts[0] if parts else torch.zeros((), dtype=torch.float64, device=self.fabric.torch_device)
            # every rank contributes its slot: rank r of column 0 fills entry r // m
            buf = torch.zeros(self.plan.data_shards + 1, dtype=torch.float64, device=self.fabric.torch_device)
            if parts:
                buf[self.fabric.rank // m] = mine
            buf[-1] = flag()
            torch.distributed.all_reduce(buf)
            return self._check_loss(buf.cpu().numpy())
        return self._check_loss(torch.stack(parts + [flag()]).cpu().numpy())

    def _check_loss(self, host) -> float:
        """host = [replica losses (ascending replica), label-error count]."""
        if host[-1] != 0:
            raise ValidationError(f"labels must lie in [0, {self.cs.base.classes})")
        total = 0.0
        for v in host[:-1]:
            total += float(v)
        return total


def _runner(fabric: Fabric, plan: ParallelPlan, cs: ColumnizedSpec, shard: int):
    r = getattr(fabric, "_runner", None)
    if r is None or r.shard != shard or r.cs is not cs:
        if r is not None and hasattr(r, "close"):
            r.close()
        if fabric.multi:
            from .multidev import PeerRunner
            r = PeerRunner(fabric, plan, cs, shard)
        else:
            r = _Runner(fabric, plan, cs, shard)
        fabric._runner = r
    return r


def _meter_step(fabric: Fabric, cs: ColumnizedSpec, shard: int) -> None:
    _, acts = column_footprint_elements(cs, shard)
    nbytes = acts * fabric.device.wire_element_size
    for wid in range(fabric.n):
        fabric.meter.alloc(wid, nbytes)
        fabric.meter_assert(wid)
    for wid in range(fabric.n):
        fabric.meter.free(wid, nbytes)


def hybrid_step(fabric: Fabric, plan: ParallelPlan, cs: ColumnizedSpec, batch_x, batch_y,
                meter: bool = True) -> StepResult:
    """One synchronous update of the plan (`schemes.py:500-569`).

    Asynchronous contract: the loss is read back as soon as the forward is done
    (single replica per process), so the call returns while the backward and the
    update still run on the device; the next call (or any read of the
    parameters) is ordered after them. A device fault in the backward therefore
    surfaces at the next call. ``fabric.sync_step = True`` (or PC_SYNC_STEP=1)
    synchronises before returning."""
    d, m = plan.data_shards, plan.model_columns
    if fabric.n != plan.workers:
        raise ValidationError(f"plan grid {plan.describe()} needs {plan.workers} workers, "
                              f"fabric has {fabric.n}")
    if cs.columns != m:
        raise ValidationError("columnized spec does not match the plan's column count")
    b = int(np.shape(batch_x)[0])
    if b % d != 0:
        raise ValidationError(f"batch size {b} not divisible by {d} data shards")
    labels = batch_y.cpu().numpy().astype(np.int64) if isinstance(batch_y, torch.Tensor) \
        else np.asarray(batch_y, dtype=np.int64)
    k = cs.base.classes
    if labels.size and (labels.min() < 0 or labels.max() >= k):
        raise ValidationError(f"labels must lie in [0, {k})")
    if getattr(fabric, "_hyper", None) is None:
        raise ValidationError("setup_workers must run before hybrid_step")
    shard = b // d
    if shard == 0:
        raise ValidationError("hybrid_step needs a non-empty batch")
    before_b, before_m = fabric.ledger.total_bytes, fabric.ledger.total_messages
    if meter:
        _meter_step(fabric, cs, shard)
    run = _runner(fabric, plan, cs, shard)
    if fabric.multi:      # one host thread per worker, each on its own GPU / stream
        run.upload(batch_x, labels)
        run.step(1.0 / b)
        loss = run.loss()
    else:
        with torch.cuda.device(fabric.torch_device):
            run.upload(batch_x, labels)
            run.program(1.0 / b)
            loss = run.loss()
    if getattr(fabric, "sync_step", os.environ.get("PC_SYNC_STEP", "0") == "1"):
        for dev in {fabric.device_of(w) for w in fabric.local_wids}:
            torch.cuda.synchronize(dev)
    book_step(fabric, plan, cs, shard)
    return StepResult(loss=loss, ledger_bytes=fabric.ledger.total_bytes - before_b,
                      ledger_messages=fabric.ledger.total_messages - before_m)


def data_parallel_step(fabric, plan, cs, batch_x, batch_y, meter: bool = True) -> StepResult:
    if plan.model_columns != 1:
        raise ValidationError("data_parallel_step requires a plan with model_columns == 1")
    return hybrid_step(fabric, plan, cs, batch_x, batch_y, meter=meter)


def model_parallel_step(fabric, plan, cs, batch_x, batch_y, meter: bool = True) -> StepResult:
    if plan.data_shards != 1:
        raise ValidationError("model_parallel_step requires a plan with data_shards == 1")
    return hybrid_step(fabric, plan, cs, batch_x, batch_y, meter=meter)


def column_params(fabric: Fabric, wid: int) -> dict:
    """Reference-layout parameters of a hosted worker (device -> host)."""
    eng = fabric._engines.get(wid)
    if eng is not None:
        return eng.params_host()
    return dict.__getitem__(fabric._local[wid], "host_params")


def gather_dense_params(fabric: Fabric, plan: ParallelPlan, cs: ColumnizedSpec) -> dict:
    m = plan.model_columns
    if fabric.dist:
        cols = []
        for j in range(m):
            obj = [column_params(fabric, j) if fabric.rank == j else None]
            torch.distributed.broadcast_object_list(obj, src=j)
            cols.append(obj[0])
    else:
        cols = [column_params(fabric, plan.worker_of(0, j)) for j in range(m)]
    return merge_params(cols, cs)


def _eval_engines(fabric: Fabric, cs: ColumnizedSpec, b: int, wids: list) -> list:
    """Forward-only engines of replica 0's hosted columns for evaluation batch b,
    cached on the fabric (train() evaluates shard after shard of the test split:
    one allocation per batch size, not per call); parameters are refreshed from
    the training engines (or the host copy before the first step) at every call."""
    cache = fabric.__dict__.setdefault("_eval_cache", {})
    key = (id(cs), b, tuple(wids))
    engines = cache.get(key)
    if engines is None:
        if len(cache) >= 2:          # full shards + one ragged tail
            cache.pop(next(iter(cache)))
        engines = []
        for j in wids:
            eng = ColumnEngine(cs, j, 0, j, b, fabric.prec, fabric.device_of(j), fabric._hyper, fabric.cprec)
            eng.training = False     # dropout is the identity at evaluation
            engines.append(eng)
        cache[key] = engines
    for eng in engines:
        src = fabric._engines.get(eng.wid)
        if src is not None:
            eng.p32.copy_(src.p32)
            if eng.plow is not None:
                eng.plow.copy_(src.plow)
            eng._host_src = None
        else:
            hp = dict.__getitem__(fabric._local[eng.wid], "host_params")
            if getattr(eng, "_host_src", None) is not hp:    # setup_workers' host copy, loaded once
                eng.load_params(hp)
                eng._host_src = hp
    return engines


def _book_eval(fabric: Fabric, plan: ParallelPlan, cs: ColumnizedSpec, b: int) -> None:
    """The reference's evaluation ledgers replica 0's cross-layer forward exchange
    like any other message (`schemes.py:600-645`, FabricExchange.cross_forward)."""
    m, wire = plan.model_columns, fabric.device.wire_element_size
    for cl in cs.col_layers:
        if not cl.cross:
            continue
        nbytes = b * (math.prod(cl.in_shape) // m) * wire
        for j in range(m):
            for k in range(m):
                if k != j:
                    fabric.ledger.record(j, k, nbytes)


def evaluation_errors(fabric: Fabric, plan: ParallelPlan, cs: ColumnizedSpec, x, labels) -> int:
    """Misclassifications of replica 0's columns (forward only; argmax ties ->
    lowest class), `schemes.py:600-645`. Under torchrun the ranks of replica 0
    run their column's forward with the column group's all-gather; every rank
    returns rank 0's count."""
    labels = np.asarray(labels, dtype=np.int64)
    b = int(np.shape(x)[0])
    if b == 0:
        return 0
    d, m = plan.data_shards, plan.model_columns
    if fabric.n != plan.workers:
        raise ValidationError(f"plan grid {plan.describe()} needs {plan.workers} workers, "
                              f"fabric has {fabric.n}")
    if getattr(fabric, "_hyper", None) is None:
        raise ValidationError("setup_workers must run before evaluation_errors")
    _book_eval(fabric, plan, cs, b)
    dev = fabric.torch_device
    wids = [w for w in fabric.local_wids if w < m]      # replica 0 = workers 0 .. m-1
    if fabric.dist:
        col_g, _ = fabric.groups(d, m)                  # collective: every rank creates the groups
        ex = NcclExchange(col_g) if m > 1 else None
    else:
        ex = LocalExchange(dev) if m > 1 else None
    count = -1
    if fabric.multi:
        from .multidev import evaluate
        engines = _eval_engines(fabric, cs, b, wids)
        if isinstance(x, torch.Tensor) and x.is_cuda:
            x = x.float().cpu().numpy()
        return evaluate(fabric, plan, cs, x, labels, {e.wid: e for e in engines})
    if wids:
        with torch.cuda.device(dev):
            engines = _eval_engines(fabric, cs, b, wids)
            if isinstance(x, torch.Tensor) and x.is_cuda:
                # a device-resident test split (train() with device_data): used in place
                xd = x.to(dev).contiguous()
                if xd.dtype not in (torch.float32, torch.bfloat16) or \
                        (xd.dtype == torch.bfloat16 and not all(e.s2d and e.prec == L.PC_BF16 for e in engines)):
                    xd = xd.float()
            elif isinstance(x, np.ndarray) and x.dtype == np.float64 and all(e.s2d and e.in_c == 3 for e in engines):
                # float64 test images travel raw (threaded copy into cached pinned memory); the
                # input kernel rounds them on the device
                pin = fabric.__dict__.get("_eval_pinned")
                if pin is None or tuple(pin.shape) != tuple(x.shape):
                    pin = torch.empty(tuple(x.shape), dtype=torch.float64).pin_memory()
                    fabric._eval_pinned = pin
                _parallel_copy(pin.numpy(), np.ascontiguousarray(x))
                xd = pin.to(dev, non_blocking=True)
            else:
                xd = torch.as_tensor(np.ascontiguousarray(x, dtype=np.float32)).to(dev)
            yd = torch.zeros(b, dtype=torch.int32, device=dev)
            for e in engines:
                e.load_batch(xd, yd)
            n = len(cs.col_layers)
            for i in range(n - 1):      # stop before the softmax: logits = head output
                if cs.col_layers[i].cross and ex is not None:
                    ex.all_gather(i, engines)
                for e in engines:
                    e.forward(i, 1.0)
            if engines[0].wid == 0:
                head = engines[0].layers[n - 2]
                logits = head.out[: b * cs.base.classes].float().reshape(b, cs.base.classes)
                pred = torch.argmax(logits, dim=1).cpu().numpy()   # first maximum, like np.argmax
                count = int(np.count_nonzero(pred != labels))
    if fabric.dist:
        t = torch.tensor([count], dtype=torch.int64, device=dev)
        torch.distributed.broadcast(t, src=0)
        count = int(t.item())
    return count


def reference_step(net: NetworkSpec, params: dict, batch, sgd, precision: str = "fp32") -> StepResult:
    """Dense single-worker step on the device (the reference's oracle entry,
    `schemes.py:439-458`); returns fresh dense params and SgdState."""
    from .kernels import SgdState
    from .fabric import spawn
    x, labels = batch
    if np.shape(x)[0] < 1:
        raise ValidationError("reference_step needs a non-empty batch")
    cs = columnize(net, 1)
    fab = spawn(1, precision=precision)
    vel = lists_as_params(list(sgd.velocity), cs) if sgd.velocity else None
    setup_workers(fab, ParallelPlan(1, 1), cs, params, sgd, meter=False, _velocity=vel)
    res = hybrid_step(fab, ParallelPlan(1, 1), cs, x, labels, meter=False)
    eng = fab._engines[0]
    new_sgd = SgdState(sgd.learning_rate, sgd.momentum, sgd.weight_decay,
                       params_as_lists(eng.velocity_host(), cs))
    return StepResult(loss=res.loss, params=eng.params_host(), sgd=new_sgd)
