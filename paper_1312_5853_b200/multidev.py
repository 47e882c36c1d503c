"""Single-process multi-GPU fabric: ``spawn(n)`` over the visible GPUs.

The reference runs every worker of a plan as a Python thread of one process
and moves data through an in-process message fabric (`pkg/src/parconv/
fabric.py:280-339`); ``hybrid_step(fabric, ...)`` is one call that drives all
of them. This module keeps exactly that execution model on B200s — SURVEY
§8 b3's recommended alternative to torchrun — with one host thread per worker
(its own CUDA stream on its own GPU) and the fabric's messages replaced by
device-side transfers over NVLink:

* cross-layer forward (`schemes.py:296-305`): every column copies the other
  columns' slices straight from their memory (peer copies) into its
  channel-blocked concatenation buffer;
* cross-layer backward (`schemes.py:307-318`): column k sums piece k of every
  column's input gradient, ascending column order, reading peer memory in
  one kernel (pc_sum_buffers over peer pointers);
* data-parallel leg (reduce-to-root + broadcast, `schemes.py:540-558`): the
  replicas of a column split the flat gradient into d slices; replica r sums
  slice r over all replicas in ascending replica order (reduce-scatter), then
  copies the other slices from their owners (all-gather) — the same per-element
  ascending sum as the one-device path, so every plan is bit-identical to its
  single-GPU run; every replica then applies the identical SGD update.

Ordering between workers uses CUDA events (a worker's stream waits for the
producer's event before it reads peer memory); a host barrier per exchange
point guarantees the producer's event is recorded before anyone waits on it.
At the start of every step each stream waits for every worker's end-of-step
event of the previous step, so no buffer is rewritten while a peer may still
read it. The lowest failing worker's exception is re-raised after all threads
unwind (`fabric.py:335-338`). ``devices=[0, 0, ...]`` runs the same machinery
with every worker on one GPU (separate streams): that is how it is tested on a
one-GPU box, bit-identical to the single-stream path.
"""

from __future__ import annotations

import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

from . import _lib as L
from .engine import ColumnEngine
from .errors import ValidationError

ALIGN = 32   # elements: slice boundaries of the replica reduction (128-byte aligned in fp32)


def _ptrs(tensors, device):
    return torch.tensor([t.data_ptr() for t in tensors], dtype=torch.int64, device=device)


class PeerRunner:
    """Engines of every worker of one (plan, shard) on their own GPUs/streams."""

    def __init__(self, fabric, plan, cs, shard: int, engines: dict | None = None, train: bool = True):
        self.fabric, self.plan, self.cs, self.shard, self.train = fabric, plan, cs, shard, train
        d, m = plan.data_shards, plan.model_columns
        self.d, self.m = d, m
        self.wids = sorted(engines) if engines is not None else list(range(fabric.n))
        self.engines = {}
        self.streams = {}
        for wid in self.wids:
            dev = fabric.device_of(wid)
            with torch.cuda.device(dev):
                self.streams[wid] = torch.cuda.Stream(device=dev)
                if engines is not None:
                    self.engines[wid] = engines[wid]
                    continue
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
                # d == 1: no reduction between backward and update -> fuse the update into
                # the weight-gradient kernels (bf16), as on one device
                eng.configure_fused_sgd(d == 1 and getattr(fabric, "fuse_sgd", True))
                self.engines[wid] = eng
        if engines is None:
            fabric._engines.update(self.engines)
        self._peer_setup()
        self.pool = ThreadPoolExecutor(max_workers=len(self.wids), thread_name_prefix="pc-worker")
        self.end_events = {}
        self.xbuf, self.ybuf = {}, {}
        self._ptr_cache = {}
        self.slices = self._slices()
        self.steps = 0

    # ----------------------------------------------------------------- setup
    def _peer_setup(self):
        devs = sorted({self.fabric.device_of(w).index for w in self.wids})
        lib = L.lib()
        for a in devs:
            with torch.cuda.device(a):
                for b in devs:
                    if a != b:
                        lib.call("pc_enable_peer_access", b)

    def _slices(self):
        """[lo, hi) of the flat gradient owned by each replica in the reduction."""
        if self.d <= 1 or not self.train:
            return None
        n = next(iter(self.engines.values())).n_flat
        per = -(-n // self.d)
        per = -(-per // ALIGN) * ALIGN
        return [(min(n, r * per), min(n, (r + 1) * per)) for r in range(self.d)]

    def replica_columns(self, replica: int):
        return [self.engines[replica * self.m + j] for j in range(self.m)]

    def column_replicas(self, column: int):
        return [self.engines[r * self.m + column] for r in range(self.d)]

    # ----------------------------------------------------------------- batch
    def upload(self, batch_x, labels: np.ndarray):
        """Each worker copies its replica's rows of the global batch (pinned host
        staging, one host->device copy per worker on its own stream)."""
        if isinstance(batch_x, torch.Tensor) and batch_x.is_cuda:
            host = batch_x.float().cpu()
        elif isinstance(batch_x, torch.Tensor):
            host = batch_x.float()
        else:
            host = torch.as_tensor(np.ascontiguousarray(batch_x, dtype=np.float32))
        if not host.is_pinned():
            host = host.pin_memory()
        y = torch.as_tensor(np.asarray(labels, dtype=np.int32)).pin_memory()
        self._host = (host, y)            # alive until the copies are done (synchronised per step)
        for wid, e in self.engines.items():
            lo = e.replica * self.shard
            xs, ys = host[lo:lo + self.shard], y[lo:lo + self.shard]
            dev = e.device
            if wid not in self.xbuf or tuple(self.xbuf[wid].shape) != tuple(xs.shape):
                self.xbuf[wid] = torch.empty(tuple(xs.shape), dtype=torch.float32, device=dev)
                self.ybuf[wid] = torch.empty(tuple(ys.shape), dtype=torch.int32, device=dev)
            s = self.streams[wid]
            for ev in self.end_events.values():
                s.wait_event(ev)
            with torch.cuda.device(dev), torch.cuda.stream(s):
                self.xbuf[wid].copy_(xs, non_blocking=True)
                self.ybuf[wid].copy_(ys, non_blocking=True)

    # ----------------------------------------------------------------- step
    def step(self, loss_scale: float):
        barrier = threading.Barrier(len(self.wids))
        shared = {"fwd": {}, "bwd": {}, "grad": {}, "rs": {}}
        futs = {wid: self.pool.submit(self._worker, wid, loss_scale, barrier, shared) for wid in self.wids}
        errors = {}
        for wid, f in futs.items():
            try:
                f.result()
            except threading.BrokenBarrierError:
                pass
            except BaseException as err:   # noqa: BLE001 (re-raised below)
                errors[wid] = err
        if errors:
            raise errors[min(errors)]
        self.steps += 1

    def _event(self, wid):
        ev = torch.cuda.Event()
        ev.record(self.streams[wid])
        return ev

    def _sync(self, wid, table, key, barrier):
        """Publish this worker's event under ``key`` and wait until every worker has."""
        table.setdefault(key, {})[wid] = self._event(wid)
        barrier.wait()
        return table[key]

    def _worker(self, wid: int, loss_scale: float, barrier, shared):
        e = self.engines[wid]
        s = self.streams[wid]
        try:
            with torch.cuda.device(e.device), torch.cuda.stream(s):
                self._program(wid, e, s, loss_scale, barrier, shared)
        except BaseException:
            barrier.abort()
            raise

    def _program(self, wid, e, s, loss_scale, barrier, shared):
        lib = L.lib()
        cs, m = self.cs, self.m
        n = len(cs.col_layers)
        last = n if self.train else n - 1          # evaluation stops before the softmax
        e.load_batch(self.xbuf[wid], self.ybuf[wid])
        for i in range(last):
            cl = cs.col_layers[i]
            if cl.cross and m > 1:
                evs = self._sync(wid, shared["fwd"], i, barrier)
                st = e.layers[i]
                per = st.rs.numel()
                for k, src in enumerate(self.replica_columns(e.replica)):
                    if src is not e:
                        s.wait_event(evs[src.wid])
                    out = src.layers[i - 1].out
                    lib.call("pc_copy_async", st.inp[k * per:].data_ptr(), out.data_ptr(),
                             per * out.element_size(), s.cuda_stream)
            e.forward(i, loss_scale)
        if not self.train:
            self.end_events[wid] = self._event(wid)
            return
        for i in range(n - 1, -1, -1):
            e.backward(i)
            cl = cs.col_layers[i]
            if cl.cross and m > 1 and i > 0:
                evs = self._sync(wid, shared["bwd"], i, barrier)
                cols = self.replica_columns(e.replica)
                for src in cols:
                    if src is not e:
                        s.wait_event(evs[src.wid])
                st = e.layers[i]
                per = st.rs.numel()
                key = ("rs", wid, i)
                if key not in self._ptr_cache:
                    self._ptr_cache[key] = _ptrs([c.layers[i].gin[e.column * per:(e.column + 1) * per]
                                                  for c in cols], e.device)
                lib.call("pc_sum_buffers", m, per, self._ptr_cache[key].data_ptr(), st.rs.data_ptr(), e.prec,
                         s.cuda_stream)
        if self.d > 1:
            reps = self.column_replicas(e.column)
            evs = self._sync(wid, shared["grad"], e.column, barrier)
            for src in reps:
                if src is not e:
                    s.wait_event(evs[src.wid])
            lo, hi = self.slices[e.replica]
            if hi > lo:   # reduce-scatter: slice r = ascending sum over the replicas (peer reads)
                key = ("dp", wid)
                if key not in self._ptr_cache:
                    self._ptr_cache[key] = _ptrs([r.g32[lo:hi] for r in reps], e.device)
                lib.call("pc_sum_buffers", self.d, hi - lo, self._ptr_cache[key].data_ptr(), e.g32[lo:].data_ptr(),
                         L.PC_FP32, s.cuda_stream)
            evs = self._sync(wid, shared["rs"], e.column, barrier)
            for src in reps:           # all-gather: the other slices from their owners
                if src is e:
                    continue
                s.wait_event(evs[src.wid])
                olo, ohi = self.slices[src.replica]
                if ohi > olo:
                    lib.call("pc_copy_async", e.g32[olo:].data_ptr(), src.g32[olo:].data_ptr(), (ohi - olo) * 4,
                             s.cuda_stream)
        e.join_side()
        e.sgd()
        self.end_events[wid] = self._event(wid)

    # ----------------------------------------------------------------- results
    def loss(self) -> float:
        """Sum over replicas of column 0's loss (the reference's StepResult.loss);
        raises ValidationError when a label was out of range."""
        total, bad = 0.0, 0
        for e in self.engines.values():
            self.streams[e.wid].synchronize()
        for e in sorted(self.engines.values(), key=lambda e: e.replica):   # ascending, schemes.py:562-564
            if e.column == 0:
                total += float(e.loss.item())
            bad += int(e.bad_label.item())
        if bad:
            raise ValidationError(f"labels must lie in [0, {self.cs.base.classes})")
        return total

    def close(self):
        self.pool.shutdown(wait=True)


def evaluate(fabric, plan, cs, x, labels, engines: dict) -> int:
    """Forward-only pass of replica 0's columns (``engines``: wid -> engine, one per
    column) on their GPUs with the peer exchange; returns the misclassifications."""
    b = int(np.shape(x)[0])
    run = PeerRunner(fabric, type(plan)(1, plan.model_columns, plan.cross_layers), cs, b, engines=engines,
                     train=False)
    try:
        run.upload(x, np.zeros(b, dtype=np.int64))
        run.step(1.0)
        for wid in run.wids:
            run.streams[wid].synchronize()
        n = len(cs.col_layers)
        head = engines[0].layers[n - 2]
        logits = head.out[: b * cs.base.classes].float().reshape(b, cs.base.classes)
        pred = torch.argmax(logits, dim=1).cpu().numpy()
        return int(np.count_nonzero(pred != np.asarray(labels, dtype=np.int64)))
    finally:
        run.close()
