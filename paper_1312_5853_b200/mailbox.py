"""Point-to-point messaging and worker scheduling behind ``Fabric.run``
(the reference's ``Worker.send/recv``, ``reduce_to_root``,
``broadcast_from_root`` and its two scheduling modes, `pkg/src/parconv/fabric.py:98-339`).

The training step never goes through here (it is one device program per
worker: `schemes.py`, `multidev.py`); this is the general ``Fabric.run`` RPC a
caller's own worker programs use, with the reference's semantics kept:

* a payload is copied at ``send`` (mutating the buffer afterwards does not reach
  the receiver); numpy-like values travel as float64 at full precision while the
  ledger books ``elements x wire_element_size`` bytes (`fabric.py:116-128`);
* FIFO per (src, dst, tag); ``reduce_to_root`` sums in ascending worker order;
* ``lockstep``: exactly one worker program runs at a time and the turn passes to
  the next runnable worker (ascending, cyclic) when the running one blocks or
  finishes, so a run is deterministic; no runnable worker while some are
  unfinished = ``DeadlockError``. ``threads``: the programs run concurrently and
  a deadlock is declared when every unfinished worker is blocked and nothing has
  moved for ``idle_timeout`` seconds;
* the lowest failing worker's exception is raised after every thread unwinds.

B200 additions: a CUDA tensor payload is copied onto the receiver's GPU (peer
copy when the workers sit on different GPUs) on the sender's stream, and the
receiver's current stream waits for that copy before the value is handed out;
``reduce_to_root`` of CUDA tensors sums on the root's device, still in ascending
worker order. Under torchrun a message to a worker of another rank goes over
``torch.distributed`` send/recv (a small header carrying the tag, dtype and
shape, then the payload); messages that arrive ahead of the tag a ``recv`` waits
for are held in the mailbox, so per-tag FIFO order is kept. A cross-rank
deadlock is not detected (it blocks until the process group's timeout).
"""

from __future__ import annotations

import pickle
import threading
import time
from collections import deque

import numpy as np
import torch

from .errors import DeadlockError, ValidationError

_POLL = 0.02          # seconds between idle checks in threads mode


class _Unwind(Exception):
    """Unwinds a worker thread after another worker failed or a deadlock was declared."""


def _copy_payload(value, fabric, dst):
    """The message as the receiver will see it, plus the element count the ledger books."""
    if isinstance(value, torch.Tensor):
        if value.is_cuda:
            dev = fabric.device_of(dst) if dst in fabric.local_wids else value.device
            out = value.to(dev, copy=True, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(value.device))
            return (out, ev), value.numel()
        return (value.detach().clone(), None), value.numel()
    arr = np.array(value, dtype=np.float64, copy=True)
    return (arr, None), arr.size


def _deliver(item, fabric, wid):
    val, ev = item
    if ev is not None:
        torch.cuda.current_stream(val.device).wait_event(ev)
    return val


class Mailbox:
    """Channels and scheduler state of one fabric (reset at every ``run``)."""

    def __init__(self, fabric):
        self.fabric = fabric
        self.cond = threading.Condition()
        self.channels: dict = {}
        self.error: BaseException | None = None
        self.blocked: dict = {}      # wid -> (src, dst, tag) it waits on
        self.finished: set = set()
        self.turn = None
        self.last_move = time.monotonic()
        self.remote = None           # torchrun: _RemoteLink

    # ------------------------------------------------------------- run control
    def reset(self, wids: list) -> None:
        with self.cond:
            self.error = None
            self.blocked = {}
            self.finished = set(range(self.fabric.n)) - set(wids)
            self.turn = min(wids) if wids else None
            self.last_move = time.monotonic()

    def _ready(self, wid: int) -> bool:
        if wid in self.finished:
            return False
        key = self.blocked.get(wid)
        return key is None or bool(self.channels.get(key))

    def _pass_turn(self, wid: int) -> None:
        """lockstep: hand the turn to the next runnable worker after wid (cyclic)."""
        n = self.fabric.n
        for k in range(1, n + 1):
            w = (wid + k) % n
            if self._ready(w):
                self.turn = w
                self.cond.notify_all()
                return
        if len(self.finished) < n and self.error is None:
            self.error = self._deadlock()
        self.cond.notify_all()

    def _deadlock(self) -> DeadlockError:
        waiting = {w: {"src": key[0], "tag": key[2]} for w, key in sorted(self.blocked.items())
                   if w not in self.finished}
        what = "; ".join(f"worker {w} waits on recv(src={i['src']}, tag={i['tag']!r})" for w, i in waiting.items())
        return DeadlockError(f"fabric deadlock: no worker can make progress ({what})", waiting)

    def wait_turn(self, wid: int) -> None:
        if self.fabric.scheduling != "lockstep":
            return
        with self.cond:
            while self.turn != wid:
                if self.error is not None:
                    raise _Unwind()
                self.cond.wait()

    def done(self, wid: int, err: BaseException | None) -> None:
        with self.cond:
            if err is not None and self.error is None:
                self.error = err
            self.finished.add(wid)
            self.blocked.pop(wid, None)
            self.last_move = time.monotonic()
            if self.fabric.scheduling == "lockstep" and self.turn == wid:
                self._pass_turn(wid)
            self.cond.notify_all()

    # --------------------------------------------------------------- messaging
    def send(self, src: int, dst: int, tag, value) -> None:
        fab = self.fabric
        if not 0 <= dst < fab.n or dst == src:
            raise ValidationError(f"worker {src}: invalid destination {dst}")
        item, elements = _copy_payload(value, fab, dst)
        if dst not in fab.local_wids:            # torchrun: the receiver lives in another process
            self._remote().send(dst, tag, item)
        else:
            with self.cond:
                if self.error is not None:
                    raise _Unwind()
                self.channels.setdefault((src, dst, tag), deque()).append(item)
                self.last_move = time.monotonic()
                self.cond.notify_all()
        fab.ledger.record(src, dst, elements * fab.device.wire_element_size)

    def recv(self, wid: int, src: int, tag):
        fab = self.fabric
        if not 0 <= src < fab.n or src == wid:
            raise ValidationError(f"worker {wid}: invalid source {src}")
        if src not in fab.local_wids:
            return _deliver(self._remote().recv(src, tag), fab, wid)
        key = (src, wid, tag)
        with self.cond:
            while True:
                if self.error is not None:
                    raise _Unwind()
                q = self.channels.get(key)
                if q:
                    return _deliver(q.popleft(), fab, wid)
                self._block(wid, key)

    def _block(self, wid: int, key) -> None:
        """Called with the condition held; returns when key's channel may be non-empty."""
        self.blocked[wid] = key
        try:
            if self.fabric.scheduling == "lockstep":
                self._pass_turn(wid)
                while not (self.turn == wid and self._ready(wid)):
                    if self.error is not None:
                        raise _Unwind()
                    self.cond.wait()
                return
            while not self.channels.get(key):
                if self.error is not None:
                    raise _Unwind()
                idle = time.monotonic() - self.last_move
                if len(self.blocked) >= self.fabric.n - len(self.finished) and idle > self.fabric.idle_timeout:
                    self.error = self._deadlock()
                    self.cond.notify_all()
                    raise _Unwind()
                self.cond.wait(_POLL)
        finally:
            if self.error is None:
                self.blocked.pop(wid, None)

    def _remote(self) -> "_RemoteLink":
        if self.remote is None:
            self.remote = _RemoteLink(self.fabric)
        return self.remote


class _RemoteLink:
    """Messages between ranks (torchrun): header (tag, dtype, shape) then payload."""

    def __init__(self, fabric):
        import torch.distributed as dist
        self.dist = dist
        self.fabric = fabric
        self.held: dict = {}         # (src, tag) -> deque of payloads that arrived early
        self.pending: list = []      # isend handles (+ their buffers) not yet completed
        nccl = dist.get_backend() == "nccl"
        self.wire_dev = fabric.torch_device if nccl else torch.device("cpu")

    def send(self, dst: int, tag, item) -> None:
        val, ev = item
        if ev is not None:
            ev.synchronize()
        is_torch = isinstance(val, torch.Tensor)
        t = val if is_torch else torch.from_numpy(np.ascontiguousarray(val))
        head = pickle.dumps((tag, is_torch, str(t.dtype).replace("torch.", ""), tuple(t.shape)))
        # non-blocking: a ring of sends must not wait for the matching receives
        bufs = (torch.tensor([len(head)], dtype=torch.int64, device=self.wire_dev),
                torch.frombuffer(bytearray(head), dtype=torch.uint8).to(self.wire_dev),
                t.contiguous().to(self.wire_dev, copy=True))
        for b in bufs:
            self.pending.append((self.dist.isend(b, dst), b))

    def flush(self) -> None:
        """Wait for every outstanding send (end of a run)."""
        for work, _ in self.pending:
            work.wait()
        self.pending.clear()

    def recv(self, src: int, tag):
        q = self.held.get((src, tag))
        if q:
            return q.popleft()
        while True:
            n = torch.zeros(1, dtype=torch.int64, device=self.wire_dev)
            self.dist.recv(n, src)
            head = torch.empty(int(n.item()), dtype=torch.uint8, device=self.wire_dev)
            self.dist.recv(head, src)
            rtag, is_torch, dtype, shape = pickle.loads(head.cpu().numpy().tobytes())
            t = torch.empty(shape, dtype=getattr(torch, dtype), device=self.wire_dev)
            self.dist.recv(t, src)
            if is_torch:
                item = (t if t.is_cuda else t.clone(), None)
            else:
                item = (t.cpu().numpy(), None)
            if rtag == tag:
                return item
            self.held.setdefault((src, rtag), deque()).append(item)


def reduce_to_root(ctx, group, root: int, value, tag="reduce"):
    """Root returns the elementwise sum over the group in ascending worker order
    (`fabric.py:146-156`); CUDA tensors are summed on the root's device."""
    members = sorted(group)
    if ctx.wid != root:
        ctx.send(root, tag, value)
        return None
    acc = None
    for w in members:
        t = value if w == ctx.wid else ctx.recv(w, tag)
        if isinstance(t, torch.Tensor):
            acc = t.clone() if acc is None else acc.add_(t.to(acc.device))
        else:
            acc = np.array(t, dtype=np.float64, copy=True) if acc is None else acc + t
    return acc


def broadcast_from_root(ctx, group, root: int, value, tag="bcast"):
    """`fabric.py:158-165`."""
    if ctx.wid == root:
        if value is None:
            raise ValidationError(f"worker {root}: broadcast root needs a value")
        for w in sorted(group):
            if w != root:
                ctx.send(w, tag, value)
        return value
    return ctx.recv(root, tag)


def run_programs(fabric, program, args) -> list:
    """``Fabric.run``: program(Worker, *args[wid]) on every worker this process
    hosts, one thread each; the lowest failing worker's exception is raised."""
    from .fabric import Worker
    box = fabric.mailbox
    wids = list(fabric.local_wids)
    box.reset(wids)
    results = [None] * fabric.n
    failures: dict = {}

    def body(wid):
        err = None
        try:
            box.wait_turn(wid)
            results[wid] = program(Worker(fabric, wid), *args[wid])
        except _Unwind:
            pass
        except BaseException as e:  # noqa: BLE001 - re-raised by the caller below
            failures[wid] = err = e
        finally:
            box.done(wid, err)

    if len(wids) == 1:
        body(wids[0])
    else:
        threads = [threading.Thread(target=body, args=(w,), daemon=True, name=f"pc-worker-{w}") for w in wids]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    if box.remote is not None:
        box.remote.flush()
    if failures:
        raise failures[min(failures)]
    if box.error is not None:
        raise box.error
    return results
