"""Device fabric: the B200 replacement of the reference's simulated fabric
(`pkg/src/parconv/fabric.py:36-345`).

Process model. One process per GPU under torchrun (``torch.distributed``
initialised, world size == plan workers): worker w = rank w, its column group
and replica group are NCCL sub-communicators, the cross-layer exchange is
``all_gather_into_tensor`` / ``reduce_scatter_tensor`` in the column group
and the data-parallel leg is one ``all_reduce`` over the flat gradient in
the replica group. Without a process group, one process drives every worker
of the plan like the reference's ``Fabric.run`` threads: on several visible
GPUs (or with ``devices=``) one host thread per worker on its own GPU and
stream, exchanging through peer memory (``multidev.py``); on one GPU every
worker shares the device and the same exchange is done with device copies and
the deterministic ``pc_sum_buffers`` kernel in ascending worker order — the
reference's summation order exactly (`fabric.py:146-156`, `schemes.py:307-318`);
both single-process forms give bit-identical results.

Bookkeeping kept from the reference so its callers keep working:
``ledger`` books every logical message the reference protocol would send
(element count x 4 B, `fabric.py:116-128`), so ``ledger.total_bytes``
equals ``comm_volume`` per step; ``meter`` books the accounted resident
bytes (`fabric.py:80-95`, `netdef.worker_footprint_bytes`).
"""

from __future__ import annotations

import math
import threading
from dataclasses import dataclass

import torch

from . import _lib as L
from . import mailbox as _mb
from .errors import CapacityError, ValidationError


@dataclass
class DeviceSpec:
    memory_capacity: int = 6 * 1024 ** 3
    wire_element_size: int = 4

    def __post_init__(self):
        if self.memory_capacity <= 0 or self.wire_element_size <= 0:
            raise ValidationError("device capacity and wire element size must be positive")


class CommLedger:
    """Bytes and message counts per ordered link (src, dst)."""

    def __init__(self):
        self._links: dict = {}
        self._lock = threading.Lock()

    def record(self, src: int, dst: int, nbytes: int) -> None:
        with self._lock:
            e = self._links.setdefault((src, dst), [0, 0])
            e[0] += int(nbytes)
            e[1] += 1

    def link(self, src: int, dst: int) -> tuple:
        e = self._links.get((src, dst), (0, 0))
        return e[0], e[1]

    @property
    def total_bytes(self) -> int:
        with self._lock:
            return sum(e[0] for e in self._links.values())

    @property
    def total_messages(self) -> int:
        with self._lock:
            return sum(e[1] for e in self._links.values())

    def snapshot(self) -> dict:
        with self._lock:
            return {k: (v[0], v[1]) for k, v in sorted(self._links.items())}


class MemoryMeter:
    def __init__(self, n: int):
        self.current = [0] * n
        self.peak = [0] * n

    def alloc(self, wid: int, nbytes: int) -> None:
        self.current[wid] += nbytes
        self.peak[wid] = max(self.peak[wid], self.current[wid])

    def free(self, wid: int, nbytes: int) -> None:
        self.current[wid] -= nbytes
        if self.current[wid] < 0:
            raise ValidationError(f"worker {wid}: freed more bytes than allocated")


class _LocalState(dict):
    """``ctx.local`` of the reference: per-worker state; "params"/"velocity"
    are materialised from the device engine on access."""

    def __init__(self, fabric, wid):
        super().__init__()
        self._fabric, self._wid = fabric, wid

    def __getitem__(self, key):
        eng = self._fabric._engines.get(self._wid)
        if eng is not None and key == "params":
            return eng.params_host()
        if eng is not None and key == "velocity":
            return eng.velocity_host() if self.get("holds_velocity") else None
        return super().__getitem__(key)

    def get(self, key, default=None):
        try:
            return self[key]
        except KeyError:
            return default


class Worker:
    """Handle passed to programs run with ``Fabric.run`` (identity + metering)."""

    def __init__(self, fabric: "Fabric", wid: int):
        self.fabric, self.wid, self.n = fabric, wid, fabric.n

    @property
    def local(self) -> dict:
        return self.fabric._local[self.wid]

    def alloc(self, elements: int) -> int:
        nbytes = int(elements) * self.fabric.device.wire_element_size
        self.fabric.meter.alloc(self.wid, nbytes)
        return nbytes

    def free_bytes(self, nbytes: int) -> None:
        self.fabric.meter.free(self.wid, nbytes)

    def assert_capacity(self) -> None:
        self.fabric.meter_assert(self.wid)

    # messaging (mailbox.py): the reference's semantics, device tensors move GPU to GPU
    def send(self, dst: int, tag, value) -> None:
        self.fabric.mailbox.send(self.wid, dst, tag, value)

    def recv(self, src: int, tag):
        return self.fabric.mailbox.recv(self.wid, src, tag)

    def reduce_to_root(self, group, root: int, value, tag="reduce"):
        return _mb.reduce_to_root(self, group, root, value, tag)

    def broadcast_from_root(self, group, root: int, value, tag="bcast"):
        return _mb.broadcast_from_root(self, group, root, value, tag)


class Fabric:
    """n workers of a plan mapped onto B200s (see module docstring)."""

    def __init__(self, n: int, device: DeviceSpec | None = None, scheduling: str = "lockstep",
                 idle_timeout: float = 5.0, precision: str = "bf16", devices: list | None = None):
        if n < 1:
            raise ValidationError(f"fabric needs at least one worker, got {n}")
        if scheduling not in ("lockstep", "threads"):
            raise ValidationError(f"unknown scheduling mode {scheduling!r}")
        if precision not in ("bf16", "fp32", "tf32"):
            raise ValidationError(f"unknown precision {precision!r} (bf16 | tf32 | fp32)")
        self.n = n
        self.device = device or DeviceSpec()
        self.scheduling, self.idle_timeout = scheduling, idle_timeout
        self.precision = precision
        # storage precision of activations, and the contractions' (tf32: float storage,
        # tcgen05 kind::tf32 tensor-core math; fp32: the exact SIMT verification mode)
        self.prec = L.PC_BF16 if precision == "bf16" else L.PC_FP32
        self.cprec = L.PC_TF32 if precision == "tf32" else self.prec
        self.ledger = CommLedger()
        self.meter = MemoryMeter(n)
        self._local = [_LocalState(self, w) for w in range(n)]
        self._engines: dict = {}
        self.dist = torch.distributed.is_available() and torch.distributed.is_initialized() \
            and torch.distributed.get_world_size() > 1
        if self.dist:
            ws = torch.distributed.get_world_size()
            if ws != n:
                raise ValidationError(f"fabric of {n} workers needs world size {n}, got {ws}")
            self.rank = torch.distributed.get_rank()
            self.local_wids = [self.rank]
        else:
            self.rank = 0
            self.local_wids = list(range(n))
        self.mailbox = _mb.Mailbox(self)
        self._groups = {}
        # without a CUDA device the fabric still runs worker programs (messaging,
        # metering); every device use (setup_workers, the steps) raises
        self._torch_device = None
        self.multi = False
        self._device_of = [None] * n
        if not torch.cuda.is_available():
            if devices is not None:
                raise ValidationError("devices= given but no CUDA device is visible")
            return
        idx = torch.cuda.current_device()
        if self.dist:
            import os
            idx = int(os.environ.get("LOCAL_RANK", self.rank % torch.cuda.device_count()))
            torch.cuda.set_device(idx)
        self._torch_device = torch.device("cuda", idx)
        # single process, several workers: one host thread + stream per worker on its GPU
        # (multidev.PeerRunner), the workers spread over the visible GPUs in contiguous
        # blocks (the columns of a replica share a GPU when there are fewer GPUs than
        # workers). devices=[...] pins worker w to GPU devices[w] (repeats allowed: the
        # same machinery on one GPU, which is how a one-GPU box tests it).
        self._device_of = [self.torch_device] * n
        if not self.dist and n > 1:
            if devices is not None:
                if len(devices) != n:
                    raise ValidationError(f"devices: need one GPU index per worker ({n}), got {len(devices)}")
                count = torch.cuda.device_count()
                if any(not 0 <= int(g) < count for g in devices):
                    raise ValidationError(f"devices {list(devices)}: only {count} GPU(s) visible")
                self._device_of = [torch.device("cuda", int(g)) for g in devices]
                self.multi = True
            elif torch.cuda.device_count() > 1:
                c = min(n, torch.cuda.device_count())
                self._device_of = [torch.device("cuda", w * c // n) for w in range(n)]
                self.multi = True
        elif devices is not None and list(devices) not in ([idx], [idx] * n):
            raise ValidationError("devices= applies to single-process fabrics")

    @property
    def torch_device(self) -> torch.device:
        if self._torch_device is None:
            raise ValidationError("the device fabric needs a CUDA device (B200); none is visible")
        return self._torch_device

    def device_of(self, wid: int) -> torch.device:
        if self._device_of[wid] is None:
            raise ValidationError("the device fabric needs a CUDA device (B200); none is visible")
        return self._device_of[wid]

    @property
    def num_links(self) -> int:
        return self.n * (self.n - 1)

    def meter_assert(self, wid: int) -> None:
        if self.meter.current[wid] > self.device.memory_capacity:
            raise CapacityError(wid, self.meter.current[wid], self.device.memory_capacity)

    def run(self, program, args: list | None = None) -> list:
        """program(ctx, *args[wid]) on every worker hosted by this process, one
        host thread each, scheduled ``lockstep`` or ``threads`` (mailbox.py);
        other processes' entries are None. Lowest failing worker's error wins."""
        if args is None:
            args = [() for _ in range(self.n)]
        if len(args) != self.n:
            raise ValidationError(f"need args for {self.n} workers, got {len(args)}")
        return _mb.run_programs(self, program, args)

    # --------------------------------------------------------- process groups
    def groups(self, d: int, m: int):
        """(column_group, replica_group) of this rank, created collectively once."""
        key = (d, m)
        if key not in self._groups:
            self._groups[key] = make_groups(d, m, self.rank)
        return self._groups[key]


def group_members(d: int, m: int) -> tuple:
    """Rank lists of the column groups (replica i: {i*m .. i*m+m-1}) and the
    replica groups (column j: {j, m+j, ...}), `schemes.py:84-85, 541-542`."""
    cols = [[i * m + j for j in range(m)] for i in range(d)]
    reps = [[r * m + j for r in range(d)] for j in range(m)]
    return cols, reps


def make_groups(d: int, m: int, rank: int):
    """Create every column and replica group (a collective call: all ranks
    create all groups in the same order) and return this rank's pair; None
    where the group would have one member."""
    dist = torch.distributed
    cols, reps = group_members(d, m)
    col = rep = None
    for i, ranks in enumerate(cols):
        g = dist.new_group(ranks) if m > 1 else None
        if rank // m == i:
            col = g
    for j, ranks in enumerate(reps):
        g = dist.new_group(ranks) if d > 1 else None
        if rank % m == j:
            rep = g
    return col, rep


def spawn(n: int, device: DeviceSpec | None = None, scheduling: str = "lockstep",
          idle_timeout: float = 5.0, precision: str = "bf16", devices: list | None = None) -> Fabric:
    """`fabric.py:342-345`. Under torchrun: worker = rank. In one process: every
    worker of the plan, spread over the visible GPUs (``devices`` to pin them)."""
    return Fabric(n, device=device, scheduling=scheduling, idle_timeout=idle_timeout,
                  precision=precision, devices=devices)


# ----------------------------------------------------------------------------
# Column exchange and data-parallel reduction
# ----------------------------------------------------------------------------


def _ptr_array(tensors, device):
    return torch.tensor([t.data_ptr() for t in tensors], dtype=torch.int64, device=device)


class LocalExchange:
    """All m columns of a replica on one device: copies + ascending-order sums."""

    def __init__(self, device):
        self.device = device
        self._ptrs = {}

    def all_gather(self, i: int, engines: list):
        for dst in engines:
            st = dst.layers[i]
            per = st.rs.numel()
            for k, src in enumerate(engines):
                st.inp[k * per:(k + 1) * per].copy_(src.layers[i - 1].out[:per])

    def reduce_scatter(self, i: int, engines: list):
        lib = L.lib()
        m = len(engines)
        for k, dst in enumerate(engines):
            st = dst.layers[i]
            per = st.rs.numel()
            key = (i, k, id(engines[0]))
            if key not in self._ptrs:
                self._ptrs[key] = _ptr_array([e.layers[i].gin[k * per:(k + 1) * per] for e in engines],
                                             self.device)
            lib.call("pc_sum_buffers", m, per, self._ptrs[key].data_ptr(), st.rs.data_ptr(),
                     dst.prec, dst.stream)


class NcclExchange:
    """One column per rank: all-gather / reduce-scatter in the column group."""

    def __init__(self, group):
        self.group = group

    def all_gather(self, i: int, engines: list):
        (e,) = engines
        st = e.layers[i]
        per = st.rs.numel()
        torch.distributed.all_gather_into_tensor(st.inp[: per * e.m], e.layers[i - 1].out[:per],
                                                 group=self.group)

    def reduce_scatter(self, i: int, engines: list):
        (e,) = engines
        st = e.layers[i]
        per = st.rs.numel()
        torch.distributed.reduce_scatter_tensor(st.rs[:per], st.gin[: per * e.m], group=self.group)


class LocalReducer:
    """d replicas of each column on one device: deterministic ascending sum
    into replica 0's gradient, which every replica's SGD then reads."""

    def __init__(self, device):
        self.device = device
        self._ptrs = {}

    def reduce(self, per_column: dict):
        lib = L.lib()
        for j, engines in per_column.items():
            if len(engines) < 2:
                continue
            key = (j, id(engines[0]))
            if key not in self._ptrs:
                self._ptrs[key] = _ptr_array([e.g32 for e in engines], self.device)
                for e in engines[1:]:
                    e.set_grad_source(engines[0].g32)
            e0 = engines[0]
            lib.call("pc_sum_buffers", len(engines), e0.n_flat, self._ptrs[key].data_ptr(),
                     e0.g32.data_ptr(), L.PC_FP32, e0.stream)


class NcclReducer:
    """One replica per rank: sum the flat gradient over the replica group.

    Overlapped with the backward: the flat gradient is in ascending layer order
    and the backward runs in descending order, so as soon as a layer's weight
    gradient kernels are enqueued its region is final. ``layer_done`` then
    issues an asynchronous all-reduce of that region (NCCL's stream waits for
    the compute stream at the call, then runs beside the rest of the backward);
    ``reduce`` makes the compute stream wait for every bucket before the SGD.
    Buckets are layers (AlexNet: fc8 4.1M, fc7 16.8M, fc6 37.7M, then the convs)."""

    def __init__(self, group):
        self.group = group
        self.works = []

    def layer_done(self, e, lo: int, hi: int):
        self.works.append(torch.distributed.all_reduce(e.g32[lo:hi], group=self.group, async_op=True))

    def reduce(self, per_column: dict):
        if not self.works:   # nothing was bucketed (no layer_done calls): one all-reduce per engine
            for engines in per_column.values():
                for e in engines:
                    torch.distributed.all_reduce(e.g32, group=self.group)
            return
        for w in self.works:
            w.wait()
        self.works = []


def book_step(fabric: Fabric, plan, cs, shard: int) -> None:
    """Book the messages the reference protocol sends in one step."""
    d, m, wire = plan.data_shards, plan.model_columns, fabric.device.wire_element_size
    led = fabric.ledger
    for leg in ("fwd", "bwd"):
        for cl in cs.col_layers:
            if not cl.cross:
                continue
            nbytes = shard * (math.prod(cl.in_shape) // m) * wire
            for r in range(d):
                for j in range(m):
                    for k in range(m):
                        if k != j:
                            led.record(r * m + j, r * m + k, nbytes)
    if d > 1:
        col = cs.column_param_count * wire
        for j in range(m):
            root = j
            for r in range(1, d):
                led.record(r * m + j, root, col)
            for r in range(1, d):
                led.record(root, r * m + j, col)
