"""Multi-process host logic of the N>1 path on CPU (gloo), no GPU needed.

The device step of a multi-GPU plan is one process per GPU; what crosses
processes is the column exchange (all-gather / reduce-scatter in the column
group, `schemes.py:287-318`) and the data-parallel gradient sum in the
replica group (`fabric.py:146-156`). These tests run the SAME exchange and
reducer classes the GPU path uses (``fabric.NcclExchange`` /
``fabric.NcclReducer`` over ``fabric.make_groups``) on CPU tensors with the
gloo backend, world sizes 2 and 4, and check them against the reference's
semantics restated in numpy: concatenation along channels in ascending
column order, each column receiving the sum of everyone's piece k, replica
gradients summed. The ledger booked per step equals ``comm_volume``.
"""

import os
import socket
import types

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import CONFIGS


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _fake_engine(m, per, column, replica, seed):
    """Minimal stand-in for a ColumnEngine: layer 1 is a cross layer fed by layer 0."""
    rs = np.random.default_rng(seed)
    lay0 = types.SimpleNamespace(out=torch.from_numpy(rs.standard_normal(per).astype(np.float32)))
    lay1 = types.SimpleNamespace(inp=torch.zeros(m * per), rs=torch.zeros(per),
                                 gin=torch.from_numpy(rs.standard_normal(m * per).astype(np.float32)))
    return types.SimpleNamespace(layers=[lay0, lay1], m=m, column=column, replica=replica,
                                 g32=torch.from_numpy(rs.standard_normal(64).astype(np.float32)))


def _expected(d, m, per, seed0):
    """numpy restatement of the reference exchange / reduction over all workers."""
    engines = {}
    for r in range(d):
        for j in range(m):
            engines[(r, j)] = _fake_engine(m, per, j, r, seed0 + r * m + j)
    gather, scatter, grad = {}, {}, {}
    for r in range(d):
        cat = np.concatenate([engines[(r, j)].layers[0].out.numpy() for j in range(m)])
        for k in range(m):
            gather[(r, k)] = cat
            acc = None
            for src in range(m):          # ascending source column (schemes.py:315-317)
                piece = engines[(r, src)].layers[1].gin.numpy()[k * per:(k + 1) * per].astype(np.float64)
                acc = piece if acc is None else acc + piece
            scatter[(r, k)] = acc
    for j in range(m):
        tot = sum(engines[(r, j)].g32.numpy().astype(np.float64) for r in range(d))
        for r in range(d):
            grad[(r, j)] = tot
    return gather, scatter, grad


def _worker(rank, world, port, d, m, per, seed0, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1312_5853_b200.fabric import NcclExchange, NcclReducer, make_groups
        replica, column = divmod(rank, m)
        col_g, rep_g = make_groups(d, m, rank)
        eng = _fake_engine(m, per, column, replica, seed0 + rank)
        if m > 1:
            ex = NcclExchange(col_g)
            ex.all_gather(1, [eng])
            ex.reduce_scatter(1, [eng])
        if d > 1:
            NcclReducer(rep_g).reduce({column: [eng]})
        q.put((rank, eng.layers[1].inp.numpy().copy(), eng.layers[1].rs.numpy().copy(), eng.g32.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("d,m", [(1, 2), (2, 1), (2, 2)])
def test_exchange_and_reduction_match_reference_semantics(d, m):
    world, per, seed0 = d * m, 96, 1234
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, d, m, per, seed0, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    gather, scatter, grad = _expected(d, m, per, seed0)
    for rank, inp, rs, g in got:
        r, j = divmod(rank, m)
        if m > 1:
            assert np.array_equal(inp, gather[(r, j)].astype(np.float32))
            np.testing.assert_allclose(rs, scatter[(r, j)], rtol=1e-6, atol=1e-6)
        if d > 1:
            np.testing.assert_allclose(g, grad[(r, j)], rtol=1e-6, atol=1e-6)


def test_group_layout_matches_reference_worker_ids():
    from paper_1312_5853_b200.fabric import group_members
    cols, reps = group_members(4, 2)
    assert cols == [[0, 1], [2, 3], [4, 5], [6, 7]]          # replica i: columns 0..m-1
    assert reps == [[0, 2, 4, 6], [1, 3, 5, 7]]               # column j across replicas
    from paper_1312_5853_b200.plan import ParallelPlan
    plan = ParallelPlan(4, 2, (6,))
    for i in range(4):
        for j in range(2):
            assert plan.worker_of(i, j) == cols[i][j] == reps[j][i]


@pytest.mark.parametrize("d,m,cross", [(2, 1, ()), (4, 1, ()), (1, 2, (3,)), (2, 2, (3,)), (1, 4, (3,))])
def test_booked_ledger_equals_comm_volume(d, m, cross):
    """Per step the device fabric books exactly the reference protocol's
    logical bytes and messages (`tests/test_schemes.py:370-394`)."""
    import paper_1312_5853_b200 as P
    from paper_1312_5853_b200.fabric import CommLedger, DeviceSpec, book_step
    from paper_1312_5853_b200.plan import plan_columnized
    net = P.load_network(CONFIGS / "tinynet.net")
    plan = P.ParallelPlan(d, m, cross)
    cs = plan_columnized(net, plan)
    fab = types.SimpleNamespace(ledger=CommLedger(), device=DeviceSpec())
    book_step(fab, plan, cs, 4)
    vol = P.comm_volume(plan, net, 4 * d)
    assert fab.ledger.total_bytes == vol.bytes
    assert fab.ledger.total_messages == vol.messages


def _bucket_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1312_5853_b200.fabric import NcclReducer, make_groups
        _, rep_g = make_groups(world, 1, rank)
        rs = np.random.default_rng(100 + rank)
        eng = types.SimpleNamespace(g32=torch.from_numpy(rs.standard_normal(64).astype(np.float32)))
        red = NcclReducer(rep_g)
        for lo, hi in ((40, 64), (16, 40), (0, 16)):      # backward order: last layer first
            red.layer_done(eng, lo, hi)
        red.reduce({0: [eng]})
        q.put((rank, eng.g32.numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_bucketed_gradient_allreduce_overlapped_with_backward():
    """Data-parallel reduction issued per layer region as the backward finishes it
    (async all-reduce buckets, waited before the SGD) sums the replicas exactly
    like one all-reduce of the flat gradient."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bucket_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = sum(np.random.default_rng(100 + r).standard_normal(64).astype(np.float32).astype(np.float64)
               for r in range(world))
    for r in range(world):
        np.testing.assert_allclose(got[r], want, rtol=1e-6, atol=1e-6)


def _ring_program(ctx):
    """Ring exchange with out-of-order tags, then reduce + broadcast (the
    reference's determinism program, `tests/test_fabric.py:219-240`)."""
    acc = np.full(4, float(ctx.wid) + 0.25)
    nxt, prv = (ctx.wid + 1) % ctx.n, (ctx.wid - 1) % ctx.n
    for step in range(3):
        ctx.send(nxt, ("late", step), acc * 2)
        ctx.send(nxt, ("ring", step), acc)
        acc = acc + ctx.recv(prv, ("ring", step))       # arrives behind the "late" message
        acc = acc - 0.5 * ctx.recv(prv, ("late", step))
    ctx.send(nxt, "t", torch.arange(3, dtype=torch.float32) + ctx.wid)
    t = ctx.recv(prv, "t")
    total = ctx.reduce_to_root(range(ctx.n), 0, acc)
    out = ctx.broadcast_from_root(range(ctx.n), 0, total if ctx.wid == 0 else None)
    return out, t


def _mailbox_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1312_5853_b200.fabric import spawn
        fab = spawn(world)
        res = fab.run(_ring_program)
        out, t = res[rank]
        q.put((rank, out, t.numpy(), fab.ledger.snapshot()))
    finally:
        dist.destroy_process_group()


def test_fabric_run_messaging_across_ranks_matches_one_process():
    """Fabric.run under a process group (one worker per rank): send/recv cross
    ranks over torch.distributed, tags matched out of order, CPU tensors kept as
    tensors; results equal the single-process run, and each rank books its own
    sends."""
    from paper_1312_5853_b200.fabric import spawn
    world = 3
    fab = spawn(world, scheduling="threads")
    want = fab.run(_ring_program)
    want_snap = fab.ledger.snapshot()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mailbox_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    booked = {}
    for rank, out, t, snap in got:
        assert np.array_equal(out, want[rank][0])
        assert np.array_equal(t, want[rank][1].numpy())
        for link, v in snap.items():
            assert link[0] == rank
            booked[link] = v
    assert booked == want_snap
