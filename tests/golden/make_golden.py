"""Generate the golden fixtures from the REAL reference (build container only).

Run:  python tests/golden/make_golden.py
It imports ``parconv`` from /root/reference/pkg/src (read-only) and writes
small ``.npz`` files next to this script. The GPU box never runs this; the
committed fixtures travel with the repo. Every array here is produced by
the reference's own functions on seeded inputs:

* kernels.npz  — kernels.py ops on random small shapes (incl. stride-4,
                 padded, overlapping-pool ties, label edge cases, SGD).
* steps.npz    — reference_step / hybrid_step trajectories on tinynet and
                 alexnet_small64 (losses + parameters after each step).
* alexnet.npz  — AlexNet-227 reference_step at B=2: loss and per-tensor
                 digests (sum, L2) of gradients-as-updates.
* host.npz     — SplitMix64 streams, permutations, synthetic data, comm
                 volumes, shape reports (host-logic KATs).
* eval.npz     — evaluation_errors after one hybrid_step of four plans:
                 misclassification counts and the exchange bytes it ledgers.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))

from parconv import kernels as K, rng, schemes as S, netdef as N, data as D  # noqa: E402
from parconv.fabric import spawn  # noqa: E402

OUT = Path(__file__).resolve().parent
CONFIGS = Path(__file__).resolve().parents[2] / "configs"


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def kernels_fixture():
    rs = np.random.RandomState(1234)
    out = {}
    geoms = [  # (B, C, H, W, N, k, s, p)
        (2, 3, 9, 9, 4, 3, 1, 1),
        (2, 4, 9, 9, 5, 3, 2, 0),
        (1, 3, 23, 23, 6, 11, 4, 0),
        (2, 6, 7, 7, 8, 5, 1, 2),
        (3, 16, 6, 6, 16, 3, 1, 1),
    ]
    for gi, (b, c, h, w, n, k, s, p) in enumerate(geoms):
        x = f32(rs.randn(b, c, h, w))
        wt = f32(rs.randn(n, c, k, k) * 0.3)
        bias = f32(rs.randn(n) * 0.1)
        cp = K.ConvParams(wt, bias, s, p)
        y = K.conv2d_forward(x, cp)
        gy = f32(rs.randn(*y.shape))
        gx, gw, gb = K.conv2d_backward(x, cp, gy)
        out.update({f"conv{gi}_geom": np.array([b, c, h, w, n, k, s, p]), f"conv{gi}_x": x,
                    f"conv{gi}_w": wt, f"conv{gi}_b": bias, f"conv{gi}_y": y, f"conv{gi}_gy": gy,
                    f"conv{gi}_gx": gx, f"conv{gi}_gw": gw, f"conv{gi}_gb": gb})
    for gi, (b, d, u) in enumerate([(4, 24, 16), (3, 72, 10), (8, 128, 64)]):
        x, w, bias = f32(rs.randn(b, d)), f32(rs.randn(d, u) * 0.2), f32(rs.randn(u))
        y = K.fc_forward(x, w, bias)
        gy = f32(rs.randn(b, u))
        gx, gw, gb = K.fc_backward(x, w, gy)
        out.update({f"fc{gi}_x": x, f"fc{gi}_w": w, f"fc{gi}_b": bias, f"fc{gi}_y": y,
                    f"fc{gi}_gy": gy, f"fc{gi}_gx": gx, f"fc{gi}_gw": gw, f"fc{gi}_gb": gb})
    xr = f32(rs.randn(3, 4, 5, 5))
    xr[0, 0, 0, :3] = 0.0
    xr[1, 1, 2, 2] = -0.0
    gr = f32(rs.randn(*xr.shape))
    out.update({"relu_x": xr, "relu_y": K.relu_forward(xr), "relu_g": gr,
                "relu_gx": K.relu_backward(xr, gr)})
    for gi, (shape, k, s) in enumerate([((2, 3, 7, 7), 3, 2), ((1, 2, 6, 6), 2, 2),
                                        ((2, 4, 13, 13), 3, 2), ((2, 2, 9, 9), 3, 2)]):
        x = f32(rs.randn(*shape))
        if gi == 3:  # quantised values => many ties inside windows
            x = np.round(x * 2.0) / 2.0
        y, arg = K.maxpool_forward(x, k, s)
        gy = f32(rs.randn(*y.shape))
        out.update({f"pool{gi}_x": x, f"pool{gi}_ks": np.array([k, s]), f"pool{gi}_y": y,
                    f"pool{gi}_arg": arg, f"pool{gi}_gy": gy,
                    f"pool{gi}_gx": K.maxpool_backward(x, k, s, gy, arg)})
    for gi, (b, kk, scale) in enumerate([(4, 10, 0.25), (6, 1000, 1 / 256), (3, 7, 1.0)]):
        logits = f32(rs.randn(b, kk) * 3.0)
        if gi == 2:
            logits[0] = 0.0
            logits[1, :] = 80.0
            logits[1, 3] = 120.0
        labels = rs.randint(0, kk, size=b)
        labels[0] = kk - 1
        loss, grad = K.softmax_xent_scaled(logits, labels, scale)
        out.update({f"sm{gi}_logits": logits, f"sm{gi}_labels": labels,
                    f"sm{gi}_scale": np.array(scale), f"sm{gi}_loss": np.array(loss),
                    f"sm{gi}_grad": grad})
    ps = [f32(rs.randn(5, 3)), f32(rs.randn(7))]
    gs = [f32(rs.randn(5, 3)), f32(rs.randn(7))]
    st = K.SgdState(0.01, 0.9, 0.0005, [f32(rs.randn(5, 3) * 0.01), f32(rs.randn(7) * 0.01)])
    newp, newst = K.sgd_step(ps, gs, st)
    for i in range(2):
        out.update({f"sgd_p{i}": ps[i], f"sgd_g{i}": gs[i], f"sgd_v{i}": st.velocity[i],
                    f"sgd_np{i}": newp[i], f"sgd_nv{i}": newst.velocity[i]})
    np.savez_compressed(OUT / "kernels.npz", **out)


def _tree(prefix, tree):
    return {f"{prefix}_{i}_{k}": v for i, t in tree.items() for k, v in t.items()}


def _digest(prefix, tree):
    """(sum, L2 norm, max |.|) per tensor — size-independent summaries."""
    return {f"{prefix}_{i}_{k}": np.array([v.sum(), np.sqrt((v ** 2).sum()), np.abs(v).max()])
            for i, t in tree.items() for k, v in t.items()}


def steps_fixture():
    out = {}
    tiny = N.load_network(CONFIGS / "tinynet.net")
    small = N.load_network(CONFIGS / "alexnet_small64.net")
    for name, net, batch, nsteps in (("tiny", tiny, 8, 3), ("small64", small, 4, 2)):
        train, _ = D.gen_synthetic(net.classes, max(1, (batch * nsteps) // net.classes + 1),
                                   net.input_shape, seed=7)
        params = S.init_dense_params(net, 3)
        params = {i: {k: f32(v) for k, v in t.items()} for i, t in params.items()}
        full = name == "tiny"   # small64 is 3.3M params: store digests only
        out.update(_tree(f"{name}_p0", params) if full else _digest(f"{name}_p0", params))
        sgd = K.SgdState()
        order = rng.permutation(7, 0, train.size)
        for st in range(nsteps):
            idx = order[st * batch:(st + 1) * batch]
            x, y = train.images[idx], train.labels[idx]
            out[f"{name}_x{st}"], out[f"{name}_y{st}"] = x, y
            res = S.reference_step(net, params, (x, y), sgd)
            delta = {i: {k: res.params[i][k] - params[i][k] for k in t} for i, t in params.items()}
            params, sgd = res.params, res.sgd
            out[f"{name}_loss{st}"] = np.array(res.loss)
            out.update(_tree(f"{name}_p{st + 1}", params) if full
                       else _digest(f"{name}_d{st + 1}", delta))
    # hybrid plans on tinynet: losses and per-column params after 2 steps
    plans = {"d2m1": S.ParallelPlan(2, 1), "d1m2x3": S.ParallelPlan(1, 2, (3,)),
             "d2m2x3": S.ParallelPlan(2, 2, (3,)), "d1m4x3": S.ParallelPlan(1, 4, (3,)),
             "d1m2grp": S.ParallelPlan(1, 2, ())}
    p0 = {i: {"w": out[f"tiny_p0_{i}_w"], "b": out[f"tiny_p0_{i}_b"]} for i in (0, 3, 5, 7)}
    for pname, plan in plans.items():
        cs = S.plan_columnized(tiny, plan)
        fab = spawn(plan.workers)
        S.setup_workers(fab, plan, cs, p0, K.SgdState())
        for st in range(2):
            res = S.hybrid_step(fab, plan, cs, out[f"tiny_x{st}"], out[f"tiny_y{st}"])
            out[f"hyb_{pname}_loss{st}"] = np.array(res.loss)
            out[f"hyb_{pname}_ledger{st}"] = np.array([res.ledger_bytes, res.ledger_messages])
        cols = fab.run(lambda ctx: ctx.local["params"] if ctx.local["replica"] == 0 else None)
        for j in range(plan.model_columns):
            out.update(_tree(f"hyb_{pname}_col{j}", cols[j]))
    np.savez_compressed(OUT / "steps.npz", **out)


def alexnet_fixture():
    net = N.load_network(CONFIGS / "alexnet.net")
    train, _ = D.gen_synthetic(2, 1, net.input_shape, seed=0)
    x, y = train.images, np.array([3, 999])
    params = S.init_dense_params(net, 0)
    params = {i: {k: f32(v) for k, v in t.items()} for i, t in params.items()}
    res = S.reference_step(net, params, (x, y), K.SgdState())
    out = {"x": x.astype(np.float32), "y": y, "loss": np.array(res.loss)}
    out.update(_digest("p0", params))
    out.update(_digest("d", {i: {k: res.params[i][k] - v for k, v in t.items()}
                             for i, t in params.items()}))
    np.savez_compressed(OUT / "alexnet.npz", **out)


def host_fixture():
    out = {}
    for seed, dom, idx in ((0, 1, 0), (42, 2, 3), (2**63 + 5, 4, 17)):
        s = rng.derive(seed, dom, idx)
        out[f"derive_{seed}_{dom}_{idx}"] = np.array([s.next_u64() for _ in range(4)], dtype=np.uint64)
    g = rng.derive(9, 1)
    out["gauss"] = g.gauss_array((3, 5), std=0.7)
    out["uniform"] = rng.derive(9, 3, 2).uniform_array(11, -1.0, 1.0)
    out["perm"] = rng.permutation(0, 0, 1000)
    out["perm_e3"] = rng.permutation(5, 3, 37)
    tr, te = D.gen_synthetic(3, 2, (2, 4, 4), seed=11)
    out.update({"syn_train_x": tr.images, "syn_train_y": tr.labels, "syn_test_x": te.images})
    nets = {n: N.load_network(CONFIGS / f"{n}.net") for n in ("alexnet", "tinynet", "alexnet_small64")}
    plans = [("alexnet", (1, 1, ())), ("alexnet", (2, 1, ())), ("alexnet", (8, 1, ())),
             ("alexnet", (1, 2, (6,))), ("alexnet", (4, 2, (6,))), ("alexnet", (2, 2, (3, 6, 8, 10))),
             ("tinynet", (2, 2, (3,))), ("tinynet", (1, 4, (3,))), ("alexnet_small64", (1, 2, (6,)))]
    rows = []
    for nname, (d, m, cross) in plans:
        plan = S.ParallelPlan(d, m, cross)
        cv = S.comm_volume(plan, nets[nname], 256 * d if nname == "alexnet" else 8 * d)
        cs = S.plan_columnized(nets[nname], plan)
        rep = N.shape_report(cs, 256)
        rows.append([cv.bytes, cv.messages, cs.column_param_count, rep.total_flops,
                     N.worker_footprint_bytes(cs, 32), len(cs.cross_layers)])
    out["plan_rows"] = np.array(rows, dtype=np.int64)
    np.savez_compressed(OUT / "host.npz", **out)


def eval_fixture():
    """evaluation_errors (`schemes.py:600-645`) after one step of several plans:
    misclassification counts and the ledger bytes / messages the evaluation books."""
    out = {}
    tiny = N.load_network(CONFIGS / "tinynet.net")
    small = N.load_network(CONFIGS / "alexnet_small64.net")
    cases = {"tiny_d1m2x3": (tiny, S.ParallelPlan(1, 2, (3,)), 8, 7),
             "tiny_d2m2x3": (tiny, S.ParallelPlan(2, 2, (3,)), 8, 7),
             "tiny_d2m1": (tiny, S.ParallelPlan(2, 1), 8, 7),
             "small64_d1m2x6": (small, S.ParallelPlan(1, 2, (6,)), 4, 3)}
    for name, (net, plan, batch, seed) in cases.items():
        train, test = D.gen_synthetic(net.classes, 2, net.input_shape, seed=seed, test_per_class=1)
        params = S.init_dense_params(net, 3)
        params = {i: {k: f32(v) for k, v in t.items()} for i, t in params.items()}
        cs = S.plan_columnized(net, plan)
        fab = spawn(plan.workers)
        S.setup_workers(fab, plan, cs, params, K.SgdState())
        x, y = train.images[:batch], train.labels[:batch]
        S.hybrid_step(fab, plan, cs, x, y)
        n_eval = min(test.size, 40 if net is tiny else 16)
        b0, m0 = fab.ledger.total_bytes, fab.ledger.total_messages
        wrong = S.evaluation_errors(fab, plan, cs, test.images[:n_eval], test.labels[:n_eval])
        out[f"{name}_x"], out[f"{name}_y"] = x.astype(np.float32), y      # float32-exact
        out[f"{name}_tx"], out[f"{name}_ty"] = test.images[:n_eval].astype(np.float32), test.labels[:n_eval]
        out[f"{name}_wrong"] = np.array(wrong)
        out[f"{name}_ledger"] = np.array([fab.ledger.total_bytes - b0, fab.ledger.total_messages - m0])
    np.savez_compressed(OUT / "eval.npz", **out)


if __name__ == "__main__":
    eval_fixture()
    kernels_fixture()
    host_fixture()
    steps_fixture()
    alexnet_fixture()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
