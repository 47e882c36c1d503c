"""Parity helpers shared by the GPU step tests.

ReLU decisions get the same treatment as max-pool ties below: a pre-activation
within the step's rounding of zero can be positive in one precision and not in
the other (AlexNet fp32 at b256: a few dozen of 74M conv1 outputs), which moves
one pixel's whole gradient; the checker asserts each such flip is a near-zero
and replays the device's mask in the oracle.

End-to-end protocol: max-pool argmax is bit-exact at kernel
level; end to end, a window whose two largest inputs differ by less than the
float32 rounding of the step can legitimately rank differently in float32
and float64 (measured: 1 of 18,432 windows of AlexNet pool5 at B=2). The
checker therefore (1) asserts every argmax disagreement is such a near-tie and
(2) replays the device's argmax in the float64 oracle, so the tolerance
measures the arithmetic of the step rather than one tie's routing.
"""

import numpy as np

from oracle import ref_kernels as O
from oracle.ref_engine import OracleFabric


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def device_argmax(fab, plan):
    """{layer: [replica][column] argmax} from the device engines of a local fabric."""
    d, m = plan.data_shards, plan.model_columns
    per = {}
    for r in range(d):
        for j in range(m):
            for layer, a in fab._engines[plan.worker_of(r, j)].pool_argmax_host().items():
                per.setdefault(layer, [[None] * m for _ in range(d)])[r][j] = a
    return per


def device_relu_masks(fab, plan):
    """{relu layer: [replica][column] bool NCHW mask (device ReLU output > 0)}: the
    decisions the device's backward applies (fused producer ReLU, consumer mask)."""
    d, m = plan.data_shards, plan.model_columns
    per = {}
    for r in range(d):
        for j in range(m):
            eng = fab._engines[plan.worker_of(r, j)]
            for pos, st in enumerate(eng.layers):
                if st.kind == "relu":
                    mask = eng.activation_host(pos, "out") > 0
                    per.setdefault(st.cl.index, [[None] * m for _ in range(d)])[r][j] = mask
    return per


def assert_relu_near_ties(trace, forced, tie_tol):
    """Every ReLU decision the device made differently (replica 0) sits at a
    pre-activation within rounding of zero; returns the number of flips."""
    flips = 0
    for layer, per_rep in forced.items():
        for j, mask in enumerate(per_rep[0]):
            a = trace["fwd"][layer - 1][j]
            bad = mask != (a > 0)
            if bad.any():
                scale = max(float(np.max(np.abs(a))), 1e-30)
                worst = float(np.max(np.abs(a[bad])))
                assert worst <= tie_tol * scale, (layer, j, int(bad.sum()), worst, scale)
                flips += int(bad.sum())
    return flips


def assert_near_ties(trace, forced, cs, tie_tol=1e-5):
    """Every device/oracle argmax disagreement (replica 0) must be a near-tie."""
    flips = 0
    for layer, per_rep in forced.items():
        pool = next(c for c in cs.col_layers if c.index == layer)
        prev = trace["fwd"][layer - 1]
        for j, dev_arg in enumerate(per_rep[0]):
            x = prev[j]
            _, nat = O.maxpool_forward(x, pool.layer.kernel, pool.layer.stride)
            bad = np.argwhere(nat != dev_arg)
            scale = max(float(np.max(np.abs(x))), 1e-30)
            k, s = pool.layer.kernel, pool.layer.stride
            for b, c, oy, ox in bad:
                va = x[b, c, oy * s + nat[b, c, oy, ox] // k, ox * s + nat[b, c, oy, ox] % k]
                vb = x[b, c, oy * s + dev_arg[b, c, oy, ox] // k, ox * s + dev_arg[b, c, oy, ox] % k]
                assert abs(va - vb) <= tie_tol * scale, (layer, j, (b, c, oy, ox), va, vb)
            flips += len(bad)
    return flips


def oracle_replay(net, plan, dense, x, y, fab, tie_tol=None):
    """Oracle step with the device's pool decisions; returns (oracle, loss, trace, flips).
    tie_tol: 1e-5 of the layer's max in fp32 mode; 2e-2 in the bf16 / tf32 modes
    (2^-8 / 2^-11 relative operand rounding, accumulated through the layers)."""
    if tie_tol is None:
        tie_tol = 2e-2 if fab.precision in ("bf16", "tf32") else 1e-5
    forced = device_argmax(fab, plan)
    relu = device_relu_masks(fab, plan)
    trace = {}
    of = OracleFabric(net, plan, dense)
    loss = of.step(x, y, trace=trace, force_argmax=forced, force_relu=relu)
    flips = assert_near_ties(trace, forced, of.cs, tie_tol)
    flips += assert_relu_near_ties(trace, relu, tie_tol)
    return of, loss, trace, flips
