import sys
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools", 1)[0])
sys.path.insert(0, __file__.rsplit("/tools", 1)[0] + "/tests")
import paper_1312_5853_b200 as P
from oracle import ref_kernels as O
from oracle.ref_engine import OracleFabric
from paper_1312_5853_b200.plan import plan_columnized
from parity import device_argmax, rel
STEPS = np.load("tests/golden/steps.npz")
prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
net = P.load_network("configs/alexnet_small64.net")
plan = P.ParallelPlan(1, 2, (6,))
cs = plan_columnized(net, plan)
dense = {i: {k: v.astype(np.float32).astype(np.float64) for k, v in t.items()} for i, t in P.init_dense_params(net, 3).items()}
x, y = STEPS["small64_x0"], STEPS["small64_y0"]
fab = P.spawn(2, precision=prec)
P.setup_workers(fab, plan, cs, dense, P.SgdState())
res = P.hybrid_step(fab, plan, cs, x, y)
trace = {}
of = OracleFabric(net, plan, dense)
of.step(x, y, trace=trace)
forced = device_argmax(fab, plan)
for j in range(2):
    eng = fab._engines[j]
    dev_in = eng.activation_host(0, "out")   # conv1 (+relu) output
    ref_in = trace["fwd"][1][j]
    print("col", j, "conv1 out maxrel", rel(dev_in, ref_in))
    for layer in (2, 5, 12):
        pool = next(c for c in cs.col_layers if c.index == layer)
        i = [c.index for c in cs.col_layers].index(layer)
        xd = eng.activation_host(i - 1, "out") if not eng.layers[i-1].relu_fused_fwd else eng.activation_host(i - 2, "out")
        xr = trace["fwd"][layer - 1][j]
        _, nat = O.maxpool_forward(xr, 3, 2)
        _, natd = O.maxpool_forward(xd, 3, 2)
        dev = forced[layer][0][j]
        bad = np.argwhere(nat != dev)
        print(f" pool {layer}: in maxrel {rel(xd, xr):.2e}  mismatches oracle-vs-device {len(bad)}; "
              f"device-kernel vs numpy-on-device-input {int((natd != dev).sum())}")
        for b, c, oy, ox in bad[:3]:
            k = 3; s = 2
            win_r = xr[b, c, oy*s:oy*s+3, ox*s:ox*s+3].ravel()
            win_d = xd[b, c, oy*s:oy*s+3, ox*s:ox*s+3].ravel()
            print("   win ref", np.round(win_r, 6), "nat", nat[b, c, oy, ox])
            print("   win dev", np.round(win_d, 6), "dev", dev[b, c, oy, ox])
