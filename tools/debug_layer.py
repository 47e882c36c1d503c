"""Check one conv layer's backward on the engine's own device buffers (AlexNet fp32)."""
import sys, math
import numpy as np, torch
sys.path.insert(0, __file__.rsplit("/tools", 1)[0])
import paper_1312_5853_b200 as P
from paper_1312_5853_b200 import kernels as K
from oracle import ref_kernels as O
from paper_1312_5853_b200.plan import plan_columnized

def rel(a, b): return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))
prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
# 1) kernel level at the AlexNet L10 / L8 shapes
for geom in [(2, 384, 13, 13, 256, 3, 1, 1), (2, 256, 13, 13, 384, 3, 1, 1), (2, 96, 27, 27, 256, 5, 1, 2)]:
    b, c, h, w, n, k, s, p = geom
    rs = np.random.RandomState(1)
    x = np.maximum(rs.randn(b, c, h, w), 0).astype(np.float32).astype(np.float64)
    wt = (rs.randn(n, c, k, k) * 0.05).astype(np.float32).astype(np.float64)
    gy = rs.randn(b, n, h, w).astype(np.float32).astype(np.float64) * 1e-3
    K.set_precision(prec)
    cp = K.ConvParams(wt, np.zeros(n), s, p)
    gx, gw, gb = K.conv2d_backward(x, cp, gy)
    rgx, rgw, rgb = O.conv2d_backward(x, wt, gy, s, p)
    print(geom, "kernel gx", rel(gx, rgx), "gw", rel(gw, rgw), "gb", rel(gb, rgb))
# 2) engine buffers
net = P.load_network("configs/alexnet.net")
plan = P.ParallelPlan(1, 1)
cs = plan_columnized(net, plan)
dense = {i: {k: v.astype(np.float32).astype(np.float64) for k, v in t.items()} for i, t in P.init_dense_params(net, 0).items()}
tr, _ = P.gen_synthetic(2, 1, net.input_shape, seed=0)
x, y = tr.images[:2], np.array([0, 7])
fab = P.spawn(1, precision=prec)
P.setup_workers(fab, plan, cs, dense, P.SgdState())
P.hybrid_step(fab, plan, cs, x, y)
eng = fab._engines[0]
g = eng.grads_host()
for li in (10, 8, 6, 3):
    i = [c.index for c in cs.col_layers].index(li)
    st = eng.layers[i]
    xin = eng.activation_host(i, "in") if False else None
    B = eng.B
    hh, ww, cc = st.in_nhwc
    xa = st.inp[: B * hh * ww * cc].float().cpu().numpy().astype(np.float64).reshape(B, hh, ww, cc).transpose(0, 3, 1, 2)
    ho, wo, nn = st.out_nhwc
    ga = st.gout[: B * ho * wo * nn].float().cpu().numpy().astype(np.float64).reshape(B, ho, wo, nn).transpose(0, 3, 1, 2)
    wd = dense[li]["w"]
    _, rgw, rgb = O.conv2d_backward(xa, wd, ga, st.cl.layer.stride, st.cl.layer.pad)
    print("engine L", li, "gw vs oracle-on-engine-buffers", rel(g[li]["w"], rgw), "gb", rel(g[li]["b"], rgb))
