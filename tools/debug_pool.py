import sys
import numpy as np, torch
sys.path.insert(0, __file__.rsplit("/tools", 1)[0])
import paper_1312_5853_b200 as P
from paper_1312_5853_b200 import kernels as K
from oracle import ref_kernels as O
from paper_1312_5853_b200.plan import plan_columnized
def rel(a, b): return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))
for shape in [(2, 256, 13, 13), (2, 96, 55, 55), (2, 48, 7, 7)]:
    rs = np.random.RandomState(0)
    x = np.maximum(rs.randn(*shape), 0).astype(np.float32).astype(np.float64)
    y, arg = K.maxpool_forward(x, 3, 2)
    ry, rarg = O.maxpool_forward(x, 3, 2)
    gy = rs.randn(*ry.shape)
    gx = K.maxpool_backward(x, 3, 2, gy, arg)
    rgx = O.maxpool_backward(x.shape, 3, 2, gy, rarg)
    print(shape, "y", rel(y, ry), "argmax mismatches", int((arg != rarg).sum()), "gx", rel(gx, rgx))
net = P.load_network("configs/alexnet.net")
plan = P.ParallelPlan(1, 1)
cs = plan_columnized(net, plan)
dense = {i: {k: v.astype(np.float32).astype(np.float64) for k, v in t.items()} for i, t in P.init_dense_params(net, 0).items()}
tr, _ = P.gen_synthetic(2, 1, net.input_shape, seed=0)
fab = P.spawn(1, precision="fp32")
P.setup_workers(fab, plan, cs, dense, P.SgdState())
P.hybrid_step(fab, plan, cs, tr.images[:2], np.array([0, 7]))
eng = fab._engines[0]
for li in (12, 5, 2):
    i = [c.index for c in cs.col_layers].index(li)
    st = eng.layers[i]
    B = eng.B
    hh, ww, cc = st.in_nhwc
    xa = st.inp[: B * hh * ww * cc].float().cpu().numpy().astype(np.float64).reshape(B, hh, ww, cc).transpose(0, 3, 1, 2)
    ho, wo, _ = st.out_nhwc
    ga = st.gout[: B * ho * wo * cc].float().cpu().numpy().astype(np.float64).reshape(B, ho, wo, cc).transpose(0, 3, 1, 2)
    ea = st.argmax[: B * ho * wo * cc].cpu().numpy().reshape(B, ho, wo, cc).transpose(0, 3, 1, 2).astype(np.int64)
    ry, rarg = O.maxpool_forward(xa, 3, 2)
    rgx = O.maxpool_backward(xa.shape, 3, 2, ga, rarg) * (xa > 0)
    gx = st.gin[: B * hh * ww * cc].float().cpu().numpy().astype(np.float64).reshape(B, hh, ww, cc).transpose(0, 3, 1, 2)
    print("engine pool", li, "argmax mismatches", int((ea != rarg).sum()), "of", ea.size, "gx", rel(gx, rgx),
          "zeros-in-x", float((xa == 0).mean()))
