"""Layer-by-layer error report of the device step vs the float64 oracle (AlexNet-227)."""
import sys
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools", 1)[0])
import paper_1312_5853_b200 as P
from oracle.ref_engine import OracleFabric
from paper_1312_5853_b200.plan import plan_columnized

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 2
std = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
net = P.load_network("configs/alexnet.net")
plan = P.ParallelPlan(1, 1)
cs = plan_columnized(net, plan)
init = P.init_dense_params(net, 0, std=std if std > 0 else None)
dense = {i: {k: v.astype(np.float32).astype(np.float64) for k, v in t.items()} for i, t in init.items()}
tr, _ = P.gen_synthetic(2, (B + 1) // 2, net.input_shape, seed=0)
x, y = tr.images[:B], np.arange(B) * 7 % 1000
trace = {}
of = OracleFabric(net, plan, dense)
ol = of.step(x, y, trace=trace)
fab = P.spawn(1, precision=prec)
P.setup_workers(fab, plan, cs, dense, P.SgdState())
res = P.hybrid_step(fab, plan, cs, x, y)
print(f"loss dev {res.loss:.8f} oracle {ol:.8f} rel {abs(res.loss-ol)/abs(ol):.2e}")
eng = fab._engines[0]
def rel(a, b): return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))
def rl2(a, b): return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
for i, cl in enumerate(cs.col_layers):
    st = eng.layers[i]
    if st.kind == "softmax" or (st.kind == "relu" and st.relu_fused_fwd):
        continue
    ref = trace["fwd"][cl.index + 1 if st.relu_after else cl.index][0]
    got = eng.activation_host(i, "out")
    print(f"fwd L{cl.index:2d} {st.kind:5s} maxrel {rel(got, ref):.2e} relL2 {rl2(got, ref):.2e}")
g = eng.grads_host()
for i in sorted(g):
    for k in ("w", "b"):
        print(f"grad L{i:2d} {k} maxrel {rel(g[i][k], trace['grads'][0][i][k]):.2e} relL2 {rl2(g[i][k], trace['grads'][0][i][k]):.2e}")
# input-gradient buffers vs the oracle's trace (grad w.r.t. each layer's input)
for i, cl in enumerate(cs.col_layers):
    st = eng.layers[i]
    if i == 0 or st.gin is None:
        continue
    try:
        got = eng.activation_host(i, "gin")
    except Exception as e:  # noqa
        print("gin", cl.index, "n/a", e); continue
    ref = trace["bwd"][cl.index][0]
    if st.kind == "fc" and ref.ndim == 2 and got.ndim == 4:
        ref = ref.reshape(got.shape)
    if got.shape != ref.shape:
        ref = ref.reshape(got.shape)
    print(f"gin L{cl.index:2d} {st.kind:7s} maxrel {rel(got, ref):.2e} relL2 {rl2(got, ref):.2e}")
# pool 12 deep-dive
i12 = [c.index for c in cs.col_layers].index(12)
st = eng.layers[i12]
B = eng.B
hh, ww, cc = st.in_nhwc
ho, wo, _ = st.out_nhwc
nchw = lambda t, s: t[: int(np.prod(s))].float().cpu().numpy().astype(np.float64).reshape(s).transpose(0, 3, 1, 2)
xin = nchw(st.inp, (B, hh, ww, cc))
gout = nchw(st.gout, (B, ho, wo, cc))
gin = nchw(st.gin, (B, hh, ww, cc))
arg = st.argmax[: B * ho * wo * cc].cpu().numpy().reshape(B, ho, wo, cc).transpose(0, 3, 1, 2)
print("inp12 vs fwd[11]", rel(xin, trace["fwd"][11][0]))
print("gout12 vs bwd[13]", rel(gout, trace["bwd"][13][0].reshape(gout.shape)))
print("argmax12 mismatches", int((arg != trace["argmax"][12][0]).sum()))
print("gin12 vs bwd[11]", rel(gin, trace["bwd"][11][0]), "vs bwd[12]*mask", rel(gin, trace["bwd"][12][0] * (trace["fwd"][11][0] > 0)))
print("oracle self-consistency bwd[11] vs bwd[12]*(fwd[10]>0)", rel(trace["bwd"][11][0], trace["bwd"][12][0] * (trace["fwd"][10][0] > 0)))
