"""Kernel timeline of the timed step (CUDA-graph replay, AlexNet-227 d1m1 b256 bf16,
the bench's setup) from CUPTI activity records via torch.profiler: start offset,
duration and stream of every kernel of one replayed step, the busy time per
stream and the main stream's idle gaps. python tools/timeline.py [out.txt]"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1312_5853_b200 as P  # noqa: E402
from paper_1312_5853_b200 import schemes as S  # noqa: E402
from paper_1312_5853_b200.data import synthetic_rows  # noqa: E402
from paper_1312_5853_b200.plan import plan_columnized  # noqa: E402
from paper_1312_5853_b200 import rng as R  # noqa: E402

net = P.load_network(ROOT / "configs" / "alexnet.net")
plan = P.ParallelPlan(1, 1)
cs = plan_columnized(net, plan)
xb, yb = synthetic_rows(1000, 1, net.input_shape, 0, R.permutation(0, 0, 1000)[:256])
x = torch.from_numpy(np.ascontiguousarray(xb, dtype=np.float32)).to(torch.bfloat16).pin_memory()
y = torch.from_numpy(yb.astype(np.int32)).pin_memory()
fab = P.spawn(1, precision="bf16")
P.setup_workers(fab, plan, cs, P.init_dense_params(net, 0, std=0.01), P.SgdState())
P.hybrid_step(fab, plan, cs, x, y)
run = S._runner(fab, plan, cs, 256)
for _ in range(5):
    run.program(1.0 / 256)
torch.cuda.synchronize()

from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        run.program(1.0 / 256)
    torch.cuda.synchronize()

evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0]
kern = sorted(((e.time_range.start, e.time_range.end, getattr(e, "device_resource_id", 0), e.name) for e in evs
               if "memcpy" not in e.name.lower() and "memset" not in e.name.lower()), key=lambda t: t[0])
# one step = from the last input-layer kernel (the step's first launch) to the end
firsts = [i for i, k in enumerate(kern) if "s2d_rows" in k[3] or "s2d_k<" in k[3]]
kern = kern[firsts[-1]:] if firsts else kern
t0 = kern[0][0]
t1 = max(k[1] for k in kern)
out = [f"# one replayed step: {len(kern)} kernels, {t1 - t0:.1f} us first start -> last end",
       "#  start_us    dur_us  stream  kernel"]
busy = {}
for s, e, sid, name in kern:
    out.append(f"{s - t0:10.1f} {e - s:9.1f} {sid:7d}  {name[:110]}")
    busy[sid] = busy.get(sid, 0.0) + (e - s)
main = max(busy, key=lambda k: sum(1 for q in kern if q[2] == k))
gaps, last = [], None
for s, e, sid, name in kern:
    if sid != main:
        continue
    if last is not None and s - last[0] > 1.0:
        gaps.append((s - last[0], last[1], name))
    last = (e, name)
out.append("# busy us per stream: " + ", ".join(f"{k}: {v:.1f}" for k, v in sorted(busy.items())))
out.append(f"# main stream {main}: idle gaps > 1 us: {len(gaps)}, total {sum(g[0] for g in gaps):.1f} us")
for g, a, b in sorted(gaps, reverse=True)[:15]:
    out.append(f"#   {g:7.1f} us  after {a[:60]}  before {b[:60]}")
text = "\n".join(out)
print(text)
if len(sys.argv) > 1:
    Path(sys.argv[1]).write_text(text + "\n")
