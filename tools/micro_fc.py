"""Microbenchmark of the small-batch FC forward / data gradient (AlexNet fc6-8 at
b256, bf16): python tools/micro_fc.py  (PC_FC_CLUSTER=0: the two-kernel split-K path)."""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1312_5853_b200 import _lib as L  # noqa: E402

lib = L.lib()
st = torch.cuda.current_stream()
flush = torch.zeros(128 << 20, dtype=torch.int32, device="cuda")


def graph_time(fn, reps=10):
    """Device time per call of fn, launched from a CUDA graph (no host gaps)."""
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    ts = []
    for it in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / reps)
    ts.sort()
    return ts[len(ts) // 2]


def timeit(fn):
    """(cold: L2 flushed by a 512 MB read before every call, warm: back to back)"""
    t_flush = graph_time(lambda: flush.max())
    return graph_time(lambda: (flush.max(), fn())) - t_flush, graph_time(fn)


B = 256
once = "--once" in sys.argv      # one call of each (for ncu)
for name, D, U in (("fc6", 9216, 4096), ("fc7", 4096, 4096), ("fc8", 4096, 1000)):
    if len(sys.argv) > 1 and sys.argv[1].startswith("fc") and sys.argv[1] != name:
        continue
    x = torch.randn(B, D, device="cuda").bfloat16()
    w = (torch.randn(U, D, device="cuda") * D ** -0.5).bfloat16()
    bias = torch.randn(U, device="cuda")
    y = torch.empty(B, U, device="cuda", dtype=torch.bfloat16)
    gy = torch.randn(B, U, device="cuda").bfloat16()
    gx = torch.empty(B, D, device="cuda", dtype=torch.bfloat16)
    wsf = int(lib.raw("pc_fc_forward_workspace")(B, D, U, L.PC_BF16))
    wsb = int(lib.raw("pc_fc_backward_workspace")(B, D, U, L.PC_BF16))
    ws = torch.empty(max(wsf, wsb, 16), dtype=torch.uint8, device="cuda")
    xm, gm = L.Mat(x.data_ptr(), D, D, 0), L.Mat(gx.data_ptr(), D, D, 0)

    def fwd():
        lib.call("pc_fc_forward_ex", B, D, U, C.byref(xm), w.data_ptr(), bias.data_ptr(), y.data_ptr(), L.PC_BF16,
                 L.PC_RELU, ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream)

    def dgrad():
        lib.call("pc_fc_backward", B, D, U, C.byref(xm), w.data_ptr(), gy.data_ptr(), C.byref(gm), None,
                 None, None, L.PC_BF16, L.PC_WANT_DX, ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream)

    if once:
        fwd()
        dgrad()
        torch.cuda.synchronize()
        continue
    (tf, tfw), (td, tdw) = timeit(fwd), timeit(dgrad)
    wb = U * D * 2
    print(f"{name}: forward {tf:.1f} us cold ({wb / tf / 1e3:.0f} GB/s weights), {tfw:.1f} warm;  "
          f"dgrad {td:.1f} us cold ({wb / td / 1e3:.0f} GB/s), {tdw:.1f} warm")
