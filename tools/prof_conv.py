"""Run one AlexNet conv layer's fwd / dgrad / wgrad (bf16, B=256) through the C ABI,
timed with CUDA events; used for ncu captures of single kernels."""
import sys, ctypes as C
import torch
sys.path.insert(0, __file__.rsplit("/tools", 1)[0])
from paper_1312_5853_b200 import _lib as L

LAYERS = {  # name: (C, H, N, k, s, p)
    "L0": (64, 57, 96, 3, 1, 0), "L3": (96, 27, 256, 5, 1, 2), "L6": (256, 13, 384, 3, 1, 1),
    "L8": (384, 13, 384, 3, 1, 1), "L10": (384, 13, 256, 3, 1, 1)}
name = sys.argv[1] if len(sys.argv) > 1 else "L3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
B = 256
c, h, n, k, s, p = LAYERS[name]
ho = (h + 2 * p - k) // s + 1
g = L.ConvGeom(B, h, h, c, n, k, s, p, ho, ho, c, 0)
dev = torch.device("cuda")
x = torch.randn(B * h * h * c, device=dev).bfloat16()
w = (torch.randn(n * k * k * c, device=dev) * 0.05).bfloat16()
bias = torch.zeros(n, device=dev)
y = torch.empty(B * ho * ho * n, device=dev, dtype=torch.bfloat16)
gy = torch.randn(B * ho * ho * n, device=dev).bfloat16()
gx = torch.empty_like(x)
gw = torch.empty(n * k * k * c, device=dev)
gb = torch.empty(n, device=dev)
lib = L.lib()
wsb = lib.raw("pc_conv2d_backward_workspace")(C.byref(g), L.PC_BF16)
ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream().cuda_stream
flops = 2 * B * ho * ho * n * c * k * k
import os
FWD_FLAGS = 1 | (L.PC_ZERO_TAIL16 if os.environ.get("PROF_ZERO_TAIL") == "1" else 0)   # PC_RELU (+ zero tail)
def fwd(): lib.call("pc_conv2d_forward", C.byref(g), x.data_ptr(), w.data_ptr(), bias.data_ptr(), y.data_ptr(), L.PC_BF16, FWD_FLAGS, st)
def dgrad(): lib.call("pc_conv2d_backward", C.byref(g), x.data_ptr(), w.data_ptr(), gy.data_ptr(), gx.data_ptr(), None, gw.data_ptr(), gb.data_ptr(), L.PC_BF16, L.PC_WANT_DX, ws.data_ptr(), wsb, st)
def wgrad(): lib.call("pc_conv2d_backward", C.byref(g), x.data_ptr(), w.data_ptr(), gy.data_ptr(), gx.data_ptr(), None, gw.data_ptr(), gb.data_ptr(), L.PC_BF16, L.PC_WANT_DW, ws.data_ptr(), wsb, st)
for fn_name, fn in (("fwd", fwd), ("dgrad", dgrad), ("wgrad", wgrad)):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    print(f"{name} {fn_name}: {ms*1e3:8.1f} us  {flops/ms/1e9:7.1f} TFLOP/s")
