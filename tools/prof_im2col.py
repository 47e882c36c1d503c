"""Is the TMA im2col operand the limiter? Time a conv layer's forward (A by TMA
im2col) against the plain GEMM of the same M x N x K (A by tiled TMA from a
materialised im2col matrix)."""
import sys, ctypes as C
import torch
sys.path.insert(0, __file__.rsplit("/tools", 1)[0])
from paper_1312_5853_b200 import _lib as L
LAYERS = {"L3": (96, 27, 256, 5, 1, 2), "L6": (256, 13, 384, 3, 1, 1), "L8": (384, 13, 384, 3, 1, 1),
          "L0": (64, 57, 96, 3, 1, 0)}
name = sys.argv[1] if len(sys.argv) > 1 else "L8"
B = 256
c, h, n, k, s, p = LAYERS[name]
ho = (h + 2 * p - k) // s + 1
M, K = B * ho * ho, k * k * c
dev = torch.device("cuda")
lib = L.lib()
st = torch.cuda.current_stream().cuda_stream
x = torch.randn(B * h * h * c, device=dev).bfloat16()
w = (torch.randn(n * K, device=dev) * 0.05).bfloat16()
bias = torch.zeros(n, device=dev)
y = torch.empty(M * n, device=dev, dtype=torch.bfloat16)
g = L.ConvGeom(B, h, h, c, n, k, s, p, ho, ho, c, 0)
A = torch.randn(M * K, device=dev).bfloat16()
am = L.Mat(A.data_ptr(), K, K, 0)
def conv(): lib.call("pc_conv2d_forward", C.byref(g), x.data_ptr(), w.data_ptr(), bias.data_ptr(), y.data_ptr(), L.PC_BF16, 1, st)
def gemm(): lib.call("pc_fc_forward", M, K, n, C.byref(am), w.data_ptr(), bias.data_ptr(), y.data_ptr(), L.PC_BF16, 1, st)
fl = 2.0 * M * n * K
for nm, fn in (("conv(im2col TMA)", conv), ("gemm(tiled TMA)", gemm)):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): fn()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    print(f"{name} {nm:18s} M={M} N={n} K={K}: {ms*1e3:8.1f} us {fl/ms/1e9:7.1f} TFLOP/s")
