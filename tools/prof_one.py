"""Single launches for ncu: plain 8192^3 GEMM (ours, then cuBLAS), AlexNet conv4 (L8) forward, L0 (s2d) forward."""
import sys, ctypes as C
import torch
sys.path.insert(0, __file__.rsplit("/tools", 1)[0])
from paper_1312_5853_b200 import _lib as L
dev = torch.device("cuda"); lib = L.lib(); st = torch.cuda.current_stream().cuda_stream
n = 8192
x = torch.randn(n * n, device=dev).bfloat16(); w = torch.randn(n * n, device=dev).bfloat16()
bias = torch.zeros(n, device=dev); y = torch.empty(n * n, device=dev, dtype=torch.bfloat16)
xm = L.Mat(x.data_ptr(), n, n, 0)
lib.call("pc_fc_forward", n, n, n, C.byref(xm), w.data_ptr(), bias.data_ptr(), y.data_ptr(), L.PC_BF16, 0, st)
torch.matmul(x.view(n, n), w.view(n, n).t())
for (c, h, nn, k, s, p) in ((384, 13, 384, 3, 1, 1), (64, 57, 96, 3, 1, 0)):
    B = 256; ho = (h + 2 * p - k) // s + 1
    xx = torch.randn(B * h * h * c, device=dev).bfloat16(); ww = torch.randn(nn * k * k * c, device=dev).bfloat16()
    yy = torch.empty(B * ho * ho * nn, device=dev, dtype=torch.bfloat16); bb = torch.zeros(nn, device=dev)
    g = L.ConvGeom(B, h, h, c, nn, k, s, p, ho, ho, c, 0)
    lib.call("pc_conv2d_forward", C.byref(g), xx.data_ptr(), ww.data_ptr(), bb.data_ptr(), yy.data_ptr(), L.PC_BF16, 1, st)
torch.cuda.synchronize()
print("ok")
