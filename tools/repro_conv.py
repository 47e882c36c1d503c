"""Debug: one bf16 conv forward + backward through pc_conv2d_* at a given geometry
(argv: B C H W N k s p), each pass synchronised and reported."""
import sys, ctypes as C
import torch
sys.path.insert(0, __file__.rsplit("/tools", 1)[0])
from paper_1312_5853_b200 import _lib as L
B, Ci, H, W, N, k, s, p = (int(v) for v in sys.argv[1:9])
Ho, Wo = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
g = L.ConvGeom(B, H, W, Ci, N, k, s, p, Ho, Wo, Ci, 0)
dev = torch.device("cuda"); lib = L.lib(); st = torch.cuda.current_stream().cuda_stream
x = torch.randn(B * H * W * Ci, device=dev).bfloat16(); w = (torch.randn(N * k * k * Ci, device=dev) * .05).bfloat16()
bias = torch.zeros(N, device=dev); y = torch.empty(B * Ho * Wo * N, device=dev, dtype=torch.bfloat16)
gy = torch.randn(B * Ho * Wo * N, device=dev).bfloat16(); gx = torch.empty_like(x)
gw = torch.empty(N * k * k * Ci, device=dev); gb = torch.empty(N, device=dev)
wsb = lib.raw("pc_conv2d_backward_workspace")(C.byref(g), L.PC_BF16)
ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
for name, f in (("fwd", lambda: lib.call("pc_conv2d_forward", C.byref(g), x.data_ptr(), w.data_ptr(), bias.data_ptr(), y.data_ptr(), L.PC_BF16, 1, st)),
                ("dgrad", lambda: lib.call("pc_conv2d_backward", C.byref(g), x.data_ptr(), w.data_ptr(), gy.data_ptr(), gx.data_ptr(), None, gw.data_ptr(), gb.data_ptr(), L.PC_BF16, L.PC_WANT_DX, ws.data_ptr(), wsb, st)),
                ("wgrad", lambda: lib.call("pc_conv2d_backward", C.byref(g), x.data_ptr(), w.data_ptr(), gy.data_ptr(), gx.data_ptr(), None, gw.data_ptr(), gb.data_ptr(), L.PC_BF16, L.PC_WANT_DW, ws.data_ptr(), wsb, st))):
    f(); torch.cuda.synchronize(); print("ok", name, flush=True)
