"""Does a side-stream SGD update overlap a persistent tensor-core GEMM?
Times conv2 (layer 3) data+weight gradient GEMMs alone, the FC-head-sized SGD
alone (full grid and background grid), and both issued on two streams."""
import sys, ctypes as C
import torch
sys.path.insert(0, __file__.rsplit("/tools", 1)[0])
from paper_1312_5853_b200 import _lib as L

dev = torch.device("cuda"); lib = L.lib()
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
B, c, h, n, k, s, p = 256, 256, 13, 384, 3, 1, 1
ho = (h + 2 * p - k) // s + 1
x = torch.randn(B * h * h * c, device=dev).bfloat16(); w = (torch.randn(n * k * k * c, device=dev) * .05).bfloat16()
gy = torch.randn(B * ho * ho * n, device=dev).bfloat16(); gx = torch.empty_like(x)
gw = torch.empty(n * k * k * c, device=dev); gb = torch.empty(n, device=dev)
g = L.ConvGeom(B, h, h, c, n, k, s, p, ho, ho, c, 0)
wsb = lib.raw("pc_conv2d_backward_workspace")(C.byref(g), L.PC_BF16)
ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
NP = 58_631_144
P, V, G = (torch.randn(NP, device=dev) for _ in range(3))
tab = L.SgdTensor(P.data_ptr(), V.data_ptr(), G.data_ptr(), None, NP)
tdev = torch.frombuffer(bytearray(bytes(tab)), dtype=torch.uint8).to(dev)


def gemms(st):
    for _ in range(4):
        lib.call("pc_conv2d_backward", C.byref(g), x.data_ptr(), w.data_ptr(), gy.data_ptr(), gx.data_ptr(), None,
                 gw.data_ptr(), gb.data_ptr(), L.PC_BF16, L.PC_WANT_DX | L.PC_WANT_DW, ws.data_ptr(), wsb,
                 st.cuda_stream)


def sgd(st, ctas):
    lib.call("pc_sgd_step_ex", 1, tdev.data_ptr(), NP, 1e-4, 0.9, 5e-4, ctas, st.cuda_stream)


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    a.record(cur)
    sa.wait_stream(cur); sb.wait_stream(cur)
    fn()
    cur.wait_stream(sa); cur.wait_stream(sb)
    b.record(cur)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3


t_g = timed(lambda: gemms(sa))
for ctas in (0, 1, 2, 3, 4):
    t_s = timed(lambda: sgd(sb, ctas))
    t_both = timed(lambda: (gemms(sa), sgd(sb, ctas)))
    t_both2 = timed(lambda: (sgd(sb, ctas), gemms(sa)))
    print(f"ctas/SM {ctas}: gemms {t_g:7.1f} us  sgd {t_s:7.1f} us  both(gemm first) {t_both:7.1f}  "
          f"both(sgd first) {t_both2:7.1f}  serial {t_g + t_s:7.1f}")
