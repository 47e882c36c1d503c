"""Time the FC entry points on a square problem: fwd (K-major A,B), dgrad (K-major A,
MN-major B) and wgrad (MN-major A,B), to isolate operand-major effects."""
import sys, ctypes as C
import torch
sys.path.insert(0, __file__.rsplit("/tools", 1)[0])
from paper_1312_5853_b200 import _lib as L
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = 10
dev = torch.device("cuda")
B = D = U = n
x = torch.randn(B * D, device=dev).bfloat16()
w = (torch.randn(U * D, device=dev) * 0.02).bfloat16()
bias = torch.zeros(U, device=dev)
y = torch.empty(B * U, device=dev, dtype=torch.bfloat16)
gy = torch.randn(B * U, device=dev).bfloat16()
gx = torch.empty_like(x)
gw = torch.empty(U * D, device=dev)
gb = torch.empty(U, device=dev)
lib = L.lib()
wsb = int(lib.raw("pc_fc_backward_workspace")(B, D, U, L.PC_BF16))
ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream().cuda_stream
xm, gm = L.Mat(x.data_ptr(), D, D, 0), L.Mat(gx.data_ptr(), D, D, 0)
fl = 2.0 * B * D * U
def fwd(): lib.call("pc_fc_forward", B, D, U, C.byref(xm), w.data_ptr(), bias.data_ptr(), y.data_ptr(), L.PC_BF16, 0, st)
def dgrad(): lib.call("pc_fc_backward", B, D, U, C.byref(xm), w.data_ptr(), gy.data_ptr(), C.byref(gm), None, gw.data_ptr(), gb.data_ptr(), L.PC_BF16, L.PC_WANT_DX, ws.data_ptr(), wsb, st)
def wgrad(): lib.call("pc_fc_backward", B, D, U, C.byref(xm), w.data_ptr(), gy.data_ptr(), C.byref(gm), None, gw.data_ptr(), gb.data_ptr(), L.PC_BF16, L.PC_WANT_DW, ws.data_ptr(), wsb, st)
for name, fn in (("fwd K/K", fwd), ("dgrad K/MN", dgrad), ("wgrad MN/MN", wgrad)):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    print(f"n={n} {name:12s} {ms*1e3:8.1f} us {fl/ms/1e9:7.1f} TFLOP/s")
# cuBLAS reference on the same shape (library GEMM, for calibration only)
xa, wa = x.view(B, D), w.view(U, D)
torch.matmul(xa, wa.t()); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps): torch.matmul(xa, wa.t())
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
print(f"n={n} {'cuBLAS':12s} {ms*1e3:8.1f} us {fl/ms/1e9:7.1f} TFLOP/s")
