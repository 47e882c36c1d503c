"""AlexNet pool1 (L2) forward / backward (bf16, B=256) through the C ABI, for ncu."""
import sys, ctypes as C
import torch
sys.path.insert(0, __file__.rsplit("/tools", 1)[0])
from paper_1312_5853_b200 import _lib as L
B, H, Cc = 256, int(sys.argv[1]) if len(sys.argv) > 1 else 55, int(sys.argv[2]) if len(sys.argv) > 2 else 96
Ho = (H - 3) // 2 + 1
dev = torch.device("cuda"); lib = L.lib(); st = torch.cuda.current_stream().cuda_stream
x = torch.randn(B * H * H * Cc, device=dev).relu().bfloat16()
y = torch.empty(B * Ho * Ho * Cc, device=dev, dtype=torch.bfloat16)
arg = torch.empty(B * Ho * Ho * Cc, device=dev, dtype=torch.uint8)
gy = torch.randn(B * Ho * Ho * Cc, device=dev).bfloat16()
gx = torch.empty_like(x)
def fwd(): lib.call("pc_maxpool_forward", B, H, H, Cc, 3, 2, x.data_ptr(), y.data_ptr(), arg.data_ptr(), L.PC_BF16, st)
def bwd(): lib.call("pc_maxpool_backward", B, H, H, Cc, 3, 2, gy.data_ptr(), arg.data_ptr(), x.data_ptr(), gx.data_ptr(), L.PC_BF16, st)
for nm, fn, byts in (("fwd", fwd, x.numel() * 2 + y.numel() * 3), ("bwd", bwd, gy.numel() * 3 + x.numel() * 4)):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): fn()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    print(f"pool H={H} C={Cc} {nm}: {ms*1e3:7.1f} us  {byts/ms/1e6:7.1f} GB/s (min traffic {byts/1e6:.1f} MB)")
