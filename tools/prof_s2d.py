"""Time pc_space_to_depth on the AlexNet input (bf16 and fp32 sources)."""
import sys
import torch
sys.path.insert(0, __file__.rsplit("/tools", 1)[0])
from paper_1312_5853_b200 import _lib as L
lib = L.lib(); st = torch.cuda.current_stream().cuda_stream
B, C, H, W, s, p = 256, 3, 227, 227, 4, 0
Hs = (H + 2 * p + s - 1) // s
out = torch.empty(B * Hs * Hs * 64, dtype=torch.bfloat16, device="cuda")
for dt, pc in ((torch.bfloat16, L.PC_BF16), (torch.float32, L.PC_FP32)):
    x = torch.randn(B, C, H, W, device="cuda").to(dt)
    f = lambda: lib.call("pc_space_to_depth", B, C, H, W, s, p, 64, x.data_ptr(), pc, out.data_ptr(), st)
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): f()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    byts = x.numel() * x.element_size() + out.numel() * 2
    print(f"s2d {dt}: {ms*1e3:.1f} us {byts/ms/1e6:.0f} GB/s")
