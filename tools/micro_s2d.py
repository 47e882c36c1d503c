"""Microbenchmark of the input layer's space-to-depth (AlexNet-227 b256) per
source type: python tools/micro_s2d.py (PC_S2D_ROWS=0 for the per-block kernel)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1312_5853_b200 import _lib as L  # noqa: E402

lib = L.lib()
B, C, H, W, s, p = 256, 3, 227, 227, 4, 0
Hs = (H + 2 * p + s - 1) // s
dst = torch.empty(B * Hs * Hs * 64, dtype=torch.bfloat16, device="cuda")
flush = torch.zeros(128 << 20, dtype=torch.int32, device="cuda")   # 512 MB, read between runs:
# evicts L2 with clean lines (a write flush would leave dirty lines to drain inside the timed kernel)
st = torch.cuda.current_stream()
for name, dt, prec in (("bf16", torch.bfloat16, L.PC_BF16), ("f32", torch.float32, L.PC_FP32),
                       ("f64", torch.float64, L.PC_FP64)):
    x = torch.randn(B, C, H, W, device="cuda").to(dt)
    ts = []
    for it in range(12):
        flush.max()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        lib.call("pc_space_to_depth_ex", B, C, H, W, s, p, 64, x.data_ptr(), prec, 63, dst.data_ptr(), st.cuda_stream)
        b.record()
        torch.cuda.synchronize()
        if it >= 2:
            ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    nbytes = x.numel() * x.element_size() + dst.numel() * 2
    print(f"{name}: {ts[len(ts) // 2]:.1f} us  {nbytes / ts[len(ts) // 2] / 1e3:.0f} GB/s")
