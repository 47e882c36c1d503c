"""AlexNet max-pool forward / backward (bf16, B=256) through the C ABI, timed back to
back (20 reps) and usable under ncu: python tools/prof_pool.py [H C [mask|nomask|bias]]
(pool1 = 55 96, pool2 = 27 256, pool5 = 13 256; the step's backward has no mask —
the ReLU decision is folded into the argmax — and pools 2 and 5 reduce the bias)."""
import sys, ctypes as C
import torch
sys.path.insert(0, __file__.rsplit("/tools", 1)[0])
from paper_1312_5853_b200 import _lib as L
B, H, Cc = 256, int(sys.argv[1]) if len(sys.argv) > 1 else 55, int(sys.argv[2]) if len(sys.argv) > 2 else 96
mode = sys.argv[3] if len(sys.argv) > 3 else "nomask"
Ho = (H - 3) // 2 + 1
dev = torch.device("cuda"); lib = L.lib(); st = torch.cuda.current_stream().cuda_stream
x = torch.randn(B * H * H * Cc, device=dev).relu().bfloat16()
y = torch.empty(B * Ho * Ho * Cc, device=dev, dtype=torch.bfloat16)
arg = torch.empty(B * Ho * Ho * Cc, device=dev, dtype=torch.uint8)
gy = torch.randn(B * Ho * Ho * Cc, device=dev).bfloat16()
gx = torch.empty_like(x)
gb = torch.empty(Cc, device=dev)
wsn = int(lib.raw("pc_maxpool_backward_bias_workspace")(Cc))
ws = torch.empty(max(wsn, 16), dtype=torch.uint8, device=dev)
mask = x.data_ptr() if mode == "mask" else None
def fwd(): lib.call("pc_maxpool_forward", B, H, H, Cc, 3, 2, x.data_ptr(), y.data_ptr(), arg.data_ptr(), L.PC_BF16, st)
def bwd():
    if mode == "bias":
        lib.call("pc_maxpool_backward_bias", B, H, H, Cc, 3, 2, gy.data_ptr(), arg.data_ptr(), None, gx.data_ptr(),
                 L.PC_BF16, gb.data_ptr(), ws.data_ptr(), ws.numel(), st)
    else:
        lib.call("pc_maxpool_backward", B, H, H, Cc, 3, 2, gy.data_ptr(), arg.data_ptr(), mask, gx.data_ptr(),
                 L.PC_BF16, st)
bwd_bytes = gy.numel() * 3 + x.numel() * (4 if mode == "mask" else 2)
for nm, fn, byts in (("fwd", fwd, x.numel() * 2 + y.numel() * 3), ("bwd", bwd, bwd_bytes)):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): fn()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    print(f"pool H={H} C={Cc} {mode} {nm}: {ms*1e3:7.1f} us  {byts/ms/1e6:7.1f} GB/s (min traffic {byts/1e6:.1f} MB)")
