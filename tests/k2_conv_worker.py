"""Subprocess for tests/test_gpu_kernels_k2.py: bf16 conv forward + data gradient
on tensor cores at several geometries; the GEMM variant is chosen by PC_K2 (read
once per process). Writes the outputs to the .npz path in argv[1]."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1312_5853_b200 import _lib as L  # noqa: E402

lib = L.lib()
st = torch.cuda.current_stream().cuda_stream
out = {}
for gi, (B, H, C, N, k, pad) in enumerate([(256, 27, 96, 256, 5, 2), (20, 27, 96, 256, 5, 2), (64, 13, 384, 384, 3, 1),
                                            (64, 13, 256, 384, 3, 1), (7, 13, 384, 256, 3, 1)]):
    g = torch.Generator(device="cuda").manual_seed(gi)
    x = torch.randn(B, H, H, C, device="cuda", generator=g).relu().bfloat16()
    w = (torch.randn(N, k, k, C, device="cuda", generator=g) * 0.05).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g)
    Ho = H + 2 * pad - k + 1
    geom = L.ConvGeom(B, H, H, C, N, k, 1, pad, Ho, Ho, C, 0)
    y = torch.empty(B, Ho, Ho, N, device="cuda", dtype=torch.bfloat16)
    import ctypes as Ct
    lib.call("pc_conv2d_forward", Ct.byref(geom), x.data_ptr(), w.data_ptr(), bias.data_ptr(), y.data_ptr(),
             L.PC_BF16, L.PC_RELU, st)
    gy = torch.randn(B, Ho, Ho, N, device="cuda", generator=g).bfloat16()
    gx = torch.empty_like(x)
    ws_n = lib.raw("pc_conv2d_backward_workspace")(Ct.byref(geom), L.PC_BF16)
    ws = torch.empty(max(int(ws_n), 16), dtype=torch.uint8, device="cuda")
    lib.call("pc_conv2d_backward", Ct.byref(geom), x.data_ptr(), w.data_ptr(), gy.data_ptr(), gx.data_ptr(),
             x.data_ptr(), None, None, L.PC_BF16, L.PC_WANT_DX | L.PC_MASK_DX, ws.data_ptr(), ws.numel(), st)
    gx2 = torch.empty_like(x)   # no ReLU mask: the TMA-store epilogue path of the data gradient
    lib.call("pc_conv2d_backward", Ct.byref(geom), x.data_ptr(), w.data_ptr(), gy.data_ptr(), gx2.data_ptr(),
             None, None, None, L.PC_BF16, L.PC_WANT_DX, ws.data_ptr(), ws.numel(), st)
    torch.cuda.synchronize()
    out[f"gx2_{gi}"] = gx2.view(torch.int16).cpu().numpy()
    out[f"y{gi}"] = y.view(torch.int16).cpu().numpy()
    out[f"gx{gi}"] = gx.view(torch.int16).cpu().numpy()
np.savez(sys.argv[1], **out)
