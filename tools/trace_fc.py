"""Trace the plain 8192^3 GEMM (pc_fc_forward) per tile, like tools/trace_gemm.py."""
import sys, ctypes as C
import numpy as np
import torch
sys.path.insert(0, __file__.rsplit("/tools", 1)[0])
from paper_1312_5853_b200 import _lib as L
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
dev = torch.device("cuda"); lib = L.lib(); st = torch.cuda.current_stream().cuda_stream
x = torch.randn(n * n, device=dev).bfloat16(); w = torch.randn(n * n, device=dev).bfloat16()
bias = torch.zeros(n, device=dev); y = torch.empty(n * n, device=dev, dtype=torch.bfloat16)
xm = L.Mat(x.data_ptr(), n, n, 0)
def run(): lib.call("pc_fc_forward", n, n, n, C.byref(xm), w.data_ptr(), bias.data_ptr(), y.data_ptr(), L.PC_BF16, 0, st)
run(); torch.cuda.synchronize()
tr = torch.zeros(160 * 64 * 16, dtype=torch.int64, device=dev)
lib.dll.pc_debug_trace_gemm(C.c_void_p(tr.data_ptr())); run(); torch.cuda.synchronize(); lib.dll.pc_debug_trace_gemm(None)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); run(); b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b)
T = tr.view(160, 64, 16).cpu().numpy().astype(np.float64)
rows = []
for i in range(148):
    t = T[i][T[i][:, 4] > 0]
    if len(t):
        t2 = t - T[i][0, 2]; t2[:, 8:12] = t[:, 8:12]; rows.append(t2)
allr = np.concatenate(rows)
med = lambda v: float(np.median(v))
print(f"fc {n}^3: {ms*1e3:.1f} us {2*n**3/ms/1e9:.1f} TFLOP/s; median per tile: mma_issue {med(allr[:,4]-allr[:,7]):.0f} "
      f"wait_acc {med(allr[:,3]-allr[:,2]):.0f} epilogue {med(allr[:,6]-allr[:,5]):.0f} prod {med(allr[:,1]-allr[:,0]):.0f}; prod empty-wait {med(allr[:,8]):.0f} tma-issue {med(allr[:,9]):.0f} mma full-wait {med(allr[:,10]):.0f} mma-issue {med(allr[:,11]):.0f}")
