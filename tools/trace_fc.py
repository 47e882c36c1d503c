"""Per-tile timeline of the FC GEMMs (clock64 stamps via pc_debug_trace_gemm).
  python tools/trace_fc.py M N K [fwd|dgrad]"""
import sys, ctypes as C
import numpy as np
import torch
sys.path.insert(0, __file__.rsplit("/tools", 1)[0])
from paper_1312_5853_b200 import _lib as L
M, N, K = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (8192, 8192, 8192)
which = sys.argv[4] if len(sys.argv) > 4 else "fwd"
dev = torch.device("cuda"); lib = L.lib(); st = torch.cuda.current_stream().cuda_stream
if which == "fwd":       # y[M][N] = x[M][K] W[N][K]^T
    x = torch.randn(M * K, device=dev).bfloat16(); w = torch.randn(N * K, device=dev).bfloat16()
    y = torch.empty(M * N, device=dev, dtype=torch.bfloat16); bias = torch.zeros(N, device=dev)
    xm = L.Mat(x.data_ptr(), K, K, 0)
    wsb = int(lib.raw("pc_fc_forward_workspace")(M, K, N, L.PC_BF16))
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device=dev)
    def run(): lib.call("pc_fc_forward_ex", M, K, N, C.byref(xm), w.data_ptr(), bias.data_ptr(), y.data_ptr(), L.PC_BF16, 0, ws.data_ptr(), wsb, st)
else:                    # gx[M][N] = gy[M][K] W[K][N]   (fc dgrad: B=M, D=N, U=K)
    gy = torch.randn(M * K, device=dev).bfloat16(); w = torch.randn(K * N, device=dev).bfloat16()
    gx = torch.empty(M * N, device=dev, dtype=torch.bfloat16); x = torch.empty_like(gx)
    gw = torch.empty(K * N, device=dev); gb = torch.empty(K, device=dev)
    xm, gm = L.Mat(x.data_ptr(), N, N, 0), L.Mat(gx.data_ptr(), N, N, 0)
    wsb = int(lib.raw("pc_fc_backward_workspace")(M, N, K, L.PC_BF16))
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device=dev)
    def run(): lib.call("pc_fc_backward", M, N, K, C.byref(xm), w.data_ptr(), gy.data_ptr(), C.byref(gm), None, gw.data_ptr(), gb.data_ptr(), L.PC_BF16, L.PC_WANT_DX, ws.data_ptr(), wsb, st)
run(); torch.cuda.synchronize()
tr = torch.zeros(160 * 64 * 16, dtype=torch.int64, device=dev)
lib.dll.pc_debug_trace_gemm(C.c_void_p(tr.data_ptr())); run(); torch.cuda.synchronize(); lib.dll.pc_debug_trace_gemm(None)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): run()
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 10
T = tr.view(160, 64, 16).cpu().numpy().astype(np.float64)
rows = []
for i in range(160):
    t = T[i][T[i][:, 4] > 0]
    if len(t):
        t2 = t - T[i][0, 2]; t2[:, 8:12] = t[:, 8:12]; rows.append(t2)
allr = np.concatenate(rows)
med = lambda v: float(np.median(v))
print(f"{which} M={M} N={N} K={K}: {ms*1e3:.1f} us {2*M*N*K/ms/1e9:.1f} TFLOP/s (incl. split-K reduction); CTAs {len(rows)}")
print(f"  median per tile: first data {med(allr[:,7]-allr[:,3]):.0f} mma_issue {med(allr[:,4]-allr[:,7]):.0f} "
      f"wait_acc {med(allr[:,3]-allr[:,2]):.0f} epilogue {med(allr[:,6]-allr[:,5]):.0f} prod {med(allr[:,1]-allr[:,0]):.0f}; "
      f"prod empty-wait {med(allr[:,8]):.0f} tma-issue {med(allr[:,9]):.0f} mma full-wait {med(allr[:,10]):.0f} mma-issue {med(allr[:,11]):.0f}")
print(f"  CTA span median {med([r[-1,6] for r in rows]):.0f} max {max(r[-1,6] for r in rows):.0f} cycles")
