"""Per-tile timeline of one tensor-core GEMM launch (clock64 stamps, debug build
hook pc_debug_trace_gemm): where does a tile's time go — waiting for the
accumulator, for the first operand stage, issuing the MMAs, the epilogue?"""
import sys, ctypes as C
import numpy as np
import torch
sys.path.insert(0, __file__.rsplit("/tools", 1)[0])
from paper_1312_5853_b200 import _lib as L
LAYERS = {"L0": (64, 57, 96, 3, 1, 0), "L3": (96, 27, 256, 5, 1, 2), "L6": (256, 13, 384, 3, 1, 1),
          "L8": (384, 13, 384, 3, 1, 1), "L10": (384, 13, 256, 3, 1, 1)}
name = sys.argv[1] if len(sys.argv) > 1 else "L8"
which = sys.argv[2] if len(sys.argv) > 2 else "fwd"
B = 256
c, h, n, k, s, p = LAYERS[name]
ho = (h + 2 * p - k) // s + 1
dev = torch.device("cuda"); lib = L.lib(); st = torch.cuda.current_stream().cuda_stream
x = torch.randn(B * h * h * c, device=dev).bfloat16(); w = (torch.randn(n * k * k * c, device=dev) * .05).bfloat16()
bias = torch.zeros(n, device=dev); y = torch.empty(B * ho * ho * n, device=dev, dtype=torch.bfloat16)
gy = torch.randn(B * ho * ho * n, device=dev).bfloat16(); gx = torch.empty_like(x)
gw = torch.empty(n * k * k * c, device=dev); gb = torch.empty(n, device=dev)
g = L.ConvGeom(B, h, h, c, n, k, s, p, ho, ho, c, 0)
wsb = lib.raw("pc_conv2d_backward_workspace")(C.byref(g), L.PC_BF16)
ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
def run():
    if which == "fwd":
        lib.call("pc_conv2d_forward", C.byref(g), x.data_ptr(), w.data_ptr(), bias.data_ptr(), y.data_ptr(), L.PC_BF16, 1, st)
    elif which == "dgrad":
        lib.call("pc_conv2d_backward", C.byref(g), x.data_ptr(), w.data_ptr(), gy.data_ptr(), gx.data_ptr(), None, gw.data_ptr(), gb.data_ptr(), L.PC_BF16, L.PC_WANT_DX, ws.data_ptr(), wsb, st)
    else:
        lib.call("pc_conv2d_backward", C.byref(g), x.data_ptr(), w.data_ptr(), gy.data_ptr(), gx.data_ptr(), None, gw.data_ptr(), gb.data_ptr(), L.PC_BF16, L.PC_WANT_DW, ws.data_ptr(), wsb, st)
run(); torch.cuda.synchronize()
tr = torch.zeros(160 * 64 * 16, dtype=torch.int64, device=dev)
lib.dll.pc_debug_trace_gemm(C.c_void_p(tr.data_ptr()))
run(); torch.cuda.synchronize()
lib.dll.pc_debug_trace_gemm(None)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); run(); b.record(); torch.cuda.synchronize()
T = tr.view(160, 64, 16).cpu().numpy().astype(np.float64)
print(f"{name} {which}: {a.elapsed_time(b)*1e3:.1f} us (untraced)")
rows = []
for blk in range(148):
    t = T[blk]
    valid = t[:, 4] > 0
    if not valid.any():
        continue
    t = t[valid]
    base = t[0, 2]
    t2 = t - base
    t2[:, 8:12] = t[:, 8:12]
    rows.append(t2)
    if blk < 3:
        print(f"CTA {blk}: tiles {len(t)}")
        for i, r in enumerate(t[:6]):
            r = r - base
            print(f"  tile {i}: prod [{r[0]:8.0f},{r[1]:8.0f}] mma wait_acc {r[2]:8.0f}->{r[3]:8.0f} first_data {r[7]:8.0f} issued {r[4]:8.0f} | epi {r[5]:8.0f}->{r[6]:8.0f}")
allr = np.concatenate(rows)
def med(x): return float(np.median(x))
def base_fix(a): return 0
print("median cycles per tile: mma_issue(first data->last commit) %.0f | wait_first_data %.0f | wait_acc %.0f | epilogue %.0f | epi_lag(after commit) %.0f | prod_issue %.0f" % (
    med(allr[:, 4] - allr[:, 7]), med(allr[:, 7] - allr[:, 3]), med(allr[:, 3] - allr[:, 2]),
    med(allr[:, 6] - allr[:, 5]), med(allr[:, 5] - allr[:, 4]), med(allr[:, 1] - allr[:, 0])))
print("median per tile: producer empty-wait %.0f tma-issue %.0f | mma full-wait %.0f mma-issue %.0f" % (
    med(allr[:, 8] + base_fix(allr)), med(allr[:, 9]), med(allr[:, 10]), med(allr[:, 11])))
tot = [r[-1, 6] for r in rows]
print("CTA span cycles: median %.0f max %.0f; tiles per CTA %s" % (np.median(tot), np.max(tot), sorted(set(len(r) for r in rows))))
ext = allr[:, 12:16]
if (ext > 0).any():
    d = [med(allr[:, 12] - allr[:, 6])] + [med(allr[:, 12 + i] - allr[:, 11 + i]) for i in range(1, 4)]
    print("epilogue tail (slots 12-15, deltas from the release): %s" % " | ".join("%.0f" % x for x in d))
