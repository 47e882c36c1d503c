"""Summarise ncu output for profiles/ (run here, no GPU needed).

  python tools/summarize_ncu.py launches <launches.csv> [per_step_launches]
      per-launch device times (ncu --metrics gpu__time_duration.sum): the last
      step's launches in order, and each kernel family's share of that step.
  python tools/summarize_ncu.py full <report.ncu-rep>
      key counters per captured launch (duration, DRAM bytes, tensor-pipe and
      L2 utilisation) from an `ncu --set full` capture.
"""

import csv
import io
import subprocess
import sys
from collections import defaultdict


def _rows(text):
    rows = list(csv.reader(io.StringIO(text)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    return rows[hi], rows[hi + 1:]


def launches(path, per_step=None):
    h, data = _rows(open(path).read())
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}
    seq = [(r[ki], float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3)) for r in data]
    if per_step:
        seq = seq[-per_step:]
    total = sum(v for _, v in seq)
    print(f"# {len(seq)} launches, {total:.1f} us summed device time (cold-cache, serialised)")
    print("# order  us      kernel")
    for i, (k, v) in enumerate(seq):
        print(f"{i:4d} {v:9.1f}  {k[:110]}")
    fam = defaultdict(float)
    for k, v in seq:
        fam[k.split("(")[0].replace("void ", "")] += v
    print("\n# share by kernel family")
    for k, v in sorted(fam.items(), key=lambda kv: -kv[1]):
        print(f"{100 * v / total:6.1f}%  {v:9.1f} us  {k}")


FULL_KEYS = [
    ("gpu__time_duration.sum", "us"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "regs"),
]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, data = rows[0], rows[1], rows[2:]
    ki = h.index("Kernel Name")
    cols = [(h.index(k) if k in h else None, lab, units[h.index(k)] if k in h else "") for k, lab in FULL_KEYS]
    print("kernel | " + " | ".join(f"{lab} [{u}]" for _, lab, u in cols))
    for r in data:
        vals = [r[i] if i is not None else "-" for i, _, _ in cols]
        print(f"{r[ki][:60]} | " + " | ".join(vals))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else None)
    else:
        full(sys.argv[2])
