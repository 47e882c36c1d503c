"""profiles/ table of one step's launches from an ncu --csv metrics log:
python tools/launch_table.py launches.csv out.txt"""
import collections
import csv
import sys

T = {"ns": 1e-3, "us": 1, "ms": 1e3, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}
B = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path, out_path, peak=6544.0):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui, idi = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = collections.OrderedDict()
    for r in data:
        per.setdefault(r[idi], {"name": r[ki]})[r[mi]] = (float(r[vi].replace(",", "")), r[ui])
    items = list(per.values())
    starts = [i for i, it in enumerate(items) if "s2d_k<" in it["name"] or "s2d_rows_" in it["name"]]
    step = items[starts[-1]:]
    out = ["# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none",
           "# python bench.py --profile-only --steps 1 --warmup 3: the launches of the last profiled step,",
           f"# serialised and cold-cache (shares, not absolute step time). GB/s = DRAM bytes / duration; HBM peak {peak:.0f} GB/s.",
           "#  order      us   DRAM_MB    GB/s  HBM%  tensor%  kernel"]
    tot = 0.0
    fam = collections.defaultdict(float)
    for i, it in enumerate(step):
        t = it["gpu__time_duration.sum"]
        us = t[0] * T[t[1]]
        tot += us
        rd, wr = it["dram__bytes_read.sum"], it["dram__bytes_write.sum"]
        mb = (rd[0] * B[rd[1]] + wr[0] * B[wr[1]]) / 1e6
        tp = it.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", (0.0, ""))[0]
        gbs = mb * 1e3 / us
        out.append(f"{i:6d} {us:8.1f} {mb:9.1f} {gbs:7.0f} {100 * gbs / peak:5.1f} {tp:7.1f}  {it['name'][:100]}")
        fam[it["name"].split("(")[0].replace("void ", "")] += us
    out.append(f"# {len(step)} launches, {tot:.1f} us summed (serialised)")
    out.append("# share by kernel family")
    for k, v in sorted(fam.items(), key=lambda kv: -kv[1]):
        out.append(f"# {100 * v / tot:5.1f}%  {v:8.1f} us  {k[:90]}")
    open(out_path, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
