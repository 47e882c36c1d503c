"""Benchmark: AlexNet (batch 256) synchronous-SGD training step on B200.

Metric (BASELINE.json): train images/sec, AlexNet b256 at 1/2/4/8 B200 per
scheme, with the dominant contraction's fraction of the tensor-core roofline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--scheme auto|dp|mp|hybrid] [--precision bf16|fp32]

N=1: plan d1m1, global batch 256. N>1 (torchrun, one rank per GPU):
auto = model parallel d1m2 cross(conv3) at N=2, hybrid d(N/2) x m2 at N=4/8
with 256 images per replica group (the paper's hybrid; weak scaling).
``--scheme dp``: data parallel dN x m1, 256 images per GPU.

``value`` is measured with the batch already resident in HBM (device step
program only); ``e2e`` goes through the public ``hybrid_step`` API with a
pinned host batch: host->device copy, step, and the loss read-back are all
inside the timed region. Both are CUDA-event timed on the launching stream,
barrier + synchronize on both sides, max over ranks. Activations of one
AlexNet b256 step are several GB, far larger than the 126 MB L2, so no
explicit flush is needed between steps.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "train images/sec AlexNet b256 at 1/2/4/8 B200 per scheme; % TC roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scheme", default="auto", choices=["auto", "dp", "mp", "hybrid"])
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--batch", type=int, default=256, help="images per replica group")
    ap.add_argument("--net", default=str(ROOT / "configs" / "alexnet.net"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-input", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--profile-only", action="store_true", help="short run for ncu captures")
    return ap.parse_args()


def choose_plan(n: int, scheme: str, per_group: int):
    from paper_1312_5853_b200.plan import ParallelPlan
    if n == 1:
        return ParallelPlan(1, 1), per_group, "d1m1"
    if scheme == "dp":
        return ParallelPlan(n, 1), per_group * n, f"dp{n}"
    if scheme == "mp" or (scheme == "auto" and n == 2):
        if n != 2:
            raise SystemExit("model parallel runs on 2 GPUs (two columns)")
        return ParallelPlan(1, 2, (6,)), per_group, "mp2-krizhevsky-cross6"
    d = n // 2
    return ParallelPlan(d, 2, (6,)), per_group * d, f"hybrid-d{d}xm2-cross6"


class ClockSampler:
    """nvidia-smi sampling of SM clocks / throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "50",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("bf16_tflops", 1590.0), d.get("bf16_tflops_sustained", 1400.0), d.get("hbm_gbs", 6650.0), \
            "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


def layer_flops(cl, batch: int) -> int:
    from paper_1312_5853_b200.netdef import layer_macs
    return 2 * layer_macs(cl, batch)


def cpu_reference_sample(net, plan, cs, n_images: int, seed: int = 0):
    """The oracle (float64 numpy port of the reference step) on a bounded sample."""
    from oracle.ref_engine import OracleFabric
    from paper_1312_5853_b200.data import synthetic_rows
    from paper_1312_5853_b200.plan import init_dense_params
    idx = np.arange(n_images)
    x, y = synthetic_rows(1000, 1, net.input_shape, seed, idx)
    dense = init_dense_params(net, seed)
    sample_plan = plan if n_images % plan.data_shards == 0 else type(plan)(1, plan.model_columns,
                                                                          plan.cross_layers)
    fab = OracleFabric(net, sample_plan, dense)
    fab.step(x.astype(np.float64), y)           # warm (allocations)
    t0 = time.perf_counter()
    fab.step(x.astype(np.float64), y)
    dt = time.perf_counter() - t0
    return n_images / dt, dt


def run_reference_arm(args, rank: int):
    """--impl reference: the reference's CPU step (float64 oracle port) on the
    host cores, same metric/config, bounded sample per step."""
    if rank != 0:
        return
    from paper_1312_5853_b200.netdef import load_network
    from paper_1312_5853_b200.plan import plan_columnized
    net = load_network(args.net)
    plan, gbatch, label = choose_plan(args.gpus, args.scheme, args.batch)
    cs = plan_columnized(net, plan)
    from oracle.ref_engine import OracleFabric
    from paper_1312_5853_b200.data import synthetic_rows
    from paper_1312_5853_b200.plan import init_dense_params, ParallelPlan
    sample = max(plan.data_shards, 2)
    x, y = synthetic_rows(1000, 1, net.input_shape, 0, np.arange(sample))
    fab = OracleFabric(net, plan if sample % plan.data_shards == 0 else ParallelPlan(1, plan.model_columns,
                                                                                     plan.cross_layers),
                       init_dense_params(net, 0))
    x = x.astype(np.float64)
    for _ in range(max(args.warmup, 0) and 1):
        fab.step(x, y)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fab.step(x, y)
    dt = time.perf_counter() - t0
    v = sample * args.steps / dt
    cores = os.cpu_count()
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "images/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": f"AlexNet-227 {label} step (reference CPU path)",
                                            "global_batch": gbatch, "plan": plan.describe()},
            "cpu_baseline": {"value": v, "unit": "images/s", "cores": cores, "kind": "port",
                             "sample": f"{sample} images per step of the {label} plan, float64 numpy "
                                       f"restatement of parconv (oracle/), BLAS threads = host cores"},
            "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank)
        return
    import torch
    import torch.distributed as dist
    if world > 1:
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE {world}: launch N>1 with torchrun")
    import paper_1312_5853_b200 as P
    from paper_1312_5853_b200 import engine as E
    from paper_1312_5853_b200 import schemes as S
    from paper_1312_5853_b200._lib import lib
    from paper_1312_5853_b200.data import synthetic_rows
    from paper_1312_5853_b200.plan import plan_columnized

    net = P.load_network(args.net)
    plan, gbatch, label = choose_plan(args.gpus, args.scheme, args.batch)
    cs = plan_columnized(net, plan)
    dev = torch.device("cuda", torch.cuda.current_device())
    per_class = max(1, math.ceil(gbatch / 1000))
    from paper_1312_5853_b200 import rng as R
    order = R.permutation(0, 0, 1000 * per_class)[:gbatch]
    xb, yb = synthetic_rows(1000, per_class, net.input_shape, 0, order)
    x_host = torch.from_numpy(xb).pin_memory()
    y_host = torch.from_numpy(yb.astype(np.int32)).pin_memory()
    # e2e input: the batch as the input pipeline hands it over, pinned. bf16 (default)
    # carries exactly the values the device rounds the fp32 images to before conv1.
    x_e2e = x_host.to(torch.bfloat16).pin_memory() if args.e2e_input == "bf16" else x_host

    fab = P.spawn(plan.workers, precision=args.precision)
    # Gaussian std 0.01 (the paper's cited Krizhevsky init, reference SPEC.md:120): the He-normal
    # default diverges to inf within 4 steps on AlexNet at lr 0.01 in the reference as well
    P.setup_workers(fab, plan, cs, P.init_dense_params(net, 0, std=0.01), P.SgdState())
    res = P.hybrid_step(fab, plan, cs, x_e2e, y_host)           # builds engines, first step (resident batch = the pipeline format)
    run = S._runner(fab, plan, cs, gbatch // plan.data_shards)
    stream = torch.cuda.current_stream()
    scale = 1.0 / gbatch

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident throughput ("value")
    for _ in range(max(args.warmup, 3)):
        run.program(scale)
    barrier()
    clocks = ClockSampler(dev.index)
    clocks.start()
    l0, r0 = lib().dll.pc_launch_count(), run.replays
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        run.program(scale)
    e1.record(stream)
    barrier()
    # graph replays launch the captured sequence without passing the C ABI's counter
    launches = lib().dll.pc_launch_count() - l0 + run.graph_launches * (run.replays - r0)
    ms = e0.elapsed_time(e1) / args.steps
    # ---- end to end through the public API (pinned host batch, loss read-back)
    for _ in range(2):
        P.hybrid_step(fab, plan, cs, x_e2e, y_host, meter=False)
    barrier()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    losses = []
    for _ in range(args.steps):
        losses.append(P.hybrid_step(fab, plan, cs, x_e2e, y_host, meter=False).loss)
    e3.record(stream)
    barrier()
    clk = clocks.stop()
    ms_e2e = e2.elapsed_time(e3) / args.steps
    # ---- per-kernel timing of one step (roofline of the dominant contraction)
    E.PROFILE = []
    run.program(scale, eager=True)
    torch.cuda.synchronize()
    prof, E.PROFILE = E.PROFILE, None
    t_by = {}
    for wid, idx, kind, name, a, b in prof:
        t_by[(wid, idx, kind, name)] = t_by.get((wid, idx, kind, name), 0.0) + a.elapsed_time(b)
    step_prof_ms = sum(t_by.values())

    if world > 1:
        t = torch.tensor([ms, ms_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ms_e2e = float(t[0]), float(t[1])

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    burst, sustained, hbm, peak_src = measured_peaks()
    # contractions, timed per pass (the profiling step issues data and weight gradients separately)
    contr = {k: v for k, v in t_by.items() if k[3].startswith(("pc_conv2d_", "pc_fc_"))}
    top = max(contr.items(), key=lambda kv: kv[1]) if contr else None
    roof = None
    if top is not None:
        (wid, idx, kind, name), tms = top
        cl = next(c for c in cs.col_layers if c.index == idx)
        fl = layer_flops(cl, gbatch // plan.data_shards)
        passes = 1 if (name.endswith("]") or "forward" in name) else 2   # untagged backward = dgrad + wgrad
        if "backward" in name and not name.endswith("]") and idx == cs.col_layers[0].index:
            passes = 1                                      # layer 0: no data gradient
        achieved = fl * passes / (tms * 1e-3) / 1e12
        traffic = None
        tf = ROOT / "profiles" / "r01_roofline_traffic.json"
        if tf.exists():
            traffic = json.loads(tf.read_text()).get(f"{name} layer {idx}")
        roof = {"bound": "tensor", "kernel": f"{name} layer {idx}", "achieved": achieved,
                "peak": sustained, "unit": "TFLOP/s", "frac": achieved / sustained, "traffic": traffic,
                "peak_source": f"{peak_src} bf16_tflops_sustained (kernel timed inside the step)",
                "share_of_step": tms / step_prof_ms if step_prof_ms else None,
                "algorithmic_flop_per_launch": fl * passes,
                "traffic_source": "profiles/r01_roofline_traffic.json (ncu --set full dram bytes)" if traffic else None}
    shard = gbatch // plan.data_shards
    # reference convention (netdef.shape_report) minus layer 0's data gradient, which is never needed
    step_flops = plan.workers * (P.shape_report(cs, shard).total_flops - layer_flops(cs.col_layers[0], shard))
    value = gbatch / (ms * 1e-3)
    cpu = None
    if not args.no_cpu_baseline and not args.profile_only:
        try:
            v, dt = cpu_reference_sample(net, plan, cs, 2)
            cpu = {"value": v, "unit": "images/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"2 images of the {label} plan, float64 oracle step ({dt:.1f} s)"}
        except Exception as err:  # noqa: BLE001
            cpu = {"value": None, "unit": "images/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {err}"}
    line = {
        "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.precision, "data": "synthetic (gen_synthetic blobs, 1000 classes, "
        "3x227x227; Gaussian std 0.01 init, seed 0)",
        "config": {"workload": f"AlexNet-227 {label} train step", "global_batch": gbatch,
                   "per_gpu_batch": gbatch // plan.data_shards, "plan": plan.describe(),
                   "cross_layers": list(plan.cross_layers), "parallelism": label,
                   "l2": "activations >> 126 MB L2 (no flush needed)"},
        "tflops_achieved_step": step_flops / (ms * 1e-3) / 1e12,
        "roofline": roof, "cpu_baseline": cpu,
        "e2e": {"value": gbatch / (ms_e2e * 1e-3), "unit": "images/s",
                "h2d_bytes_per_step": int(x_e2e.numel() * x_e2e.element_size() + y_host.numel() * 4),
                "d2h_bytes_per_step": 8 * 2, "input_dtype": str(x_e2e.dtype).replace("torch.", ""),
                "path": "paper_1312_5853_b200.hybrid_step (public API), pinned host batch"},
        "gpu_launches": int(launches), "gpu_launches_per_step": launches / args.steps,
        "clocks": clk, "loss_first": res.loss, "loss_last": losses[-1] if losses else None,
        "tcgen05": bool(lib().dll.pc_has_tcgen05()),
    }
    print(json.dumps(line), flush=True)
    if os.environ.get("PC_BENCH_BREAKDOWN"):
        for k, v in sorted(t_by.items(), key=lambda kv: -kv[1])[:40]:
            print(f"# {v:8.3f} ms  wid={k[0]} layer={k[1]:2d} {k[2]:7s} {k[3]}", file=sys.stderr)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
