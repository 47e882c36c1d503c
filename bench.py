"""Benchmark: AlexNet (batch 256) synchronous-SGD training step on B200.

Metric (BASELINE.json): train images/sec, AlexNet b256 at 1/2/4/8 B200 per
scheme, with the dominant contraction's fraction of the tensor-core roofline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--scheme auto|dp|mp|hybrid] [--precision bf16|fp32]

N=1: plan d1m1, global batch 256. N>1 (torchrun, one rank per GPU):
auto = model parallel d1m2 cross(conv3) at N=2, hybrid d(N/2) x m2 at N=4/8
with 256 images per replica group (the paper's hybrid; weak scaling).
``--scheme dp``: data parallel dN x m1, global batch 256 sharded 256/N per GPU
(BASELINE configs[2]; strong scaling).

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
    ap.add_argument("--precision", default="bf16", choices=["bf16", "tf32", "fp32"])
    ap.add_argument("--batch", type=int, default=256, help="images per replica group")
    ap.add_argument("--net", default=str(ROOT / "configs" / "alexnet.net"))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-input", default="fp32", choices=["bf16", "fp32"])
    ap.add_argument("--cpu-sample", type=int, default=32, help="images in the CPU baseline sample")
    ap.add_argument("--ref-budget", type=float, default=120.0, help="seconds of timed reference steps")
    ap.add_argument("--profile-only", action="store_true", help="short run for ncu captures")
    return ap.parse_args()


def choose_plan(n: int, scheme: str, per_group: int):
    """(plan, global batch, label) of BASELINE configs[1..4]: dp = global 256 sharded
    over the GPUs (configs[2], the paper's data-parallel scaling: strong scaling);
    mp = the two-column net on 2 GPUs (configs[3]); hybrid = 2 columns x N/2 replicas,
    256 per replica group (configs[4]: weak scaling)."""
    from paper_1312_5853_b200.plan import ParallelPlan
    if n == 1:
        return ParallelPlan(1, 1), per_group, "d1m1"
    if scheme == "dp":
        if per_group % n:
            raise SystemExit(f"global batch {per_group} does not shard over {n} GPUs")
        return ParallelPlan(n, 1), per_group, f"dp{n}"
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
    """(bf16 burst TFLOP/s, bf16 sustained TFLOP/s, HBM GB/s, source)."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("bf16_tflops", 1590.0), d.get("bf16_tflops_sustained", 1400.0), d.get("hbm_gbs", 6650.0), \
            "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


def choose_tc_peak(clk: dict):
    """The burst peak applies to a kernel timed at (near) full SM clock; the
    sustained one (measured under a 4 s power-capped GEMM at ~1335 MHz) only
    when the timed region itself ran at reduced clocks."""
    burst, sustained, _, src = measured_peaks()
    sm, mx = clk.get("sm_mhz"), clk.get("sm_max_mhz")
    if sm is None or mx is None or sm >= 0.9 * mx:
        return burst, f"{src} bf16_tflops (burst; timed region median {sm} of {mx} MHz)"
    return sustained, f"{src} bf16_tflops_sustained (timed region median {sm} of {mx} MHz)"


def gemm_flops(cs, idx: int, name: str, shard: int):
    """Algorithmic FLOP of one contraction call (reference convention, 2/MAC)."""
    if not name.startswith(("pc_conv2d_", "pc_fc_")):
        return None
    cl = next(c for c in cs.col_layers if c.index == idx)
    fl = layer_flops(cl, shard)
    if "backward" in name and not name.endswith("]") and idx != cs.col_layers[0].index:
        return 2 * fl     # untagged backward = data + weight gradient
    return fl


def bandwidth_bytes(eng, idx: int, name: str):
    """Algorithmic HBM bytes (reads + writes at the storage dtype, each tensor
    once) of one bandwidth-bound call; None for contractions / unknown calls."""
    es = eng.dtype.itemsize
    B = eng.B
    st = next((t for t in eng.layers if t.cl.index == idx), None)
    n_in = B * math.prod(st.in_nhwc) if st is not None else 0
    n_out = B * math.prod(st.out_nhwc) if st is not None else 0
    if name == "pc_maxpool_forward":
        return n_in * es + n_out * (es + 1)
    if name.startswith("pc_maxpool_backward"):
        return n_out * (es + 1) + n_in * es + (n_out * es if st.mask_dx else 0)
    if name == "pc_softmax_xent":
        return 2 * n_in * es + B * 12
    if name in ("pc_lrn_forward", "pc_dropout", "pc_relu_forward", "pc_scale"):
        return 2 * n_in * es
    if name in ("pc_lrn_backward", "pc_relu_backward"):
        return 3 * n_in * es
    if name == "pc_space_to_depth_ex":
        c, h, w = eng.cs.base.input_shape
        return B * c * h * w * eng.x_src_es + B * eng.s2d_hw[0] * eng.s2d_hw[1] * 64 * es
    if name == "pc_sgd_step":
        return eng.sgd_numel() * (22 if es == 2 else 20)
    return None


def layer_flops(cl, batch: int) -> int:
    from paper_1312_5853_b200.netdef import layer_macs
    return 2 * layer_macs(cl, batch)


def _oracle_setup(net, plan, n_images: int, seed: int = 0):
    """The oracle (float64 numpy port of the reference step, TEST/BASELINE
    infrastructure) on a bounded sample: the first ``n_images`` images of the
    synthetic set, the same init as the GPU arm (Gaussian std 0.01)."""
    from oracle.ref_engine import OracleFabric
    from paper_1312_5853_b200.data import synthetic_rows
    from paper_1312_5853_b200.plan import init_dense_params
    x, y = synthetic_rows(1000, 1, net.input_shape, seed, np.arange(n_images))
    sample_plan = plan if n_images % plan.data_shards == 0 else type(plan)(1, plan.model_columns,
                                                                          plan.cross_layers)
    fab = OracleFabric(net, sample_plan, init_dense_params(net, seed, std=0.01))
    return fab, x.astype(np.float64), y


class CpuTimer:
    """Wall time and effective cores (process CPU time / wall time)."""

    def __enter__(self):
        self.t, self.c = time.perf_counter(), os.times()
        return self

    def __exit__(self, *exc):
        c = os.times()
        self.wall = time.perf_counter() - self.t
        self.cpu = (c.user - self.c.user) + (c.system - self.c.system)
        self.cores = self.cpu / self.wall if self.wall > 0 else None


def cpu_reference_sample(net, plan, cs, n_images: int, seed: int = 0) -> dict:
    fab, x, y = _oracle_setup(net, plan, n_images, seed)
    with CpuTimer() as t:
        fab.step(x, y)
    return {"value": n_images / t.wall, "unit": "images/s", "cores": os.cpu_count(),
            "effective_cores": t.cores, "kind": "port",
            "sample": f"one step of {n_images} images of the same plan, float64 numpy restatement of parconv "
                      f"(oracle/), same init as the GPU arm ({t.wall:.1f} s)"}


def run_reference_arm(args, rank: int):
    """--impl reference: the reference's CPU step (the float64 oracle port; the
    reference is Python and cannot travel to the GPU box) on the host cores,
    same metric/config/init, a bounded sample of the global batch per step.
    Timed steps stop early once ``--ref-budget`` seconds are spent (``steps``
    reports the number actually timed)."""
    if rank != 0:
        return
    from paper_1312_5853_b200.netdef import load_network
    from paper_1312_5853_b200.plan import plan_columnized
    net = load_network(args.net)
    plan, gbatch, label = choose_plan(args.gpus, args.scheme, args.batch)
    plan_columnized(net, plan)
    sample = max(plan.data_shards, args.cpu_sample)
    sample -= sample % plan.data_shards
    fab, x, y = _oracle_setup(net, plan, sample)
    fab.step(x, y)                                   # one untimed warm-up step
    done = 0
    with CpuTimer() as t:
        t0 = time.perf_counter()
        while done < args.steps and (done == 0 or time.perf_counter() - t0 < args.ref_budget):
            fab.step(x, y)
            done += 1
    v = sample * done / t.wall
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "images/s", "n_gpus": args.gpus,
            "steps": done, "steps_requested": args.steps, "warmup": 1, "ms_per_step": 1e3 * t.wall / done,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (gen_synthetic blobs; Gaussian std 0.01 init, seed 0)",
            "config": {"workload": f"AlexNet-227 {label} train step (reference CPU path)",
                       "global_batch": gbatch, "plan": plan.describe(), "parallelism": label},
            "cpu_baseline": {"value": v, "unit": "images/s", "cores": os.cpu_count(),
                             "effective_cores": t.cores, "kind": "port",
                             "sample": f"{sample} images per step of the {label} plan (of the {gbatch}-image "
                                       f"global batch), float64 numpy restatement of parconv (oracle/), "
                                       f"numpy BLAS threads = host cores"},
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
    # the reference's images are float32-quantised float64 (data.py:63): float32 carries
    # them exactly; bf16 is the rounding the device applies before conv1 anyway
    x_f32 = torch.from_numpy(np.ascontiguousarray(xb, dtype=np.float32)).pin_memory()
    x_bf16 = x_f32.to(torch.bfloat16).pin_memory()
    y_host = torch.from_numpy(yb.astype(np.int32)).pin_memory()
    x_e2e = x_f32 if args.e2e_input == "fp32" else x_bf16

    fab = P.spawn(plan.workers, precision=args.precision)
    # Gaussian std 0.01 (the paper's cited Krizhevsky init, reference SPEC.md:120): the He-normal
    # default diverges to inf within 4 steps on AlexNet at lr 0.01 in the reference as well
    P.setup_workers(fab, plan, cs, P.init_dense_params(net, 0, std=0.01), P.SgdState())
    # builds the engines; the device-resident batch is bf16 in the bf16 mode (the rounding
    # the input layer applies anyway), float32 otherwise
    res = P.hybrid_step(fab, plan, cs, x_bf16 if args.precision == "bf16" else x_f32, y_host)
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

    # ---- per-kernel timing (resident bf16 batch, as in "value"): one eager step with CUDA events around every C-ABI call on the
    # launching stream (passes serialised; backward split into data / weight gradients)
    E.PROFILE = []
    run.program(scale, eager=True)
    torch.cuda.synchronize()
    prof, E.PROFILE = E.PROFILE, None
    t_by, n_by = {}, {}
    for wid, idx, kind, name, a, b in prof:
        key = (wid, idx, kind, name)
        t_by[key] = t_by.get(key, 0.0) + a.elapsed_time(b)
        n_by[key] = n_by.get(key, 0) + 1
    step_prof_ms = sum(t_by.values())

    # ---- end to end through the public API: host batch -> device copy, step, loss read-back
    def e2e(xh, steps):
        for _ in range(2):
            P.hybrid_step(fab, plan, cs, xh, y_host, meter=False)
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ls = [P.hybrid_step(fab, plan, cs, xh, y_host, meter=False).loss for _ in range(steps)]
        b.record(stream)
        barrier()
        return a.elapsed_time(b) / steps, ls

    ms_e2e, losses = e2e(x_e2e, args.steps)
    clk = clocks.stop()
    variants = {}
    if not args.profile_only:
        other = x_bf16 if x_e2e is x_f32 else x_f32
        ms_o, _ = e2e(other, args.steps)
        variants[str(other.dtype).replace("torch.", "") + "_pinned"] = ms_o
        # the reference caller's own format: a float64 numpy batch (Dataset.images[chosen]);
        # host-side conversion dominates, so fewer steps
        ms_f64, _ = e2e(xb.astype(np.float64), max(2, min(args.steps, 5)))
        variants["float64_numpy"] = ms_f64

    if world > 1:
        t = torch.tensor([ms, ms_e2e], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ms_e2e = float(t[0]), float(t[1])

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    tc_peak, tc_src = choose_tc_peak(clk)
    if args.precision == "tf32":   # kind::tf32 runs at half the bf16 rate (B200_PROFILING.md: 1.1 PF dense)
        tc_peak, tc_src = tc_peak / 2, "half of " + tc_src + " (tf32 tensor-core rate)"
    _, _, hbm, hbm_src = measured_peaks()
    shard = gbatch // plan.data_shards
    kernels = []
    for (wid, idx, kind, name), tms in t_by.items():
        eng = run.engines[wid]
        fl = gemm_flops(cs, idx, name, shard)
        by = None if fl is not None else bandwidth_bytes(eng, idx, name)
        row = {"call": name, "layer": idx, "worker": wid, "ms": tms, "launches": n_by[(wid, idx, kind, name)],
               "share_of_step": tms / ms}
        if fl is not None:
            ach = fl / (tms * 1e-3) / 1e12
            row.update(bound="tensor", algorithmic=fl, achieved=ach, unit="TFLOP/s", frac=ach / tc_peak)
        elif by is not None:
            ach = by / (tms * 1e-3) / 1e9
            row.update(bound="hbm", algorithmic=by, achieved=ach, unit="GB/s", frac=ach / hbm)
        kernels.append(row)
    kernels.sort(key=lambda r: -r["ms"])
    gemms = [r for r in kernels if r.get("bound") == "tensor"]
    roof = None
    if gemms:
        top = gemms[0]
        traffic = None
        for tf in (ROOT / "profiles" / "r02_roofline_traffic.json", ROOT / "profiles" / "r01_roofline_traffic.json"):
            if tf.exists():
                traffic = json.loads(tf.read_text()).get(f"{top['call']} layer {top['layer']}")
                if traffic is not None:
                    break
        roof = {"bound": "tensor", "kernel": f"{top['call']} layer {top['layer']}", "achieved": top["achieved"],
                "peak": tc_peak, "unit": "TFLOP/s", "frac": top["frac"], "traffic": traffic,
                "peak_source": tc_src, "share_of_step": top["share_of_step"],
                "algorithmic_flop_per_launch": top["algorithmic"],
                "timing": "CUDA events around the call on its launching stream, one eager step "
                          "(serialised passes); share_of_step = call time / graph-replayed ms_per_step",
                "traffic_source": f"{tf.relative_to(ROOT)} (ncu dram bytes)" if traffic else None}
    # reference convention (netdef.shape_report) minus layer 0's data gradient, which is never needed
    step_flops = plan.workers * (P.shape_report(cs, shard).total_flops - layer_flops(cs.col_layers[0], shard))
    value = gbatch / (ms * 1e-3)
    cpu = None
    if not args.no_cpu_baseline and not args.profile_only:
        try:
            cpu = cpu_reference_sample(net, plan, cs, args.cpu_sample)
        except Exception as err:  # noqa: BLE001
            cpu = {"value": None, "unit": "images/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {err}"}
    h2d = int(x_e2e.numel() * x_e2e.element_size() + y_host.numel() * 4)
    line = {
        "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        # dp (global 256 sharded) and mp (the same 256 over two columns) divide a fixed batch;
        # hybrid keeps 256 per replica group, so the total grows with the replicas
        "scaling": "weak" if plan.data_shards > 1 and plan.model_columns > 1 or plan.workers == 1 else "strong",
        "vs_baseline": None, "dtype": args.precision, "data": "synthetic (gen_synthetic blobs, 1000 classes, "
        "3x227x227; Gaussian std 0.01 init, seed 0)",
        "config": {"workload": f"AlexNet-227 {label} train step", "global_batch": gbatch,
                   "per_gpu_batch": shard, "plan": plan.describe(),
                   "cross_layers": list(plan.cross_layers), "parallelism": label,
                   "l2": "activations >> 126 MB L2 (no flush needed)",
                   "resident_input": ("bf16" if args.precision == "bf16" else "float32") +
                          " NCHW (value); e2e from the host format named in e2e.input_dtype"},
        "tflops_achieved_step": step_flops / (ms * 1e-3) / 1e12,
        "roofline_step": {"achieved": step_flops / (ms * 1e-3) / 1e12, "peak": tc_peak,
                          "frac": step_flops / (ms * 1e-3) / 1e12 / tc_peak},
        "roofline": roof, "cpu_baseline": cpu,
        "e2e": {"value": gbatch / (ms_e2e * 1e-3), "unit": "images/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": 8 * 2, "input_dtype": str(x_e2e.dtype).replace("torch.", ""),
                "path": "paper_1312_5853_b200.hybrid_step (public API), pinned host batch",
                "variants_images_per_s": {k: gbatch / (v * 1e-3) for k, v in variants.items()}},
        "kernels": kernels[:24], "kernels_profile_ms": step_prof_ms,
        "hbm_peak": {"value": hbm, "source": f"{hbm_src} hbm_gbs"},
        "gpu_launches": int(launches), "gpu_launches_per_step": launches / args.steps,
        "clocks": clk, "loss_first": res.loss, "loss_last": losses[-1] if losses else None,
        "tcgen05": bool(lib().dll.pc_has_tcgen05()),
    }
    print(json.dumps(line), flush=True)
    if os.environ.get("PC_BENCH_BREAKDOWN"):
        for r in kernels[:40]:
            extra = f"{r.get('achieved', 0):8.1f} {r.get('unit', ''):8s} frac {r.get('frac', 0):.2f}" \
                if "frac" in r else ""
            print(f"# {r['ms']:8.3f} ms  layer={r['layer']:2d} {r['call']:32s} {extra}", file=sys.stderr)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
