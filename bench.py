#!/usr/bin/env python
"""Benchmark of the depth-first stack executor on BASELINE.json's metric.

metric : "fused-stack HBM GB/s (% of B200 peak) and images/sec at 1/2/4/8 GPUs"
value  : whole-job images/s (all ranks) for one pass of every stack of the workload over one
         batch per rank (a "step"); GB/s and % of the measured HBM peak ride alongside.
default workload: configs[3], ResNet-50's stem BN->ReLU->MaxPool3x3/s2/p1 + 32 BN->ReLU stacks
         at batch 256 -- the largest BASELINE config that runs on one GPU (7.76 GB per step).
         The same run also measures configs[1] AlexNet, configs[2] VGG-16 and configs[4]
         DenseNet-121 ("workloads" key; `--no-extra` skips them) and configs[0] C1 ("c1" key:
         the GPU time and the CPU oracle's time in ms, min of 5 runs).

Multi-GPU (torchrun, one process per GPU): the batch dimension is the unit that shards (every
image is independent).  ResNet-50 / AlexNet / VGG-16 run weak-scaled (every rank
its BASELINE batch); DenseNet-121 is strong-scaled by default (BASELINE.json: its batch 256
"sharded across 8xB200").  No collective on the data path: NCCL only after the timed region
(max-over-ranks times, per-rank checksums, and an all-gather of the dominant stack's output
shards, sampled images compared with the CPU oracle on rank 0).  The aggregate images/s uses
the slower of (max over ranks of the CUDA-event time) and (max over ranks of the host
wall-clock between the barriers that bracket the timed region), so ranks sharing one GPU cannot
report more than that GPU delivers.

Timing: W warm-up steps, then K steps between barrier + cuda.synchronize on both sides, CUDA
events on the launching stream; inputs rotate over enough buffer sets to exceed 4x the L2 (or
are larger than L2).  The dominant kernel is timed alone (events around back-to-back launches)
for the roofline object; every stack is also timed alone against a same-size ideal streaming
kernel (benchlib/ceiling.cu) -- "per_stack".  `--impl reference` times the CPU oracle instead
(rank 0 only), a bounded sample of images per step.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "fused-stack HBM GB/s (% of B200 peak) and images/sec at 1/2/4/8 GPUs"
CONFIG_INDEX = {"c1": 0, "alexnet": 1, "vgg16": 2, "resnet50": 3, "densenet121": 4,
                "resnet50_residual": None}   # NEXT-1: not a BASELINE config
STRONG_BY_DEFAULT = {"densenet121"}          # BASELINE.json configs[4]: "sharded across 8xB200"
EXTRA_WORKLOADS = ("alexnet", "vgg16", "densenet121")


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json, b.copy_(a) read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def instances(cases):
    out = []
    for c in cases:
        out += [c] * c.count
    return out


def kernel_sources_hash() -> str:
    """sha256 (16 hex) of the kernel + planner sources with comments and blank lines removed: keys
    stored ncu traffic to the code that was profiled (a comment edit does not invalidate it)."""
    import glob
    import re
    h = hashlib.sha256()
    for p in sorted(glob.glob(os.path.join(ROOT, "paper_1804_08378_b200", "csrc", "*"))):
        text = open(p, encoding="utf-8").read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        lines = [re.sub(r"//.*$", "", ln).rstrip() for ln in text.splitlines()]
        h.update("\n".join(ln for ln in lines if ln.strip()).encode())
    return h.hexdigest()[:16]


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons while the timed region runs."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # no NVML: report what we have
            self.nv = None
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            self.sample()
            time.sleep(0.002)

    def sample(self):
        if self.nv is None:
            return
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for bit, name in self.REASONS.items():
                if r & bit:
                    self.reasons.add(name)
        except Exception:
            pass

    def __enter__(self):
        self.sample()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join()
        self.sample()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- multi-rank host logic
# (no CUDA here: tests/test_bench_dist.py drives these under torchrun + gloo with a stub executor)
def shard_of(n_total: int, world: int, rank: int, strong: bool):
    """(lo, hi) global image range of `rank`: strong = n_total split over the ranks, weak = every
    rank its own n_total images (the global batch is world * n_total)."""
    from paper_1804_08378_b200 import dist as bsd
    if strong:
        return bsd.shard(n_total, world, rank)
    return rank * n_total, (rank + 1) * n_total


def aggregate(images_local: int, event_ms_local: float, wall_s_local: float, steps: int, device="cpu"):
    """Whole-job rate of a timed region bracketed by barriers on every rank.  wall_s_local runs from
    the release of the opening barrier to the release of the closing one (so it spans every rank's
    work); the job time is the slower of the max-over-ranks device time and the max-over-ranks wall
    time: ranks whose work does not really overlap (several ranks on one GPU) cannot add up to
    more than the device delivers."""
    from paper_1804_08378_b200 import dist as bsd
    g = bsd.gather_stats([float(images_local), float(event_ms_local), float(wall_s_local)], device)
    images = int(round(sum(r[0] for r in g)))
    ev_max = max(r[1] for r in g)
    wall_max = max(r[2] for r in g)
    t_s = max(ev_max / 1e3, wall_max)
    return {"images_per_step": images, "event_ms_max": ev_max, "wall_s_max": wall_max,
            "time_s": t_s, "ms_per_step": 1e3 * t_s / steps, "images_per_s": images * steps / t_s,
            "timer": "wall" if wall_max >= ev_max / 1e3 else "events",
            "per_rank": [{"images": int(r[0]), "event_ms": r[1], "wall_s": r[2]} for r in g]}


def validate_gathered(gathered, n_total: int, ref_image, check, samples=3):
    """Compare sampled global images of an all-gathered output with a reference (the oracle).
    ref_image(n) -> expected output of image n (1, C, Ho, Wo); check(got, ref, ctx) raises."""
    idx = sorted({0, n_total // 2, n_total - 1} | {int(v) for v in np.linspace(0, n_total - 1, samples)})
    if os.environ.get("BS_VALIDATE_ALL"):
        idx = list(range(n_total))
    errs = []
    for n in idx:
        try:
            check(np.asarray(gathered[n:n + 1]), ref_image(n), f"image {n}")
        except AssertionError as e:
            errs.append(str(e)[:200])
    return {"images_checked": idx, "ok": not errs, "errors": errs}


# ----------------------------------------------------------------------------- CPU oracle timing
def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _oracle_image(case, k):
    shp = (1,) + tuple(case.shape[1:])
    n = int(np.prod(shp))
    x = synth.uniform_np(case.input_seed, n, start=k * n).reshape(shp)
    ops = [synth.uniform_np(sd, n, start=k * n).reshape(shp) for sd in case.operand_seeds]
    return x, ops


def time_oracle(cases, budget_s: float, max_images: int):
    """The oracle as it stands (single thread) on whole images of the workload."""
    import oracle
    oracle.build()

    def one_image(k):
        for c in cases:
            x, ops = _oracle_image(c, k)
            for _ in range(c.count):
                oracle.run_bf(c.layers, x, ops)
    t0 = time.perf_counter()
    one_image(0)
    t1 = time.perf_counter() - t0
    n = int(max(1, min(max_images, budget_s / max(t1, 1e-6))))
    t0 = time.perf_counter()
    for k in range(n):
        one_image(k)
    T = time.perf_counter() - t0
    return n / T, n, T


def time_oracle_threads(cases, budget_s: float, threads: int):
    """The same oracle run on `threads` host threads at once, one image per task (images are
    independent; the C oracle is reentrant and its ctypes calls release the GIL): the
    all-core figure beside the single-thread baseline.  The oracle itself is unchanged."""
    import concurrent.futures
    import oracle
    oracle.build()

    def one_image(k):
        for c in cases:
            x, ops = _oracle_image(c, k)
            for _ in range(c.count):
                oracle.run_bf(c.layers, x, ops)
    t0 = time.perf_counter()
    one_image(0)
    t1 = time.perf_counter() - t0
    n = int(max(threads, threads * round(budget_s * threads / max(t1, 1e-6) / threads)))
    n = max(threads, min(n, 64 * threads))
    with concurrent.futures.ThreadPoolExecutor(threads) as ex:
        t0 = time.perf_counter()
        list(ex.map(one_image, range(n)))
        T = time.perf_counter() - t0
    return n / T, n, T


def c1_oracle_ms(reps: int = 5) -> float:
    """BASELINE.json configs[0] on the CPU oracle, in ms: min of `reps` runs."""
    import oracle
    oracle.build()
    case = synth.workload("c1")[0]
    x = synth.uniform_np(case.input_seed, int(np.prod(case.shape))).reshape(case.shape)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        oracle.run_bf(case.layers, x)
        ts.append(time.perf_counter() - t0)
    return 1e3 * min(ts)


def run_reference(args):
    """--impl reference: the CPU oracle timed on the host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cases = synth.workload(args.workload, batch=1)
    import oracle
    oracle.build()

    def step(k):
        for c in cases:
            x, ops = _oracle_image(c, k)
            for _ in range(c.count):
                oracle.run_bf(c.layers, x, ops)
    for k in range(args.warmup):
        step(k)
    t0 = time.perf_counter()
    for k in range(args.steps):
        step(args.warmup + k)
    T = time.perf_counter() - t0
    ips = args.steps / T
    batch = synth.DEFAULT_BATCH[args.workload]
    line = {"impl": "reference", "metric": METRIC, "value": ips, "unit": "images/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64 arithmetic, f32 tensors", "data": "synthetic (SplitMix64, seeded)",
            "config": {"workload": args.workload, "baseline_config_index": CONFIG_INDEX[args.workload],
                       "global_batch": batch, "parallelism": "none (host CPU oracle)"},
            "cpu_baseline": {"value": ips, "unit": "images/s", "cores": 1, "kind": "oracle",
                             "sample": f"1 image of the batch-{batch} {args.workload} workload per step "
                                       f"(every stack), breadth-first C oracle, single thread"},
            "e2e": {"value": ips, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU bench
class Ctx:
    """Process-wide state of a GPU run."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.args = torch, dist, args
        import paper_1804_08378_b200 as bs
        self.bs = bs
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        # one process per GPU; BS_BENCH_BACKEND=gloo lets several ranks share one GPU (testing the
        # multi-rank path on a 1-GPU box)
        self.backend = os.environ.get("BS_BENCH_BACKEND", "nccl")
        dev_idx = self.local % torch.cuda.device_count()
        torch.cuda.set_device(dev_idx)
        self.dev = torch.device("cuda", dev_idx)
        if self.world > 1:
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=self.dev)
            else:
                dist.init_process_group(self.backend)
        self.stream = torch.cuda.Stream(device=self.dev)
        self.sh = self.stream.cuda_stream
        self.l2 = torch.cuda.get_device_properties(self.dev).L2_cache_size
        self.peak, self.peak_src = load_peaks()

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def event(self):
        return self.torch.cuda.Event(enable_timing=True)

    def launch(self, h, xs, y):
        if len(xs) == 1:
            self.bs.bs_execute(h, xs[0].data_ptr(), y.data_ptr(), self.sh)
        else:
            self.bs.bs_execute_ex(h, [t.data_ptr() for t in xs], y.data_ptr(), self.sh)

    def burst_ms(self, fn, reps=3):
        """Average time of fn() (one burst) captured once as a torch CUDA graph, over `reps` replays."""
        torch = self.torch
        with torch.cuda.stream(self.stream):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self.stream):
            fn()
        torch.cuda.synchronize()
        a, b = self.event(), self.event()
        with torch.cuda.stream(self.stream):
            g.replay()
            a.record(self.stream)
            for _ in range(reps):
                g.replay()
            b.record(self.stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        del g
        return ms


def stack_burst(ctx, case, plan, nb, extra_seed):
    """Rotating buffer sets of one stack (> 4x L2 in total) for burst timing."""
    torch = ctx.torch
    nset = min(64, int(math.ceil(4 * ctx.l2 / nb)) + 1)
    sb = [([synth.uniform_torch(sd + extra_seed * q, case.shape, device=ctx.dev)
            for sd in [case.input_seed] + case.operand_seeds],
           torch.empty(ctx.bs.bs_plan_query(plan)["out"], device=ctx.dev)) for q in range(nset)]
    R = max(8, min(64, 2 * nset))
    return sb, R


def measure_stack_alone(ctx, case, plan, info):
    """One stack alone: R back-to-back launches over rotating buffers (one CUDA graph), and the
    same-size ideal streaming kernel (fastest of benchlib.VARIANTS) on the same byte counts."""
    import benchlib
    nb = info["alg_bytes_read"] + info["alg_bytes_written"]
    sb, R = stack_burst(ctx, case, plan, nb, 13)

    def burst():
        for r in range(R):
            xs, y = sb[r % len(sb)]
            ctx.launch(plan, xs, y)
    t = ctx.burst_ms(burst) / R
    n_in = info["alg_bytes_read"] // 4
    n_out = info["alg_bytes_written"] // 4
    cin = [ctx.torch.empty(n_in, device=ctx.dev) for _ in range(len(sb))]
    cout = [y.view(-1) for _, y in sb]
    best = None
    for v in benchlib.VARIANTS:
        def cburst(v=v):
            for r in range(R):
                benchlib.launch(v, cin[r % len(sb)].data_ptr(), n_in, cout[r % len(sb)].data_ptr(), n_out, ctx.sh)
        tc = ctx.burst_ms(cburst) / R
        if best is None or tc < best[0]:
            best = (tc, v)
    del sb, cin, cout
    gbs = nb / (t / 1e3) / 1e9
    return {"stack": case.name, "count": case.count, "shape": list(case.shape), "ms": t, "gbs": gbs,
            "frac_of_copy": gbs / ctx.peak, "ceiling_ms": best[0], "ceiling_variant": "/".join(map(str, best[1])),
            "frac_of_ceiling": best[0] / t,
            "kernel": ctx.bs.KERNEL_NAMES[ctx.bs.bs_plan_query_launch(plan, 0)["kernel"]]}


def measure(ctx, wl: str, full: bool):
    """Time workload `wl` (one step = every stack of the network once over one batch per rank)."""
    torch, bs, args = ctx.torch, ctx.bs, ctx.args
    full_batch = args.batch or synth.DEFAULT_BATCH[wl]
    strong = args.strong or (wl in STRONG_BY_DEFAULT and not args.weak)
    lo, hi = shard_of(full_batch, ctx.world, ctx.rank, strong)
    batch = hi - lo
    n_total = full_batch if strong else full_batch * ctx.world
    cases = synth.workload(wl, batch=batch)
    inst = instances(cases)
    plans = {c.name: bs.bs_plan_create(c.layers, c.shape) for c in cases}
    infos = {c.name: bs.bs_plan_query(plans[c.name]) for c in cases}
    launches_per_step = sum(infos[c.name]["n_launches"] for c in inst)
    step_bytes = sum(infos[c.name]["alg_bytes_read"] + infos[c.name]["alg_bytes_written"] for c in inst)
    n_sets = 1 if step_bytes >= 8 * ctx.l2 else int(math.ceil(4 * ctx.l2 / step_bytes)) + 1
    # buffers per instance per set; each rank's inputs are its slice [lo, hi) of the global
    # image stream, so the gathered outputs are those of one global batch
    bufs = []
    for s in range(n_sets):
        row = []
        for j, c in enumerate(inst):
            chw = int(np.prod(c.shape[1:]))
            x = synth.uniform_torch(c.input_seed + 7 * j + 1000 * s, c.shape, device=ctx.dev, start=lo * chw)
            ops = [synth.uniform_torch(sd + 7 * j + 1000 * s, c.shape, device=ctx.dev, start=lo * chw)
                   for sd in c.operand_seeds]
            y = torch.empty(infos[c.name]["out"], device=ctx.dev)
            row.append(([x] + ops, y))
        bufs.append(row)
    torch.cuda.synchronize()           # inputs are generated on the default stream
    dom = max(range(len(inst)), key=lambda j: infos[inst[j].name]["alg_bytes_read"] + infos[inst[j].name]["alg_bytes_written"])
    dom_bytes = infos[inst[dom].name]["alg_bytes_read"] + infos[inst[dom].name]["alg_bytes_written"]
    handles = [plans[c.name] for c in inst]

    def eager_step(k):
        row = bufs[k % n_sets]
        for j, h in enumerate(handles):
            xs, y = row[j]
            ctx.launch(h, xs, y)

    with torch.cuda.stream(ctx.stream):
        for k in range(args.warmup):
            eager_step(k)
    torch.cuda.synchronize()
    # one CUDA graph per buffer set over every stack of the step, built by the library's own
    # bs_graph API (NEXT-3): a step is a single host call
    graphs = [bs.bs_graph_create([(h, bufs[s][j][0], bufs[s][j][1]) for j, h in enumerate(handles)])
              for s in range(n_sets)]
    torch.cuda.synchronize()

    def run_step(k):
        bs.bs_graph_launch(graphs[k % n_sets], ctx.sh)

    with torch.cuda.stream(ctx.stream):
        for k in range(args.warmup):
            run_step(k)
    torch.cuda.synchronize()
    t_start, t_end = ctx.event(), ctx.event()
    clk = ClockSampler(ctx.local)      # NVML init before the barrier: it takes tens of ms
    torch.cuda.synchronize()
    with clk:
        # wall-clock from the release of the opening barrier to the release of the closing one:
        # the job time of all ranks together
        ctx.barrier()
        w0 = time.perf_counter()
        with torch.cuda.stream(ctx.stream):
            t_start.record(ctx.stream)
            for k in range(args.steps):
                run_step(args.warmup + k)
            t_end.record(ctx.stream)
        torch.cuda.synchronize()
        ctx.barrier()
        wall = time.perf_counter() - w0
    ev_ms = t_start.elapsed_time(t_end)
    agg = aggregate(batch, ev_ms, wall, args.steps, ctx.dev)

    res = {"workload": wl, "baseline_config_index": CONFIG_INDEX[wl], "scaling": "strong" if strong else "weak",
           "global_batch": agg["images_per_step"], "per_gpu_batch": batch, "stacks_per_step": len(inst),
           "launches_per_step": launches_per_step, "value": agg["images_per_s"], "ms_per_step": agg["ms_per_step"],
           "timing": {k: agg[k] for k in ("event_ms_max", "wall_s_max", "timer")},
           "clocks": clk.summary()}
    gbs_rank = step_bytes / (ev_ms / args.steps / 1e3) / 1e9
    res["hbm"] = {"alg_gbs_per_gpu": gbs_rank, "alg_gbs_total": step_bytes * ctx.world / (agg["ms_per_step"] / 1e3) / 1e9,
                  "pct_of_measured_peak": 100 * gbs_rank / ctx.peak, "pct_of_8tbs": 100 * gbs_rank / 8000.0,
                  "alg_bytes_per_step_per_gpu": step_bytes}
    res["l2"] = (f"rotating {n_sets} buffer sets ({n_sets * step_bytes / 1e9:.2f} GB > 4x L2 {ctx.l2 / 1e6:.0f} MB)"
                 if n_sets > 1 else f"inputs larger than L2 ({step_bytes / 1e9:.2f} GB per step vs {ctx.l2 / 1e6:.0f} MB)")

    if full:   # per-step min / median (SURVEY §8(d) protocol), outside the timed region
        per_step = []
        with torch.cuda.stream(ctx.stream):
            for k in range(20):
                e0, e1 = ctx.event(), ctx.event()
                e0.record(ctx.stream)
                run_step(k)
                e1.record(ctx.stream)
                e1.synchronize()
                per_step.append(e0.elapsed_time(e1))
        res["ms_per_step_isolated"] = {"min": float(np.min(per_step)), "median": float(np.median(per_step)),
                                       "n": len(per_step)}

    # dominant kernel alone: D back-to-back launches over rotating buffer sets (one bs_graph),
    # CUDA events on the launching stream around the replays -> average launch duration
    D = max(4, min(50, int(4 * ctx.l2 // max(1, dom_bytes)) + 4))
    dom_sets = max(n_sets, int(math.ceil(4 * ctx.l2 / dom_bytes)) + 1)
    dbufs = [bufs[s % n_sets][dom] if s < n_sets else
             ([synth.uniform_torch(sd + 99 * s, inst[dom].shape, device=ctx.dev)
               for sd in [inst[dom].input_seed] + inst[dom].operand_seeds],
              torch.empty(infos[inst[dom].name]["out"], device=ctx.dev)) for s in range(dom_sets)]
    dh = handles[dom]
    dg = bs.bs_graph_create([(dh, dbufs[r % dom_sets][0], dbufs[r % dom_sets][1]) for r in range(D)])
    torch.cuda.synchronize()           # the extra input sets are generated on the default stream
    da, db = ctx.event(), ctx.event()
    reps = 5
    with torch.cuda.stream(ctx.stream):
        bs.bs_graph_launch(dg, ctx.sh)
        da.record(ctx.stream)
        for _ in range(reps):
            bs.bs_graph_launch(dg, ctx.sh)
        db.record(ctx.stream)
    torch.cuda.synchronize()
    dom_ms = da.elapsed_time(db) / (reps * D)
    del dg, dbufs
    from paper_1804_08378_b200 import dist as bsd
    dom_ms = bsd.max_over_ranks([dom_ms], ctx.dev)[0]
    dom_li = bs.bs_plan_query_launch(plans[inst[dom].name], 0)
    dom_achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    res["roofline"] = {"bound": "hbm", "achieved": dom_achieved, "peak": ctx.peak, "unit": "GB/s",
                       "frac": dom_achieved / ctx.peak, "traffic": None, "peak_source": ctx.peak_src,
                       "kernel": bs.KERNEL_NAMES[dom_li["kernel"]], "stack": inst[dom].name,
                       "alg_bytes_per_launch": dom_bytes, "avg_launch_ms": dom_ms,
                       "how": f"{D} back-to-back launches over {dom_sets} rotating buffer sets, CUDA events"}
    res["roofline"].update(stored_traffic(wl, inst[dom].name, dom_bytes))

    # checksums of the last timed step (fp64 sum per stack output) and validation of the
    # dominant stack: all-gather its output shards, compare sampled global images with the oracle
    last = bufs[(args.warmup + args.steps - 1) % n_sets]
    csum = float(sum(y.double().sum().item() for _, y in last))
    finite = all(bool(torch.isfinite(y).all()) for _, y in last)
    g = bsd.gather_stats([csum, float(finite)], ctx.dev)
    res["checksums"] = [r[0] for r in g]
    res["outputs_finite"] = all(bool(r[1]) for r in g)
    if not args.no_validate:
        res["validation"] = validate_dominant(ctx, inst[dom], last[dom], dom, n_total, lo,
                                              (args.warmup + args.steps - 1) % n_sets)
    res["_internal"] = {"cases": cases, "plans": plans, "infos": infos, "inst": inst, "bufs": bufs,
                        "n_sets": n_sets, "batch": batch, "handles": handles}
    return res


def validate_dominant(ctx, case, buf, j, n_total, lo, set_idx):
    """All-gather the dominant stack's output shards (outside the timed region) and compare
    sampled global images with the CPU oracle on rank 0."""
    from paper_1804_08378_b200 import dist as bsd
    xs, y = buf
    out = bsd.gather_shards(y, n_total, ctx.dev) if ctx.world > 1 else y
    if ctx.rank != 0:
        return None
    import oracle
    from tests import _util as U
    oracle.build()
    chw = int(np.prod(case.shape[1:]))
    shp = (1,) + tuple(case.shape[1:])
    base = case.input_seed + 7 * j + 1000 * set_idx

    def ref_image(n):
        x = synth.uniform_np(base, chw, start=n * chw).reshape(shp)
        ops = [synth.uniform_np(sd + 7 * j + 1000 * set_idx, chw, start=n * chw).reshape(shp)
               for sd in case.operand_seeds]
        return oracle.run_bf(case.layers, x, ops)

    gathered = out.cpu().numpy() if hasattr(out, "cpu") else out
    r = validate_gathered(gathered, n_total, ref_image, lambda got, ref, ctx_: U.check(got, ref, case.layers, ctx_))
    r["stack"] = case.name
    r["gathered_images"] = int(gathered.shape[0])
    return r


def stored_traffic(wl, stack, alg_bytes):
    """ncu DRAM bytes per launch of the dominant stack, from profiles/ncu_traffic.json -- used only
    if it was captured from the current kernel sources (keyed by their hash), else null."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    out = {"traffic_source": None}
    if not os.path.exists(p):
        return out
    tr = json.load(open(p))
    e = tr.get("entries", {}).get(f"{wl}:{stack}")
    if e is None:
        return out
    if tr.get("sources_sha16") != kernel_sources_hash():
        out["traffic_source"] = f"stale: {p} was captured from kernel sources {tr.get('sources_sha16')}"
        return out
    if e.get("alg_bytes_per_launch") != alg_bytes:   # another batch (e.g. a strong-scaled shard)
        out["traffic_source"] = (f"not comparable: captured at {e.get('alg_bytes_per_launch')} algorithmic bytes "
                                 f"per launch, this launch moves {alg_bytes}")
        return out
    out["traffic"] = e["dram_bytes_per_launch"]
    out["traffic_ratio_to_alg"] = e["dram_bytes_per_launch"] / alg_bytes
    out["traffic_source"] = f"ncu --set full, {tr.get('captured')} ({os.path.relpath(p, ROOT)})"
    return out


def measure_e2e(ctx, m):
    """End to end through bs_execute_host_batch: every step copies each stack's inputs from pinned
    host memory, runs the kernels and copies the outputs back (pipelined per image chunk and across
    the step's stacks)."""
    torch, bs, args = ctx.torch, ctx.bs, ctx.args
    I = m["_internal"]
    cases, infos, inst, bufs, n_sets, handles = I["cases"], I["infos"], I["inst"], I["bufs"], I["n_sets"], I["handles"]
    e2e_steps = args.e2e_steps or max(3, min(20, args.steps // 10))
    max_in = max(infos[c.name]["alg_bytes_read"] // (1 + len(c.operand_seeds)) for c in cases) // 4
    max_out = max(infos[c.name]["alg_bytes_written"] for c in cases) // 4
    h_in = torch.empty(max_in, dtype=torch.float32).pin_memory()
    h_in.copy_(synth.uniform_torch(99, (max_in,), device=ctx.dev).cpu())
    h_out = torch.empty(max_out, dtype=torch.float32).pin_memory()
    h2d = sum(infos[c.name]["alg_bytes_read"] for c in inst)
    d2h = sum(infos[c.name]["alg_bytes_written"] for c in inst)

    def e2e_step(k):
        # one call per step: every stack's copies in, kernels and copies out, pipelined across
        # the stacks (bs_execute_host_batch); all stacks read one pinned host input buffer and
        # write one pinned host output buffer (the bytes moved are the same)
        row = bufs[k % n_sets]
        bs.bs_execute_host_batch(handles, [[h_in.data_ptr()] * len(row[j][0]) for j in range(len(handles))],
                                 [h_out.data_ptr()] * len(handles), [[t.data_ptr() for t in row[j][0]] for j in range(len(handles))],
                                 [row[j][1].data_ptr() for j in range(len(handles))], 0, ctx.sh)

    e2e_step(0)
    torch.cuda.synchronize()
    a, b = ctx.event(), ctx.event()
    ctx.barrier()
    w0 = time.perf_counter()
    a.record(ctx.stream)
    for k in range(e2e_steps):
        e2e_step(k)
    b.record(ctx.stream)
    torch.cuda.synchronize()
    ctx.barrier()
    wall = time.perf_counter() - w0
    agg = aggregate(I["batch"], a.elapsed_time(b), wall, e2e_steps, ctx.dev)
    # the e2e roofline: host <-> device bandwidth of a plain pinned copy of the same bytes
    probe = int(min(h2d, 256 << 20))
    hb = torch.empty(probe // 4, dtype=torch.float32).pin_memory()
    dbuf = torch.empty(probe // 4, dtype=torch.float32, device=ctx.dev)
    pcie_gbs = d2h_gbs = 0.0
    with torch.cuda.stream(ctx.stream):
        for r in range(7):   # 2 warm-up copies each way, then the best of 5
            a.record(ctx.stream)
            dbuf.copy_(hb, non_blocking=True)
            b.record(ctx.stream)
            torch.cuda.synchronize()
            if r >= 2:
                pcie_gbs = max(pcie_gbs, probe / (a.elapsed_time(b) / 1e3) / 1e9)
            a.record(ctx.stream)
            hb.copy_(dbuf, non_blocking=True)
            b.record(ctx.stream)
            torch.cuda.synchronize()
            if r >= 2:
                d2h_gbs = max(d2h_gbs, probe / (a.elapsed_time(b) / 1e3) / 1e9)
    del hb, dbuf
    # ... and the measured ceiling: plain pinned copies of exactly the step's bytes (every stack's
    # input in on one stream, its output out on another -- PCIe full duplex), no kernels, best of 3
    row = bufs[0]
    s_in, s_out = torch.cuda.Stream(ctx.dev), torch.cuda.Stream(ctx.dev)

    def plain_copies():
        for j in range(len(handles)):
            xs, y = row[j]
            with torch.cuda.stream(s_in):
                for t in xs:
                    t.view(-1).copy_(h_in[:t.numel()], non_blocking=True)
            with torch.cuda.stream(s_out):
                h_out[:y.numel()].copy_(y.view(-1), non_blocking=True)
    t_copy = 1e30
    for r in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plain_copies()
        torch.cuda.synchronize()
        if r >= 1:
            t_copy = min(t_copy, time.perf_counter() - t0)
    t_step = agg["ms_per_step"] / 1e3
    t_bound = max(h2d / (pcie_gbs * 1e9), d2h / (d2h_gbs * 1e9))
    return {"value": agg["images_per_s"], "unit": "images/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": e2e_steps, "timer": agg["timer"],
            "path": "bs_execute_host_batch: every stack's pinned host -> device copy, kernels, device -> host copy, "
                    "pipelined per image chunk and across the step's stacks (one call per step)",
            "roofline": {"bound": "pcie_duplex", "achieved_gbs": (h2d + d2h) / t_step / 1e9,
                         "peak_gbs": (h2d + d2h) / t_copy / 1e9, "frac": t_copy / t_step,
                         "peak_source": "measured: plain pinned torch copies of the step's exact bytes, every stack's "
                                        "input host->device on one stream and output device->host on another, no "
                                        "kernels (best of 3)",
                         "unidirectional_gbs": {"h2d": pcie_gbs, "d2h": d2h_gbs},
                         "frac_vs_unidirectional_peaks": t_bound / t_step}}


def measure_lbl(ctx, m):
    """Layer-by-layer torch eager on the same GPU and tensors (the paper's comparison system)."""
    import torch.nn.functional as F
    torch, args = ctx.torch, ctx.args
    I = m["_internal"]
    cases, inst, bufs, n_sets = I["cases"], I["inst"], I["bufs"], I["n_sets"]
    params = {}
    for c in cases:
        params[c.name] = [tuple(torch.from_numpy(getattr(L, f)).to(ctx.dev) for f in ("mean", "var", "gamma", "beta"))
                          if L.kind == "batchnorm" else None for L in c.layers]

    def lbl_step(k):
        row = bufs[k % n_sets]
        for j, c in enumerate(inst):
            xs = row[j][0]
            t = xs[0]
            for L, p in zip(c.layers, params[c.name]):
                if L.kind == "batchnorm":
                    t = F.batch_norm(t, p[0], p[1], p[2], p[3], False, 0.0, L.eps)
                elif L.kind == "relu":
                    t = F.relu(t)
                elif L.kind == "maxpool":
                    t = F.max_pool2d(t, L.kernel, L.stride, L.padding)
                elif L.kind == "avgpool":
                    t = F.avg_pool2d(t, L.kernel, L.stride, L.padding, count_include_pad=L.count_include_pad)
                elif L.kind == "add":
                    t = t + xs[L.operand]
    lsteps = max(3, min(50, args.steps // 4))
    a, b = ctx.event(), ctx.event()
    with torch.cuda.stream(ctx.stream):
        for k in range(3):
            lbl_step(k)
        torch.cuda.synchronize()
        a.record(ctx.stream)
        for k in range(lsteps):
            lbl_step(k)
        b.record(ctx.stream)
    torch.cuda.synchronize()
    lbl_ms = a.elapsed_time(b) / lsteps
    return {"images_per_s": I["batch"] / (lbl_ms / 1e3), "ms_per_step": lbl_ms,
            "fused_speedup": lbl_ms / m["ms_per_step"],
            "what": "torch eager F.batch_norm/relu/max_pool2d/avg_pool2d, one kernel per layer, same GPU"}


def attach_ceiling(m, stacks):
    """The dominant kernel's time against the same-size ideal streaming kernel (per_stack): a
    fraction <= ~1 beside roofline.frac, whose copy-bandwidth peak a 4:1 read-dominated stream can
    exceed."""
    if not stacks:
        return
    for st in stacks:
        if st["stack"] == m["roofline"].get("stack"):
            m["roofline"]["frac_of_ceiling"] = st["frac_of_ceiling"]
            m["roofline"]["ceiling_gbs"] = st["gbs"] / st["frac_of_ceiling"] if st["frac_of_ceiling"] else None
            m["roofline"]["ceiling_variant"] = st["ceiling_variant"]


def per_stack(ctx, m):
    I = m["_internal"]
    return [measure_stack_alone(ctx, c, I["plans"][c.name], I["infos"][c.name]) for c in I["cases"]]


def measure_c1(ctx):
    """configs[0]: the single C1 stack on the GPU (one launch, latency-bound) and the CPU oracle in ms."""
    torch, bs = ctx.torch, ctx.bs
    case = synth.workload("c1")[0]
    plan = bs.bs_plan_create(case.layers, case.shape)
    info = bs.bs_plan_query(plan)
    sb, R = stack_burst(ctx, case, plan, info["alg_bytes_read"] + info["alg_bytes_written"], 13)

    def burst():
        for r in range(R):
            xs, y = sb[r % len(sb)]
            ctx.launch(plan, xs, y)
    gpu_ms = ctx.burst_ms(burst) / R
    out = {"stack": "BN->ReLU->MaxPool2x2/s2 (1,16,32,32)", "gpu_ms_per_launch": gpu_ms,
           "gpu_launch_how": f"{R} back-to-back launches in one CUDA graph, CUDA events"}
    if ctx.rank == 0 and not ctx.args.no_cpu_baseline:
        out["c1_oracle_ms"] = c1_oracle_ms()
        out["c1_oracle_how"] = "oracle_run_bf (plain C, 1 thread, -O2 -ffp-contract=off), min of 5 runs (P:L656-658)"
    return out


def measure_sec51(ctx):
    """PAPER.md §5.1 (NEXT-2): the synthetic network of MaxPool3x3/s1/p1 -> BN -> ReLU blocks on
    (128, 64, 56, 56) as one on-chip sequence (the planner) against one step per sequence (one HBM
    round trip per block), R back-to-back executions over rotating buffers in one CUDA graph."""
    bs = ctx.bs
    out = {"what": "PAPER.md §5.1 blocks MaxPool3x3/s1/p1 -> BN -> ReLU on (128, 64, 56, 56), us per block",
           "rows": []}
    for depth in (16, 40):
        case = synth.synthetic51(depth)
        row = {"depth": depth}
        for policy, name in ((1, "one_step_per_sequence"), (0, "planner")):
            plan = bs.bs_plan_create(case.layers, case.shape, {"max_steps_per_sequence": policy})
            info = bs.bs_plan_query(plan)
            sb, R = stack_burst(ctx, case, plan, info["alg_bytes_read"] + info["alg_bytes_written"], 29)

            def burst():
                for r in range(R):
                    xs, y = sb[r % len(sb)]
                    ctx.launch(plan, xs, y)
            ms = ctx.burst_ms(burst) / R
            row[name] = {"us_per_block": 1e3 * ms / depth, "sequences": info["n_sequences"],
                         "kernel": bs.KERNEL_NAMES[bs.bs_plan_query_launch(plan, 0)["kernel"]]}
            del sb, plan
        row["speedup"] = row["one_step_per_sequence"]["us_per_block"] / row["planner"]["us_per_block"]
        out["rows"].append(row)
    return out


def strip(m):
    return {k: v for k, v in m.items() if not k.startswith("_")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="brainslug", choices=["brainslug", "reference"])
    ap.add_argument("--workload", default="resnet50", choices=list(CONFIG_INDEX))
    ap.add_argument("--batch", type=int, default=0, help="per-rank (weak) / global (strong) batch; 0 = BASELINE.json's")
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--cpu-budget", type=float, default=10.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-lbl", action="store_true", help="skip the torch layer-by-layer context number")
    ap.add_argument("--no-extra", action="store_true", help="skip the other BASELINE workloads")
    ap.add_argument("--no-per-stack", action="store_true", help="skip per-stack / ceiling timings")
    ap.add_argument("--no-validate", action="store_true", help="skip the gathered-shard oracle check")
    ap.add_argument("--out", default="", help="also append the JSON line to this file")
    scal = ap.add_mutually_exclusive_group()
    scal.add_argument("--strong", action="store_true", help="split every workload's BASELINE batch over ranks")
    scal.add_argument("--weak", action="store_true", help="every rank runs its BASELINE batch (also DenseNet-121)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference(args)
    import benchlib
    benchlib.build()

    ctx = Ctx(args)
    do_stacks = not args.no_per_stack and ctx.world == 1
    m = measure(ctx, args.workload, full=True)
    e2e = measure_e2e(ctx, m)
    lbl = measure_lbl(ctx, m) if (not args.no_lbl and ctx.rank == 0) else None
    stacks = per_stack(ctx, m) if do_stacks else None
    attach_ceiling(m, stacks)
    cpu = None
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu_baseline:
        v, n, T = time_oracle(m["_internal"]["cases"], args.cpu_budget, 1 << 20)
        cpu = {"value": v, "unit": "images/s", "cores": 1, "kind": "oracle", "host_cores": os.cpu_count(),
               "host_cpu": _cpu_model(),
               "sample": f"{n} synthetic images shaped like the batch-{m['per_gpu_batch']} {args.workload} workload "
                         f"(all stacks), breadth-first C oracle, single thread, {T:.1f} s"}
        thr = os.cpu_count() or 1
        va, na, Ta = time_oracle_threads(m["_internal"]["cases"], args.cpu_budget / 2, thr)
        cpu["all_cores"] = {"value": va, "unit": "images/s", "threads": thr,
                            "sample": f"{na} images of the same workload, one image per task on {thr} host threads "
                                      f"(the unchanged oracle), {Ta:.1f} s"}
    del m["_internal"]
    extras = {}
    if not args.no_extra:
        for wl in EXTRA_WORKLOADS:
            if wl == args.workload:
                continue
            mw = measure(ctx, wl, full=False)
            if do_stacks:
                mw["per_stack"] = per_stack(ctx, mw)
                attach_ceiling(mw, mw["per_stack"])
            del mw["_internal"]
            extras[wl] = mw
        extras["c1"] = measure_c1(ctx)
        extras["sec51"] = measure_sec51(ctx)

    if ctx.rank == 0:
        line = {
            "metric": METRIC, "value": m["value"], "unit": "images/s", "n_gpus": ctx.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": m["ms_per_step"],
            "ms_per_step_isolated": m.get("ms_per_step_isolated"),
            "higher_is_better": True, "scaling": m["scaling"], "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (SplitMix64 seeded NCHW fp32, BN params per SURVEY §8(d))",
            "config": {"workload": args.workload, "baseline_config_index": CONFIG_INDEX[args.workload],
                       "global_batch": m["global_batch"], "per_gpu_batch": m["per_gpu_batch"],
                       "stacks_per_step": m["stacks_per_step"],
                       "backend": ctx.backend if ctx.world > 1 else None,
                       "parallelism": f"batch-sharded dp{ctx.world} (independent images, no data-path collective)",
                       "launch": "one bs_graph (CUDA graph of every stack) replay per step",
                       "l2": m["l2"]},
            "timing": m["timing"], "hbm": m["hbm"], "roofline": m["roofline"], "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": m["launches_per_step"] * args.steps,
            "clocks": m["clocks"], "layer_by_layer_torch": lbl,
            "checksums": m["checksums"], "outputs_finite": m["outputs_finite"], "validation": m.get("validation"),
            # the paper's own numbers, quoted with their hardware (context, not targets)
            "paper_context": {"best_whole_network_speedup_gpu": "35.7 % (GTX 1080 Ti, PyTorch 0.3.0 + cuDNN, fp32)",
                              "best_whole_network_speedup_cpu": "41.1 % (Xeon E5-2690v4, ISPC + TBB)",
                              "synthetic_blocks_gpu": "1.4-2.2x vs PyTorch (GTX 1080 Ti)",
                              "source": "PAPER.md P:L27-29, P:L689, P:L953"},
            "per_stack": stacks,
            "workloads": extras,
        }
        s = json.dumps(line)
        print(s, flush=True)
        if args.out:
            with open(args.out, "a") as f:
                f.write(s + "\n")
    if ctx.world > 1:
        ctx.dist.destroy_process_group()


if __name__ == "__main__":
    main()
