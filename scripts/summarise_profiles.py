"""Summarise the evidence collected by scripts/gpu_evidence.sh into profiles/.

usage: python scripts/summarise_profiles.py TAG   (reads gpurun_out/TAG/, writes profiles/TAG/ and
profiles/ncu_traffic.json keyed by the hash of the kernel sources the capture was made from)
"""
import csv
import glob
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402  (kernel_sources_hash only)
import synth  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r02_final"
SRC = os.path.join(ROOT, "gpurun_out", tag)
DST = os.path.join(ROOT, "profiles", tag)
os.makedirs(DST, exist_ok=True)

KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "dram_read"),
        ("dram__bytes_write.sum", "dram_write"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_of_nominal"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"),
        ("launch__block_size", "block"), ("sm__warps_active.avg.per_cycle_active", "warps_per_sm"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
        ("smsp__inst_executed.sum", "warp_instructions"),
        ("launch__shared_mem_per_block_dynamic", "dyn_smem")]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "nsecond": 1e-9, "msecond": 1e-3,
         "us": 1e-6, "ns": 1e-9, "ms": 1e-3, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def val(v, unit):
    return float(v.replace(",", "")) * SCALE.get(unit, 1)


def read_raw(path):
    rows = list(csv.reader(open(path)))
    h, u = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")]}
        for k, name in KEYS:
            if k in h:
                i = h.index(k)
                try:
                    d[name] = val(v[i], u[i])
                except ValueError:
                    d[name] = v[i]
        stalls = {x.split("stalled_")[1]: float(v[i]) for i, x in enumerate(h)
                  if x.startswith("smsp__pcsamp_warps_issue_stalled_") and not x.endswith("not_issued")
                  and v[i] not in ("", "n/a")}
        tot = sum(stalls.values()) or 1
        d["top_stalls"] = {k: round(100 * s / tot, 1) for k, s in sorted(stalls.items(), key=lambda kv: -kv[1])[:4]}
        out.append(d)
    return out


def read_metrics_csv(path):
    """ncu --csv --metrics ... log: one row per (launch, metric) -> {launch id: {metric: value, kernel}}."""
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                          h.index("Metric Unit"), h.index("ID"))
    out = {}
    for r in rows[1:]:
        d = out.setdefault(int(r[ii]), {"kernel": r[ki]})
        d[r[mi]] = val(r[vi], r[ui])
    return out


import paper_1804_08378_b200 as bs  # noqa: E402
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))


def alg_bytes(case):
    info = bs.bs_plan_query(bs.bs_plan_create(case.layers, case.shape, {"host_only": 1}))
    return info["alg_bytes_read"] + info["alg_bytes_written"]


# ---- full captures
summary = []
for f in sorted(glob.glob(os.path.join(SRC, "full_*.raw.csv"))):
    name = os.path.basename(f)[len("full_"):-len(".raw.csv")]
    if name == "seq16":
        case = synth.synthetic51(16)
    else:
        wl, idx = name.rsplit("_", 1)
        case = synth.workload(wl)[int(idx)]
    alg = alg_bytes(case)
    for d in read_raw(f):
        d.update({"capture": name, "stack": case.name, "shape": list(case.shape), "alg_bytes": alg,
                  "dram_bytes": d.get("dram_read", 0) + d.get("dram_write", 0)})
        d["traffic_over_alg"] = d["dram_bytes"] / alg
        d["alg_gbs_under_ncu"] = alg / d["duration"] / 1e9
        d["frac_of_measured_copy"] = d["alg_gbs_under_ncu"] / peaks["hbm_gbs"]
        if name == "seq16":   # instructions per output of the 16-step sequence
            outs = 16 * int(__import__("numpy").prod(case.shape))
            d["thread_instructions_per_output"] = 32 * d.get("warp_instructions", 0) / outs
        summary.append(d)
    shutil.copy(f.replace(".raw.csv", ".details.csv"), os.path.join(DST, os.path.basename(f).replace(".raw.csv", ".details.csv")))
if summary:
    json.dump(summary, open(os.path.join(DST, "ncu_full_summary.json"), "w"), indent=1)

# ---- DRAM traffic of each workload's dominant stack (cold cache), keyed by kernel-source hash
traffic = {"sources_sha16": bench.kernel_sources_hash(), "captured": tag,
           "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none (cache flushed "
                  "between launches), scripts/prof_one.py WORKLOAD IDX 3: median of the 3 launches", "entries": {}}
for f in sorted(glob.glob(os.path.join(SRC, "traffic_*.csv"))):
    wl, idx = os.path.basename(f)[len("traffic_"):-len(".csv")].rsplit("_", 1)
    case = synth.workload(wl)[int(idx)]
    ls = [d for d in read_metrics_csv(f).values() if "bs::" in d["kernel"]]
    if not ls:
        continue
    db = sorted(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in ls)[len(ls) // 2]
    alg = alg_bytes(case)
    traffic["entries"][f"{wl}:{case.name}"] = {"dram_bytes_per_launch": db, "alg_bytes_per_launch": alg,
                                               "ratio": db / alg, "kernel": ls[0]["kernel"].split("(")[0]}
json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)

# ---- launch list of the default bench (resnet50): per-kernel share of the step
lp = os.path.join(SRC, "launches_resnet50.csv")
if os.path.exists(lp):
    ls = sorted((lid, d) for lid, d in read_metrics_csv(lp).items() if "bs::" in d["kernel"])
    cases = synth.instances(synth.workload("resnet50")) if hasattr(synth, "instances") else None
    inst = []
    for c in synth.workload("resnet50"):
        inst += [c] * c.count
    step = ls[: 3 * len(inst)]           # the 3 eager warm-up steps: stacks in order
    per = {}
    for n, (lid, d) in enumerate(step):
        st = inst[n % len(inst)].name
        t = per.setdefault(st, [0, 0.0, 0.0, d["kernel"].split("(")[0]])
        t[0] += 1
        t[1] += d.get("gpu__time_duration.sum", 0)
        t[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    tot = sum(t[1] for t in per.values())
    with open(os.path.join(DST, "ncu_launches_resnet50.txt"), "w") as fo:
        fo.write("ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none\n"
                 "python bench.py --steps 2 --warmup 3 --no-extra ... (default workload ResNet-50, batch 256)\n"
                 "this library's launches of the 3 eager warm-up steps; cold-cache, serialised: compare SHARES\n\n")
        fo.write(f"{'stack':26s} {'kernel':28s} {'launches':>8s} {'avg_us':>8s} {'share':>7s} {'dram_MB/launch':>15s}\n")
        for st, (n, t, b, kn) in per.items():
            fo.write(f"{st:26s} {kn[:28]:28s} {n:8d} {t * 1e6 / n:8.1f} {100 * t / tot:6.1f}% {b / n / 1e6:15.1f}\n")

with open(os.path.join(DST, "ncu_full_summary.md") if summary else os.devnull, "w") as fo:
    fo.write(f"# {tag}: ncu --set full, one launch of each captured kernel\n\n")
    fo.write("`scripts/gpu_evidence.sh` (`ncu --set full --clock-control none --import-source on`, 1 launch after 1\n"
             "warm-up launch).  traffic/alg = DRAM bytes read+written / algorithmic bytes (one read of the input +\n"
             "one write of the output).  GB/s here is under the profiler (cache flushed, serialised); bench.py's\n"
             "numbers are the measured ones.\n\n")
    fo.write("| capture | stack | kernel | us | DRAM MB | alg MB | traffic/alg | alg GB/s | regs | warps/SM | issue % | top stalls |\n")
    fo.write("|---|---|---|---|---|---|---|---|---|---|---|---|\n")
    for d in summary:
        extra = f" ({d['thread_instructions_per_output']:.1f} instr/output)" if "thread_instructions_per_output" in d else ""
        fo.write(f"| {d['capture']} | {d['stack']} {tuple(d['shape'])} | `{d['kernel'].split('(')[0][:40]}`{extra} | "
                 f"{d['duration'] * 1e6:.1f} | {d['dram_bytes'] / 1e6:.1f} | {d['alg_bytes'] / 1e6:.1f} | "
                 f"{d['traffic_over_alg']:.3f} | {d['alg_gbs_under_ncu']:.0f} | {int(d.get('regs', 0))} | "
                 f"{d.get('warps_per_sm', 0):.1f} | {d.get('issue_active_pct', 0):.0f} | "
                 f"{', '.join(f'{k} {v}%' for k, v in d['top_stalls'].items())} |\n")
for f in ("bench_default.json", "bench_2rank_gloo.json", "bench_reference.json", "sec51_56.jsonl", "sec51_64.jsonl", "sec51_112.jsonl",
          "sec51_224.jsonl", "sec51_224_budget110k.jsonl", "pytest_gpu.log", "smoke.log", "gpu.txt", "nproc.txt", "sanitize_rc.txt"):
    if os.path.exists(os.path.join(SRC, f)):
        shutil.copy(os.path.join(SRC, f), os.path.join(DST, f))
for f in glob.glob(os.path.join(SRC, "sanitize_*.log")):
    shutil.copy(f, os.path.join(DST, os.path.basename(f)))
if summary:
    print(open(os.path.join(DST, "ncu_full_summary.md")).read())
if os.path.exists(os.path.join(DST, "ncu_launches_resnet50.txt")):
    print(open(os.path.join(DST, "ncu_launches_resnet50.txt")).read())
print(json.dumps(traffic, indent=1))
