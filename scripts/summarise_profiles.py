"""Summarise the ncu evidence collected by scripts/profile_round.sh into profiles/.

usage: python scripts/summarise_profiles.py ROUND   (reads gpurun_out/prof/, writes profiles/)
"""
import csv
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
SRC = os.path.join(ROOT, "gpurun_out", "prof")
DST = os.path.join(ROOT, "profiles")
rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
os.makedirs(DST, exist_ok=True)

KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "dram_read"),
        ("dram__bytes_write.sum", "dram_write"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_of_nominal"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"),
        ("launch__block_size", "block"), ("sm__warps_active.avg.per_cycle_active", "warps_per_sm"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
        ("lts__t_bytes.sum", "l2_bytes"), ("smsp__inst_executed.sum", "warp_instructions"),
        ("launch__shared_mem_per_block_dynamic", "dyn_smem"),
        ("smsp__sass_inst_executed_op_tma_ld.sum", "tma_bulk_loads")]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "nsecond": 1e-9, "msecond": 1e-3,
         "us": 1e-6, "ns": 1e-9, "ms": 1e-3, "KB": 1e3, "MB": 1e6, "GB": 1e9}


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
                    d[name] = float(v[i].replace(",", "")) * SCALE.get(u[i], 1)
                except ValueError:
                    d[name] = v[i]
        stalls = {x.split("stalled_")[1]: float(v[i]) for i, x in enumerate(h)
                  if x.startswith("smsp__pcsamp_warps_issue_stalled_") and not x.endswith("not_issued")
                  and v[i] not in ("", "n/a")}
        tot = sum(stalls.values()) or 1
        d["top_stalls"] = {k: round(100 * s / tot, 1) for k, s in sorted(stalls.items(), key=lambda kv: -kv[1])[:4]}
        out.append(d)
    return out


summary, traffic = [], {}
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
for f in sorted(os.listdir(SRC)):
    if not f.endswith(".raw.csv"):
        continue
    wl, idx = f[len("full_"):-len(".raw.csv")].rsplit("_", 1)
    case = synth.workload(wl)[int(idx)]
    import paper_1804_08378_b200 as bs
    info = bs.bs_plan_query(bs.bs_plan_create(case.layers, case.shape, {"host_only": 1}))
    alg = info["alg_bytes_read"] + info["alg_bytes_written"]
    for d in read_raw(os.path.join(SRC, f)):
        d.update({"workload": wl, "stack": case.name, "shape": list(case.shape), "alg_bytes": alg,
                  "dram_bytes": d.get("dram_read", 0) + d.get("dram_write", 0)})
        d["traffic_over_alg"] = d["dram_bytes"] / alg
        d["alg_gbs_under_ncu"] = alg / d["duration"] / 1e9
        d["frac_of_measured_copy"] = d["alg_gbs_under_ncu"] / peaks["hbm_gbs"]
        summary.append(d)
        traffic[f"{wl}:{case.name}"] = {"dram_bytes_per_launch": d["dram_bytes"], "alg_bytes_per_launch": alg,
                                        "source": f"profiles/{rnd}_ncu_full_summary.json (ncu --set full, 1 launch)"}
    shutil.copy(os.path.join(SRC, f.replace(".raw.csv", ".details.csv")),
                os.path.join(DST, f"{rnd}_{f.replace('.raw.csv', '.details.csv')}"))

json.dump(summary, open(os.path.join(DST, f"{rnd}_ncu_full_summary.json"), "w"), indent=1)
json.dump(traffic, open(os.path.join(DST, "ncu_traffic.json"), "w"), indent=1)
if os.path.exists(os.path.join(SRC, "full_alexnet_0.raw.csv")):
    shutil.copy(os.path.join(SRC, "full_alexnet_0.raw.csv"), os.path.join(DST, f"{rnd}_full_alexnet_0.raw.csv"))

# launch list of the default bench: per-kernel share of device time
lines = [l for l in open(os.path.join(SRC, "launches_alexnet.csv")) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
launches = {}
for r in rows[1:]:
    key = (r[h.index("ID")], r[ki])
    launches.setdefault(key, {})[r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
# only this library's kernels (the bench's own data fills and checksums are torch kernels);
# one step = one launch of each stack, in order: share of each stack in the step
ours = [(int(lid), k, m) for (lid, k), m in launches.items() if "bs::" in k]
ours.sort()
cases = synth.workload("alexnet")
ours = ours[: 6 * len(cases)]   # 3 warm-up + 3 timed steps, stacks in order (bursts/e2e follow)
grid_of = {}
for r in rows[1:]:
    grid_of[int(r[h.index("ID")])] = r[h.index("Grid Size")]
per = {}
for n, (lid, k, m) in enumerate(ours):
    st = cases[n % len(cases)].name
    t = per.setdefault(st, [0, 0.0, 0.0, k.split("(")[0]])
    t[0] += 1
    t[1] += m.get("gpu__time_duration.sum", 0)
    t[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
alltime = sum(t[1] for t in per.values())
with open(os.path.join(DST, f"{rnd}_ncu_launches_alexnet.txt"), "w") as fo:
    fo.write("ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none\n"
             "python bench.py --steps 3 --warmup 3 --no-graph (default workload: AlexNet, batch 128)\n"
             "this library's launches of the 3 warm-up + 3 timed steps; cold-cache, serialised: compare SHARES\n\n")
    fo.write(f"{'stack':14s} {'kernel':40s} {'launches':>8s} {'avg_us':>8s} {'share':>7s} {'dram_MB/launch':>15s}\n")
    for st, (n, t, b, kn) in per.items():
        fo.write(f"{st:14s} {kn[:40]:40s} {n:8d} {t * 1e6 / n:8.1f} {100 * t / alltime:6.1f}% {b / n / 1e6:15.1f}\n")

with open(os.path.join(DST, f"{rnd}_ncu_full_summary.md"), "w") as fo:
    fo.write(f"# {rnd}: ncu --set full, one launch of each workload's dominant kernel(s)\n\n")
    fo.write("Captured with `scripts/profile_round.sh` (`ncu --set full --clock-control none --import-source on`,\n"
             "1 launch after 2 warm-up launches, `scripts/prof_one.py`).  `traffic/alg` = DRAM bytes read+written\n"
             "/ algorithmic bytes (one read of the input + one write of the output).  GB/s here is under the\n"
             "profiler (cache flushed, serialised); bench.py's numbers are the measured ones.\n\n")
    fo.write("| stack | kernel | us | DRAM MB | alg MB | traffic/alg | alg GB/s | frac of copy | regs | warps/SM | issue % | top stalls |\n")
    fo.write("|---|---|---|---|---|---|---|---|---|---|---|---|\n")
    for d in summary:
        fo.write(f"| {d['stack']} {tuple(d['shape'])} | `{d['kernel'][:48]}` | {d['duration'] * 1e6:.1f} | "
                 f"{d['dram_bytes'] / 1e6:.1f} | {d['alg_bytes'] / 1e6:.1f} | {d['traffic_over_alg']:.3f} | "
                 f"{d['alg_gbs_under_ncu']:.0f} | {d['frac_of_measured_copy']:.3f} | {int(d.get('regs', 0))} | "
                 f"{d.get('warps_per_sm', 0):.1f} | {d.get('issue_active_pct', 0):.0f} | "
                 f"{', '.join(f'{k} {v}%' for k, v in d['top_stalls'].items())} |\n")
print(open(os.path.join(DST, f"{rnd}_ncu_full_summary.md")).read())
print(open(os.path.join(DST, f"{rnd}_ncu_launches_alexnet.txt")).read())
