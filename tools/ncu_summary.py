#!/usr/bin/env python
"""Summarise an ncu capture (.ncu-rep) of the reconstruction kernel for profiles/.

    python tools/ncu_summary.py gpurun_out/prof_C2.ncu-rep --config C2 --tag r01 \
        [--launches gpurun_out/launches_C2.csv] [--bench gpurun_out/bench_default.json]

Writes profiles/<tag>_<config>_ncu.md (metrics, top warp-stall SASS lines) and
updates profiles/ncu_traffic.json ("<config>:<kernel variant>" -> DRAM bytes per
launch), which bench.py reports as roofline.traffic.
"""
import argparse
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/smem throughput %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def ncu_csv(rep, *args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def to_bytes(v, unit):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--config", required=True)
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--kernel", default="pipelined")
    ap.add_argument("--launches")
    ap.add_argument("--bench")
    ap.add_argument("--cells", type=int, default=0, help="proxy mesh: cells of the captured launch (no traffic key)")
    ap.add_argument("--cmd", default=None, help="command line of the capture (for the header)")
    a = ap.parse_args()
    proxy = a.config.endswith("proxy")

    rows = ncu_csv(a.rep, "--page", "raw")
    hdr, units, vals = rows[0], rows[1], rows[2]
    get = {k: (vals[hdr.index(k)], units[hdr.index(k)]) for k, _ in METRICS if k in hdr}
    kname = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    rd = to_bytes(*get["dram__bytes_read.sum"])
    wr = to_bytes(*get["dram__bytes_write.sum"])
    dur_ns = float(get["gpu__time_duration.sum"][0]) * {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}[
        get["gpu__time_duration.sum"][1]]

    import gen
    from paper_1612_09335_b200 import n_modes
    cfg = gen.CONFIGS[a.config.replace("proxy", "")]
    d, M = cfg["d"], cfg["M"]
    V = gen.nvars_of(cfg["ic"])
    nm = n_modes(M, d)
    ne = d * nm
    bcell = 8 * ((nm - 1) * (ne - 1) + (d + 1) * d * d) + 4 * (ne - 1) + (d + 1) * d + 8 * V + 8 * nm * V
    n = cfg["n"]
    ncell = a.cells or (2 * n * n if d == 2 else 6 * n ** 3)
    alg = bcell * ncell

    src = ncu_csv(a.rep, "--page", "source", "--print-source", "sass")
    top = []
    if len(src) > 2:
        sh = src[1]
        si = sh.index("Warp Stall Sampling (All Samples)")
        data = [r for r in src[2:] if len(r) > si and r[si].isdigit()]
        tot = sum(int(r[si]) for r in data)
        for r in sorted(data, key=lambda r: -int(r[si]))[:12]:
            top.append((int(r[si]), 100.0 * int(r[si]) / max(tot, 1), r[1].strip()))
    stalls = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(vals[i]))
              for i, k in enumerate(hdr) if k.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not k.endswith("_not_issued") and vals[i] not in ("", "n/a")]
    stot = sum(v for _, v in stalls) or 1.0
    stalls = sorted(stalls, key=lambda x: -x[1])[:8]

    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    lines = [f"# ncu --set full: {kname} — {a.config} ({a.tag})", "",
             f"Capture: `ncu --set full --clock-control none --import-source on -k \"regex:k_pipelined|k_rowblk\" -s 3 -c 1 "
             + (a.cmd or f"python bench.py --config {a.config} --steps 3 --warmup 3 --no-cpu-baseline") + "` on one B200 "
             f"(cold L2, serialised; per-launch numbers).", "",
             "| metric | value |", "|---|---|"]
    for k, label in METRICS:
        if k in get:
            lines.append(f"| {label} (`{k}`) | {get[k][0]} {get[k][1]} |")
    lines += ["", f"Algorithmic bytes per launch (B_cell = {bcell} B × {ncell} cells): {alg / 1e6:.1f} MB; "
              f"DRAM traffic read+write {(rd + wr) / 1e6:.1f} MB = {(rd + wr) / alg:.3f} × algorithmic.",
              f"Algorithmic bandwidth at the ncu duration: {alg / dur_ns:.0f} GB/s.", "",
              "Warp-stall samples (all warps, whole kernel):", "",
              "| reason | share |", "|---|---|"]
    lines += [f"| {k} | {100 * v / stot:.1f}% |" for k, v in stalls]
    lines += ["", "Top SASS lines by stall samples:", "", "| samples | share | SASS |", "|---|---|---|"]
    lines += [f"| {n_} | {p:.1f}% | `{s}` |" for n_, p, s in top]
    if a.launches and os.path.exists(a.launches):
        lr = [r for r in csv.reader(open(a.launches)) if len(r) > 10]
        h = lr[0]
        per = {}
        for r in lr[1:]:
            try:
                per.setdefault(r[h.index("Kernel Name")], []).append(float(r[h.index("Metric Value")]))
            except ValueError:
                pass
        tot = sum(sum(v) for v in per.values())
        lines += ["", f"Launch list (`ncu --metrics gpu__time_duration.sum`, {a.launches.split('/')[-1]}): "
                  "every kernel of `bench.py --steps 3 --warmup 3` (3 warm-up + 3 timed passes, 5 e2e passes of 4 tile ranges each (cwreco_reconstruct_host), "
                  "3 L2-flush fills):", "", "| kernel | launches | mean µs | share of device time |",
                  "|---|---|---|---|"]
        for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| `{k[:70]}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {100 * sum(v) / tot:.1f}% |")
    if a.bench and os.path.exists(a.bench):
        b = json.loads(open(a.bench).read().strip().splitlines()[-1])
        lines += ["", "Bench line of the same build (CUDA events, L2 flushed between passes):", "",
                  "```", json.dumps(b), "```"]
    out = os.path.join(ROOT, "profiles", f"{a.tag}_{a.config}_ncu.md")
    open(out, "w").write("\n".join(lines) + "\n")
    if proxy:
        print(out)
        return
    tj = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    t = json.load(open(tj)) if os.path.exists(tj) else {}
    m = re.search(r"(k_[a-z_]+)", kname)      # keyed by the captured kernel (bench.py reads "<cfg>:<symbol>")
    t[f"{a.config}:{m.group(1) if m else a.kernel}"] = int(rd + wr)
    json.dump(t, open(tj, "w"), indent=1, sort_keys=True)
    print(out)


if __name__ == "__main__":
    main()
