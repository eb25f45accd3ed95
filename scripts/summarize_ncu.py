"""Summarise ncu outputs (from gpurun_out/) into committed profiles/ files.

    python scripts/summarize_ncu.py --launches gpurun_out/launches.csv \
        --rep gpurun_out/prof.ncu-rep --tag r1a

Writes profiles/launches_<tag>.md (per-kernel device-time shares of the
timed step) and profiles/ncu_<tag>.md + profiles/ncu_summary.json (per-launch
dram bytes, tensor-pipe utilisation, ... of the fully profiled launches).
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "launch__shared_mem_per_block_dynamic": "smem_dyn",
}
UNIT = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
        "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def to_num(v: str, unit: str):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    return x * UNIT.get(unit, 1)


def launches(path: str, tag: str):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    seq = []
    for r in rows[hi + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            seq.append((r[ki], to_num(r[vi], r[ui])))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for n, t in seq:
        short = re.sub(r"\(.*", "", n)[:90]
        tot[short] += t
        cnt[short] += 1
    T = sum(tot.values())
    lines = [f"# Launch list `{tag}` (ncu gpu__time_duration, --clock-control none; cold-cache, serialised)",
             "", f"source: `{os.path.basename(path)}`, {len(seq)} launches, total {T * 1e3:.3f} ms", "",
             "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| `{k}` | {cnt[k]} | {v * 1e3:.3f} | {v / T:.3f} |")
    ours = [(n, t) for n, t in seq if "pdl::" in n]
    lines += ["", "Our kernels in launch order (ms):", "",
              ", ".join(f"{t * 1e3:.3f}" for _, t in ours)]
    out = os.path.join(ROOT, "profiles", f"launches_{tag}.md")
    open(out, "w").write("\n".join(lines) + "\n")
    return out


def rep(path: str, tag: str, names: list[str] | None):
    if path.endswith(".csv"):  # `ncu -i x.ncu-rep --page raw --csv` exported on the GPU box
        raw = open(path).read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    kn = hdr.index("Kernel Name")
    res = []
    for j, r in enumerate(rows[2:]):
        d = {"kernel": re.sub(r"\(.*", "", r[kn])}
        for m, short in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                d[short] = to_num(r[i], units[i])
        if names and j < len(names):
            d["tag"] = names[j]
        d["dram_bytes"] = (d.get("dram_read") or 0) + (d.get("dram_write") or 0)
        res.append(d)
    lines = [f"# ncu --set full `{tag}`", "", f"source: `{os.path.basename(path)}`", "",
             "| launch | kernel | ms | dram R+W MB | tensor pipe % | dram % | SM thru % | regs | grid | smem bank confl |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    for d in res:
        lines.append(f"| {d.get('tag', '')} | `{d['kernel'][:60]}` | {d.get('duration', 0) * 1e3:.3f} | "
                     f"{d['dram_bytes'] / 1e6:.1f} | {d.get('tensor_pipe_pct', '')} | {d.get('dram_pct', '')} | "
                     f"{d.get('sm_throughput_pct', '')} | {d.get('regs', '')} | {d.get('grid', '')} | "
                     f"{d.get('smem_bank_conflicts', '')} |")
    open(os.path.join(ROOT, "profiles", f"ncu_{tag}.md"), "w").write("\n".join(lines) + "\n")
    summ_p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summ = json.load(open(summ_p)) if os.path.exists(summ_p) else {"kernels": {}}
    for d in res:
        if "tag" in d:
            summ["kernels"][d["tag"]] = {"dram_bytes": d["dram_bytes"], "tensor_pipe_pct": d.get("tensor_pipe_pct"),
                                         "duration_s": d.get("duration"), "source": f"ncu_{tag}.md"}
    json.dump(summ, open(summ_p, "w"), indent=1)
    return res


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--names", default="", help="comma-separated tags for the profiled launches")
    a = ap.parse_args()
    if a.launches:
        print(launches(a.launches, a.tag))
    if a.rep:
        for d in rep(a.rep, a.tag, [n for n in a.names.split(",") if n]):
            print(d)
