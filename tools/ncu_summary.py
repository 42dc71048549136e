"""Summarise ncu captures into profiles/ (tracked).

    python tools/ncu_summary.py TAG rep1.ncu-rep [rep2 ...] [--launches launches.csv]

Writes profiles/ncu_TAG.md (per-kernel metrics, stall mix, launch-time
shares) and merges per-kernel numbers into profiles/ncu_summary.json, which
bench.py reads for the roofline `traffic` field (dram bytes per launch).
"""
from __future__ import annotations

import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__occupancy_limit_registers", "occupancy limit (regs, blocks)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
              "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}


def ncu_csv(rep: str, page: str, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def raw_metrics(rep: str) -> dict:
    rows = ncu_csv(rep, "raw")
    head, units, vals = rows[0], rows[1], rows[2]
    out = {"kernel": vals[head.index("Kernel Name")]}
    for key, _ in METRICS:
        if key in head:
            i = head.index(key)
            out[key] = (vals[i], units[i])
    return out


def stall_mix(rep: str) -> list:
    rows = ncu_csv(rep, "source", ["--print-source", "sass"])
    head, data = rows[1], rows[2:]
    cols = [i for i, n in enumerate(head) if n.startswith("stall_") and "Not Issued" not in n]
    agg = {head[i][6:]: sum(float(r[i] or 0) for r in data if len(r) > i) for i in cols}
    tot = sum(agg.values()) or 1.0
    return [(k, round(v / tot, 3)) for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:6]]


def to_si(val: str, unit: str) -> float:
    v = float(val.replace(",", ""))
    return v * UNIT_SCALE.get(unit, 1.0)


def launch_shares(path: str) -> list:
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    H = rows[h]
    ki, vi, ui = H.index("Kernel Name"), H.index("Metric Value"), H.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[h + 1:]:
        if len(r) > vi:
            agg[r[ki].split("(")[0].replace("<unnamed>::", "")].append(to_si(r[vi], r[ui]))
    tot = sum(sum(v) for v in agg.values())
    return sorted(((k, len(v), sum(v), sum(v) / tot) for k, v in agg.items()), key=lambda t: -t[2])


def main(argv):
    tag = argv[0]
    reps = [a for a in argv[1:] if a.endswith(".ncu-rep")]
    launches = argv[argv.index("--launches") + 1] if "--launches" in argv else None
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    summary_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summary = json.load(open(summary_path)) if os.path.exists(summary_path) else {}
    lines = [f"# ncu summary — {tag}", "",
             "Captured with `ncu --set full --clock-control none --import-source on` on one B200 "
             "(launch: `python bench.py --steps 3 --warmup 3 --no-cpu`); cold-cache, serialised replays.", ""]
    for rep in reps:
        m = raw_metrics(rep)
        name = m["kernel"].split("(")[0].replace("<unnamed>::", "").split("<")[0].replace("void ", "").strip()
        lines.append(f"## `{m['kernel'][:120]}`")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for key, label in METRICS:
            if key in m:
                lines.append(f"| {label} (`{key}`) | {m[key][0]} {m[key][1]} |")
        st = stall_mix(rep)
        lines.append(f"| top stall reasons (share of samples) | {', '.join(f'{k} {v}' for k, v in st)} |")
        lines.append("")
        rd = to_si(*m["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in m else None
        wr = to_si(*m["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in m else None
        dur = to_si(*m["gpu__time_duration.sum"]) if "gpu__time_duration.sum" in m else None
        summary[name] = {"tag": tag, "dram_bytes_per_launch": (rd or 0) + (wr or 0), "dram_read": rd,
                         "dram_write": wr, "duration_s": dur, "stalls": st}
    if launches:
        lines.append("## Launch list (`--metrics gpu__time_duration.sum`), share of device time")
        lines.append("")
        lines.append("| kernel | launches | total | share |")
        lines.append("|---|---|---|---|")
        for k, n, t, sh in launch_shares(launches):
            lines.append(f"| `{k[:70]}` | {n} | {t * 1e6:.1f} us | {100 * sh:.1f}% |")
        lines.append("")
    with open(os.path.join(ROOT, "profiles", f"ncu_{tag}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(summary_path, "w") as f:
        json.dump(summary, f, indent=1, sort_keys=True)
    print("wrote", f"profiles/ncu_{tag}.md")


if __name__ == "__main__":
    main(sys.argv[1:])
