"""Summarise ncu output into profiles/ (committed evidence).

  python tools/ncu_summary.py full <report.ncu-rep> <out.md> [algorithmic_bytes_per_launch]
  python tools/ncu_summary.py launches <launches.csv> <out.md>

`full`: key Speed-of-Light / memory / occupancy / stall metrics of every
profiled kernel, plus DRAM traffic vs the algorithmic bytes when given.
`launches`: per-kernel launch counts and time shares of a
`--metrics gpu__time_duration.sum` run (cold-cache, serialised: compare
shares, not absolutes).
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_shared_mem", "CTA/SM limit (smem)"),
    ("launch__occupancy_limit_registers", "CTA/SM limit (regs)"),
    ("launch__grid_size", "grid"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("smsp__average_warp_latency_issue_stalled_long_scoreboard", "stall long_scoreboard"),
    ("smsp__average_warp_latency_issue_stalled_barrier", "stall barrier"),
    ("smsp__average_warp_latency_issue_stalled_short_scoreboard", "stall short_scoreboard"),
]


def _raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def full(report, out_md, algo_bytes=None):
    hdr, units, rows = _raw(report)
    idx = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu --set full summary: `{report}`", ""]
    data = []
    for r in rows:
        name = r[idx["Kernel Name"]]
        rec = {"kernel": name}
        lines.append(f"## {name}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for key, label in KEYS:
            if key in idx:
                lines.append(f"| {label} (`{key}`) | {r[idx[key]]} | {units[idx[key]]} |")
                rec[key] = r[idx[key]]
        if algo_bytes and "dram__bytes_read.sum" in idx:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd = float(r[idx["dram__bytes_read.sum"]]) * scale.get(units[idx["dram__bytes_read.sum"]], 1)
            wr = float(r[idx["dram__bytes_write.sum"]]) * scale.get(units[idx["dram__bytes_write.sum"]], 1)
            lines.append(f"| DRAM traffic / algorithmic bytes | {(rd + wr) / float(algo_bytes):.3f} | ratio |")
            rec["dram_bytes_per_launch"] = rd + wr
            rec["algorithmic_bytes"] = float(algo_bytes)
        lines.append("")
        data.append(rec)
    with open(out_md, "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(out_md.rsplit(".", 1)[0] + ".json", "w") as f:
        json.dump(data, f, indent=1)
    print("\n".join(lines))


def launches(csv_path, out_md):
    text = open(csv_path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) < len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[idx["Kernel Name"]].split("(")[0]
        val = float(r[idx["Metric Value"]].replace(",", ""))
        unit = r[idx["Metric Unit"]]
        val *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
        tot[name] += val
        cnt[name] += 1
    total = sum(tot.values())
    lines = [f"# launch list: `{csv_path}` (ncu gpu__time_duration, cold-cache, serialised)", "",
             "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for name in sorted(tot, key=lambda n: -tot[n]):
        lines.append(f"| `{name}` | {cnt[name]} | {tot[name]:.1f} | {tot[name] / total:.3f} |")
    with open(out_md, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
    else:
        launches(sys.argv[2], sys.argv[3])
