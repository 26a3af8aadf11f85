"""Summaries of ncu exports for profiles/ (committed evidence).

    # launch list (gpu__time_duration per launch, --csv --log-file X):
    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/rNN_launches.md
    # full capture (ncu -i X.ncu-rep --page raw --csv --print-units base):
    python tools/ncu_summary.py full gpurun_out/full_raw.csv profiles/ncu_traffic.json > profiles/rNN_ncu_full.md
"""
import collections
import csv
import json
import re
import sys


def short(name):
    name = name.replace("lrc::", "").replace("void ", "").replace("(bool)", "").replace("(int)", "")
    name = re.sub(r"\((?!.*<).*$", "", name)
    m = re.match(r"tiled_kernel<(\d), *(\d)>", name)
    if m:
        return f"tiled_kernel<{'UP' if m.group(1) == '1' else 'DOWN'}, NQ={m.group(2)}>"
    return name


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(r for r in rows if "Kernel Name" in r)
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    per = collections.defaultdict(list)
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) == len(hdr) and r[mi] == "gpu__time_duration.sum":
            per[short(r[ki])].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in per.values()) or 1.0
    print("| kernel | launches | avg duration | share of kernel time |")
    print("|---|---:|---:|---:|")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        unit = "ns"
        print(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.2f} us | {sum(v) / tot * 100:.1f}% |" if unit else "")
    print(f"\nTotal kernel time in the capture: {tot / 1e3:.1f} us over {sum(len(v) for v in per.values())} launches "
          "(ncu serialises launches and runs them cold-cache: compare shares, not absolutes).")


KEYS = [
    ("gpu__time_duration.sum", "duration (ns)"),
    ("dram__bytes_read.sum", "DRAM read (B)"),
    ("dram__bytes_write.sum", "DRAM write (B)"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput (% peak)"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput (% peak)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput (% peak)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active (%)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active (%)"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe active (%)"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy (%)"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def full(path, traffic_out=None):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = rows[0]
    data = [r for r in rows[1:] if len(r) == len(hdr) and r[hdr.index("Kernel Name")] != ""]
    data = [r for r in data if not r[0].startswith("ID") and r[hdr.index("Kernel Name")] != "Kernel Name"]
    # drop the units row if present
    data = [r for r in data if not all(c in ("", "ns", "byte", "%", "register/thread") for c in r[5:10])]
    print("| metric | " + " | ".join(f"`{short(r[hdr.index('Kernel Name')])}`" for r in data) + " |")
    print("|---|" + "---:|" * len(data))
    for key, label in KEYS:
        if key not in hdr:
            continue
        vals = [r[hdr.index(key)] for r in data]
        print(f"| {label} | " + " | ".join(vals) + " |")
    stall_keys = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith(
        "_per_issue_active.ratio") and "not_issued" not in h]
    print("\nTop issue-stall reasons (warps per issue-active cycle):\n")
    for r in data:
        st = sorted(((float(r[hdr.index(h)] or 0), h.split("stalled_")[1].replace("_per_issue_active.ratio", ""))
                     for h in stall_keys), reverse=True)[:5]
        print(f"- `{short(r[hdr.index('Kernel Name')])}`: " + ", ".join(f"{n} {v:.2f}" for v, n in st))
    if traffic_out:
        tr = {}
        for r in data:
            n = short(r[hdr.index("Kernel Name")])
            b = float(r[hdr.index("dram__bytes_read.sum")] or 0) + float(r[hdr.index("dram__bytes_write.sum")] or 0)
            key = "up" if "UP" in n else ("down" if "DOWN" in n else n)
            tr.setdefault(key, []).append(b)
        json.dump({k: int(sum(v) / len(v)) for k, v in tr.items()}, open(traffic_out, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
