"""Summarise ncu output brought back in gpurun_out/ into profiles/.

  python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/r1_launches.md
  python tools/ncu_summary.py full gpurun_out/prof_bench.ncu-rep > profiles/r1_kernels.md
"""
import collections
import csv
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration (ns)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_registers", "CTA/SM limit (regs)"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        try:
            agg.setdefault(r[ki].split("(")[0][:60], []).append(float(r[vi]))
        except ValueError:
            pass
    step = [k for k in agg if k.startswith("wino_")]
    tot = sum(sum(agg[k]) for k in step)  # kernels launch a different number of times per step: total time
    print(f"# Launch list ({path}), ncu --metrics gpu__time_duration.sum --clock-control none\n")
    print("cold-cache, serialised per-launch times; compare shares, not absolutes\n")
    print("| kernel | launches | mean us | share of the libwino time (launches x mean) |")
    print("|---|---|---|---|")
    for k, v in agg.items():
        mean = sum(v) / len(v) / 1e3
        share = f"{100 * sum(v) / tot:.1f}%" if k in step else "-"
        print(f"| {k} | {len(v)} | {mean:.2f} | {share} |")


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary ({path})\n")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"## {d['Kernel Name'][:60]}  grid {d.get('launch__grid_size')} block {d.get('launch__block_size')}\n")
        print("| metric | value |")
        print("|---|---|")
        for k, name in KEYS:
            if k in d and d[k] != "":
                print(f"| {name} (`{k}`) | {d[k]} {u.get(k, '')} |")
        stalls = []
        for h, v in d.items():
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v), h.replace("smsp__average_warps_issue_stalled_", "").replace(
                        "_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        top = ", ".join(f"{n} {v:.2f}" for v, n in sorted(stalls, reverse=True)[:6])
        print(f"| top stall reasons (warps per issue) | {top} |\n")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
