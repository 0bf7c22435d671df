"""Summarise ncu reports / launch lists into profiles/ (markdown).

usage: python tools/ncu_summary.py report.ncu-rep [more.ncu-rep ...] > profiles/x.md
       python tools/ncu_summary.py --launches launches.csv > profiles/y.md
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def stalls(d):
    out = []
    for k, v in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            try:
                out.append((float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(v for v, _ in out) or 1
    return ", ".join(f"{n} {v / tot * 100:.0f}%" for v, n in sorted(out, reverse=True)[:6])


def report(rep):
    print(f"### {rep.split('/')[-1]}\n")
    for d, u in raw(rep):
        print(f"kernel: `{d.get('Kernel Name', '?')[:90]}`\n")
        print("| metric | value |\n|---|---|")
        for k, name in KEYS:
            if k in d:
                print(f"| {name} (`{k}`) | {d[k]} {u.get(k, '')} |")
        print(f"| top stall reasons (pc sampling) | {stalls(d)} |\n")


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {h: j for j, h in enumerate(hdr)}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        try:
            v = float(r[ix["Metric Value"]].replace(",", ""))
        except ValueError:
            continue
        v *= {"msecond": 1e6, "usecond": 1e3, "nsecond": 1.0, "second": 1e9}.get(r[ix["Metric Unit"]], 1.0)
        name = r[ix["Kernel Name"]].split("(")[0][:80]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(t for _, t in agg.values())
    print(f"### launch list `{path.split('/')[-1]}` (ncu gpu__time_duration.sum, --clock-control none; "
          "serialised, cold-cache: compare shares)\n")
    print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
        print(f"| `{k}` | {n} | {t / 1e6:.3f} | {t / tot * 100:.1f}% |")
    print()


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        for p in sys.argv[2:]:
            launches(p)
    else:
        for p in sys.argv[1:]:
            report(p)
