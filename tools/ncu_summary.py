"""Summarise ncu outputs for profiles/.

  python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/rNN_launches.txt
  python tools/ncu_summary.py full gpurun_out/prof.ncu-rep > profiles/rNN_ncu_full.txt
"""
import collections
import csv
import io
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warp_latency_issue_stalled_barrier", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def _rows(text):
    rows = [r for r in csv.reader(io.StringIO(text)) if r]
    start = next(i for i, r in enumerate(rows) if r[0] == "ID")
    hdr = rows[start]
    return hdr, rows[start + 1:]


def launches(path, skip_prefix=None):
    text = open(path).read()
    hdr, rows = _rows(text)
    ix = {h: i for i, h in enumerate(hdr)}
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if len(r) != len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        v = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        name = r[ix["Kernel Name"]]
        name = name.split("(")[0]
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    print(f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)")
    print(f"# {sum(cnt.values())} launches, {s / 1e3:.1f} ms total; share of summed kernel time")
    print(f"{'total_us':>12} {'share':>6} {'launches':>8} {'avg_us':>9}  kernel")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v:12.1f} {100 * v / s:5.1f}% {cnt[k]:8d} {v / cnt[k]:9.1f}  {k}")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = [r for r in csv.reader(io.StringIO(out)) if r]
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        print("----", r[ix["Kernel Name"]][:100], "grid", r[ix.get("Grid Size", 0)], "block", r[ix.get("Block Size", 0)])
        for m in FULL_METRICS:
            if m in ix:
                print(f"  {m} = {r[ix[m]]} {units[ix[m]]}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
