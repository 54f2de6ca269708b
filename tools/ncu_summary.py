"""Summarise an ncu report (or a --csv launch list) into a short text file for profiles/.

  python tools/ncu_summary.py gpurun_out/rN_prof.ncu-rep > profiles/<round>_<what>.txt
  python tools/ncu_summary.py --launches gpurun_out/launches.csv > profiles/<round>_launches.txt
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

RAW = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second",
    "smsp__inst_executed.sum",
]


def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    for r in rows[2:]:
        print("kernel:", r[idx["Kernel Name"]][:150])
        for m in RAW:
            if m in idx:
                print(f"  {m:90s} {r[idx[m]]:>16s} {units[idx[m]]}")
        rd = float(r[idx["dram__bytes_read.sum"]] or 0)
        wr = float(r[idx["dram__bytes_write.sum"]] or 0)
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
        print(f"  traffic (dram read+write) = {rd * scale.get(units[idx['dram__bytes_read.sum']], 1) + wr * scale.get(units[idx['dram__bytes_write.sum']], 1):.4e} bytes")


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ki, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                      hdr.index("Metric Unit"))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[start + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            v = float(r[vi].replace(",", ""))
            v *= {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1.0)
            name = r[ki].split("(")[0][:80]
            tot[name] += v
            cnt[name] += 1
    allt = sum(tot.values())
    print(f"{'kernel':80s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
    for name, t in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{name:80s} {cnt[name]:8d} {t:10.3f} {100 * t / allt:6.1f}%")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        summary(sys.argv[1])
