#!/usr/bin/env python3
"""One line per profiled launch from an ncu report: time, DRAM bytes, throughput, occupancy, stalls."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, data = rows[0], rows[1], rows[2:]
want = {
    "time_us": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "fp64_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "l2_hit": "lts__t_sector_hit_rate.pct",
}
idx = {k: hdr.index(v) for k, v in want.items() if v in hdr}
name_i = hdr.index("Kernel Name")


def num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return float("nan")


def scale(k, v):
    u = units[idx[k]]
    f = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "msecond": 1e3, "ms": 1e3, "usecond": 1, "us": 1,
         "nsecond": 1e-3, "ns": 1e-3}.get(u, 1)
    return v * f


print(f"{'kernel':28s} {'us':>8s} {'DRAM MB':>9s} {'GB/s':>7s} {'dram%':>6s} {'sm%':>5s} {'occ%':>5s} {'regs':>4s} "
      f"{'grid':>6s} {'fp64%':>6s} {'L2hit':>6s}")
for r in data:
    v = {k: num(r[i]) for k, i in idx.items()}
    t = scale("time_us", v["time_us"])
    db = scale("dram_rd", v["dram_rd"]) + scale("dram_wr", v["dram_wr"])
    print(f"{r[name_i][:28]:28s} {t:8.1f} {db/1e6:9.1f} {db/t/1e3:7.0f} {v.get('dram_pct', 0):6.1f} "
          f"{v.get('sm_pct', 0):5.1f} {v.get('warps_active', 0):5.1f} {v.get('regs', 0):4.0f} {v.get('grid', 0):6.0f} "
          f"{v.get('fp64_pct', 0):6.1f} {v.get('l2_hit', 0):6.1f}")
