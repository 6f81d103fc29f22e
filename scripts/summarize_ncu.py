"""Summarise ncu output for profiles/: key metrics of a --set full report, or
a launch list (--metrics gpu__time_duration.sum,...) CSV.

    python scripts/summarize_ncu.py report.ncu-rep > profiles/rNN_x.txt
    python scripts/summarize_ncu.py launches.csv   > profiles/rNN_y.txt
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "L1/TEX Hit Rate", "L2 Hit Rate",
        "No Eligible"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]


def report(path):
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    hdr = rows[0]
    ik, im, iv, iu, iid = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value",
                                                  "Metric Unit", "ID"))
    per = collections.OrderedDict()
    for r in rows[1:]:
        if r[im] in KEYS:
            per.setdefault((r[iid], r[ik]), {})[r[im]] = f"{r[iv]} {r[iu]}".strip()
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    rh = rr[0]
    for r in rr[2:]:
        d = dict(zip(rh, r))
        key = (d.get("ID"), d.get("Kernel Name"))
        for k in RAW:
            if k in d and key in per:
                per[key][k] = d[k]
    for (i, name), m in per.items():
        print(f"[{i}] {name[:110]}")
        for k in KEYS + RAW:
            if k in m:
                print(f"    {k:64s} {m[k]}")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ik, im, iv, iid = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        per.setdefault((int(r[iid]), r[ik]), {})[r[im]] = r[iv]
    mets = sorted({m for v in per.values() for m in v})
    print("id,kernel," + ",".join(mets))
    for (i, name), m in per.items():
        print(f"{i},{name[:60].replace(',', ';')}," + ",".join(m.get(x, "") for x in mets))


if __name__ == "__main__":
    p = sys.argv[1]
    report(p) if p.endswith(".ncu-rep") else launches(p)
