"""Per-kernel counter table of one frame (ncu --metrics ... --csv launch list):
time, DRAM GB/s and share of the measured copy peak, L2 atomic/reduction
throughput, tensor-pipe / FP64 utilisation -- the evidence table the north
star asks for (profiles/r02_frame_counters.txt).

    python scripts/frame_counters.py launches.csv [peak_gbs]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
peak = float(sys.argv[2]) if len(sys.argv) > 2 else 6549.8
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[hi]
iname, imet, ival, iid, iunit = (hdr.index(x) for x in ("Kernel Name", "Metric Name",
                                                           "Metric Value", "ID", "Metric Unit"))
k = collections.OrderedDict()
for r in rows[hi + 1:]:
    v = r[ival].replace(",", "")
    try:
        v = float(v)
    except ValueError:
        continue
    unit = r[iunit]
    name = r[imet]
    if unit in ("Kbyte", "KB"):
        v *= 1e3
    elif unit in ("Mbyte", "MB"):
        v *= 1e6
    elif unit in ("Gbyte", "GB"):
        v *= 1e9
    elif unit == "usecond":
        v *= 1e3
    elif unit == "msecond":
        v *= 1e6
    k.setdefault((int(r[iid]), r[iname]), {})[name] = v
print(f"{'kernel':44s} {'us':>7s} {'DRAM GB/s':>9s} {'%HBM':>5s} {'red Gop/s':>9s} "
      f"{'tensor%':>7s} {'fp64%':>5s} {'IPC':>5s}")
tot = 0.0
for (i, n), m in k.items():
    t = m.get("gpu__time_duration.sum", 0.0)  # ns
    tot += t
    b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    gbs = b / t if t else 0.0
    red = (m.get("lts__t_sectors_srcunit_tex_op_red.sum", 0.0)
           + m.get("lts__t_sectors_srcunit_tex_op_atom.sum", 0.0))
    name = n.split("(")[0].replace("void ", "").replace("ls::", "").replace("unet::", "")[:44]
    print(f"{name:44s} {t / 1e3:7.1f} {gbs:9.0f} {100 * gbs / peak:5.1f} {red / t if t else 0:9.2f} "
          f"{m.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', 0):7.1f} "
          f"{m.get('sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active', 0):5.1f} "
          f"{m.get('sm__inst_executed.avg.per_cycle_active', 0):5.2f}")
print(f"{'frame (serialised, cold)':44s} {tot / 1e3:7.1f}")
