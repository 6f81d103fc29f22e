"""Per-layer table from an ncu launch-list CSV of one U-Net forward
(ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,
 sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:k_conv -c 22; 21 launches with the fused dec0_up)."""
import collections
import csv
import io
import sys

NAMES = ["e0c1", "e0c2", "e1c1", "e1c2", "e2c1", "e2c2", "e3c1", "e3c2", "b1", "b2", "d3up",
         "d3c1", "d3c2", "d2up", "d2c1", "d2c2", "d1up", "d1c1", "d1c2", "d0up", "d0c1", "d0c2h"]
txt = open(sys.argv[1]).read()
lines = [l for l in txt.splitlines() if l.startswith('"')]
rows = list(csv.reader(io.StringIO("\n".join(lines))))
h = rows[0]
iid, ik, im, iv = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
per = collections.OrderedDict()
for r in rows[1:]:
    per.setdefault(r[iid], {"k": r[ik]})[r[im]] = float(r[iv].replace(",", ""))
tot = 0.0
ids = list(per)
if any("upfuse" in per[i]["k"] for i in ids[:21]):  # dec0_up inside dec0_conv1: 21 launches
    NAMES = NAMES[:19] + ["d0up+c1", "d0c2h"]
for n, i in zip(NAMES, ids[:len(NAMES)]):
    d = per[i]
    t = d["gpu__time_duration.sum"] / 1000
    tot += t
    k = d["k"].split("(")[0].replace("void ls::unet::", "")
    print(f"{n:6s} {k:26s} {t:7.1f} us  tensor "
          f"{d['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed']:5.1f}%  "
          f"DRAM R {d['dram__bytes_read.sum'] / 1e6:6.1f} W {d['dram__bytes_write.sum'] / 1e6:6.1f} MB")
print(f"sum {tot:.1f} us")
