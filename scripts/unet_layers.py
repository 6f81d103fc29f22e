"""Per-layer table from an ncu launch CSV of scripts/time_unet.py (last forward)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[hi]
iname, imet, ival, iid = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
k = collections.OrderedDict()
for r in rows[hi + 1:]:
    k.setdefault((int(r[iid]), r[iname][:40]), {})[r[imet]] = r[ival].replace(",", "")
conv = [x for x in k.items() if "k_conv" in x[0][1]]
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 22
names = ["e0c1", "e0c2", "e1c1", "e1c2", "e2c1", "e2c2", "e3c1", "e3c2", "b1", "b2", "d3up", "d3c1",
         "d3c2", "d2up", "d2c1", "d2c2", "d1up", "d1c1", "d1c2", "d0up", "d0c1", "d0c2h"]
tot = 0
for n, ((i, kn), m) in zip(names, conv[-nl:]):
    t = float(m["gpu__time_duration.sum"]) / 1e3
    tot += t
    g = lambda key: float(m.get(key, "nan"))
    print(f"{n:6s} {kn[8:36]:28s} {t:8.1f} us  dram r/w {g('dram__bytes_read.sum')/1e6:7.1f}/"
          f"{g('dram__bytes_write.sum')/1e6:7.1f} MB  L2 {g('lts__t_bytes.sum')/1e6:8.1f} MB  "
          f"tensor {m.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed')}%")
print("total", round(tot, 1), "us")
