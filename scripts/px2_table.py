"""Last forward's k_conv_px2 launches from an ncu launch CSV: `python scripts/px2_table.py a.csv [b.csv ...]`."""
import csv, sys
for fn in sys.argv[1:]:
    rows = list(csv.reader(open(fn)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    ts = [(r[ki][13:40].split("(")[0], float(r[vi].replace(",", "")) / 1e3) for r in rows[hi + 1:]]
    print(f"{fn.split('/')[-1]:14s}", " ".join(f"{n}:{t:.1f}" for n, t in ts[-6:]))
