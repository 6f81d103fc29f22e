"""Per-CUDA-source-line totals (executed warp instructions, stall samples) of
one kernel from `ncu -i rep --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur_file, agg, hdr = None, {}, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:  # a source line row (aggregated over its SASS)
        try:
            samples = int(r[4] or 0)
            ex = int(r[7] or 0)
        except ValueError:
            continue
        key = (cur_file, int(r[0]))
        a = agg.setdefault(key, [0, 0, r[1][:90]])
        a[0] += ex
        a[1] += samples
te = sum(v[0] for v in agg.values())
ts = sum(v[1] for v in agg.values())
print(f"total warp instr {te}  stall samples {ts}")
for (f, ln), (ex, sm, src) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{sm / ts * 100:5.1f}% st {ex / te * 100:5.1f}% in  {f}:{ln:<5d} {src}")
