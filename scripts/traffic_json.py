"""profiles/r01_traffic.json from an ncu launch CSV of scripts/profile_frame.py
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum):
the LAST frame's kernels.

    python scripts/traffic_json.py launches.csv <candidates of the last frame> <command>
"""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[hi]
iname, imet, ival, iid = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
k = collections.OrderedDict()
for r in rows[hi + 1:]:
    k.setdefault((int(r[iid]), r[iname]), {})[r[imet]] = float(r[ival].replace(",", ""))
launches = list(k.items())
# the last frame starts at its cull (followed by the work-list kernels) and
# ends before the next cull (the script's candidate counting)
starts = [i for i, ((_, n), _) in enumerate(launches)
          if "k_cull" in n and i + 1 < len(launches) and "k_zero_count" in launches[i + 1][0][1]]
end = next((i for i in range(starts[-1] + 1, len(launches)) if "k_cull" in launches[i][0][1]),
           len(launches))
frame = launches[starts[-1]:end]
b = lambda m: m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
unet = [m for (_, n), m in frame if "k_conv" in n]
proj = [m for (_, n), m in frame if "k_frame_pass" in n]
cand = int(sys.argv[2])
lines = ["kernel                                                          us     R MB     W MB"]
for (_, n), m in frame:
    lines.append(f"{n.split('(')[0][-60:]:60s} {m['gpu__time_duration.sum'] / 1e3:7.1f} "
                 f"{m.get('dram__bytes_read.sum', 0) / 1e6:8.1f} {m.get('dram__bytes_write.sum', 0) / 1e6:8.1f}")
out = {
    "source": sys.argv[3] if len(sys.argv) > 3 else sys.argv[1],
    "unet_dram_bytes_per_frame": int(sum(b(m) for m in unet)),
    "unet_launches_per_frame": len(unet),
    "projection_dram_bytes": int(sum(b(m) for m in proj)),
    "projection_candidates": cand,
    "projection_dram_bytes_per_candidate": round(sum(b(m) for m in proj) / cand, 2),
    "projection_algorithmic_bytes_per_candidate": 27.0,
}
print(json.dumps(out, indent=2))
print("\n".join(lines), file=sys.stderr)
