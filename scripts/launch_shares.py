"""One frame's launches with shares from an ncu launch list of bench.py
(ncu --metrics gpu__time_duration.sum --csv --log-file X python bench.py ...):
`python scripts/launch_shares.py X`.  A frame starts at k_cull; the last
complete frame (the most launches) is printed."""
import csv
import io
import sys

txt = open(sys.argv[1]).read()
lines = [l for l in txt.splitlines() if l.startswith('"')]
rows = list(csv.reader(io.StringIO("\n".join(lines))))
h = rows[0]
ik, im, iv = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value"))
launches = [(r[ik], float(r[iv].replace(",", "")) / 1e3) for r in rows[1:]
            if r[im] == "gpu__time_duration.sum"]
frames, cur = [], None
for k, t in launches:
    if k.startswith("k_cull"):
        cur = []
        frames.append(cur)
    if cur is not None:
        cur.append((k, t))
n = max(len(f) for f in frames)
frame = [f for f in frames if len(f) == n][-1]
tot = sum(t for _, t in frame)
short = lambda k: k.split("(")[0].replace("ls::unet::", "unet::")
print(f"{'kernel':60s} {'us':>8s} {'share':>7s}")
for k, t in frame:
    print(f"{short(k)[:60]:60s} {t:8.1f} {100 * t / tot:6.1f}%")
unet = sum(t for k, t in frame if "unet::" in k)
proj = sum(t for k, t in frame if "k_frame_pass" in k)
print(f"{'total':60s} {tot:8.1f}")
print(f"U-Net share {100 * unet / tot:.1f}%  projection passes {100 * proj / tot:.1f}%  "
      f"launches in frame {len(frame)}")
