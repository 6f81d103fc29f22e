"""Summarise an ncu --set full capture: top stall reasons and hottest SASS
instructions (python scripts/ncu_stalls.py report.ncu-rep [n_top])."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
ix = {n: i for i, n in enumerate(h)}
stalls = [n for n in h if n.startswith("stall_") and "(Not" not in n]
S = "Warp Stall Sampling (All Samples)"
tot = {s: sum(int(r[ix[s]] or 0) for r in data) for s in stalls}
alls = sum(int(r[ix[S]] or 0) for r in data)
print(rows[0][1][:100], "samples", alls)
print("  ".join(f"{s[6:]} {100 * v / alls:.1f}%" for s, v in sorted(tot.items(), key=lambda x: -x[1])[:8]))
for r in sorted(data, key=lambda r: -int(r[ix[S]] or 0))[:ntop]:
    best = sorted(stalls, key=lambda s: -int(r[ix[s]] or 0))[:2]
    print(f"{r[0][-5:]} {r[1].strip()[:64]:64s} {r[ix[S]]:>5} exec {r[ix['Instructions Executed']]:>8} "
          + " ".join(f"{b[6:]}={r[ix[b]]}" for b in best))
