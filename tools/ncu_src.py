"""Top stalled SASS instructions and stall-reason totals of an ncu report (source page)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
src, samp = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
stalls = [i for i, x in enumerate(h) if x.startswith("stall_")]
data, tot_reason = [], {}
for r in rows[hi + 1:]:
    try:
        v = float(r[samp])
    except Exception:
        continue
    data.append((v, r[0], r[src].strip()[:90]))
    for i in stalls:
        try:
            tot_reason[h[i]] = tot_reason.get(h[i], 0.0) + float(r[i])
        except Exception:
            pass
tot = sum(d[0] for d in data) or 1
print("stall reasons:", ", ".join(f"{k[6:]}={100 * v / tot:.0f}%" for k, v in
                                  sorted(tot_reason.items(), key=lambda x: -x[1])[:6]))
for v, a, s in sorted(data, reverse=True)[:n]:
    print(f"{100 * v / tot:5.1f}%  {s}")
