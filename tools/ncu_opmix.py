"""Dynamic SASS opcode mix (warp-level instructions executed) from an ncu report."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
src, ie = h.index("Source"), h.index("Instructions Executed")
mix = collections.Counter()
for r in rows[hi + 1:]:
    try:
        n = float(r[ie])
    except Exception:
        continue
    toks = [t for t in r[src].split() if not t.startswith("@")]
    if toks:
        mix[toks[0].split(".")[0]] += n
tot = sum(mix.values())
print(f"total warp-instructions {tot:.0f}")
for op, n in mix.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{op:10s} {n:12.0f} {100 * n / tot:5.1f}%")
