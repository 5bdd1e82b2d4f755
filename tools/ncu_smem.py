"""Shared-memory wavefronts per SASS instruction of an ncu report (source page): totals, ideal,
excess (bank conflicts) and the instructions with the most excess.
  python tools/ncu_smem.py report.ncu-rep [top_n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
tot = [0.0, 0.0, 0.0]
lst = []
cur_line = ""
for i, r in enumerate(rows):
    if not r or r[0] != "Line No":
        continue
    h = r
    cw, ci, cx = (h.index(k) for k in ("L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal",
                                        "L1 Wavefronts Shared Excessive"))
    for q in rows[i + 1:]:
        if not q or q[0] in ("File Path", "Function Name", "Line No"):
            break
        if q[2] == "-":
            cur_line = f"{q[0]}: {q[1].strip()[:60]}"
            continue
        try:
            w, idl, x = float(q[cw] or 0), float(q[ci] or 0), float(q[cx] or 0)
        except ValueError:
            continue
        tot[0] += w; tot[1] += idl; tot[2] += x
        if x > 0:
            lst.append((x, w, q[3].strip()[:48], cur_line))
print(f"wavefronts {tot[0]:.0f}  ideal {tot[1]:.0f}  excess {tot[2]:.0f}")
for x, w, s, ln in sorted(lst, reverse=True)[:n]:
    print(f"excess {x:10.0f} of {w:10.0f}  {s:48s}  {ln}")
