"""Warp-stall samples of an ncu report aggregated per CUDA source line (--print-source cuda,sass):
the hot regions of a kernel with their dominant stall reasons.
  python tools/ncu_lines_cuda.py report.ncu-rep [top_n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
out, total, fname = [], 0.0, ""
for i, r in enumerate(rows):
    if r and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
    if not r or r[0] != "Line No":
        continue
    h = r
    samp = h.index("Warp Stall Sampling (All Samples)")
    inst = h.index("Instructions Executed")
    stalls = [k for k, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
    for q in rows[i + 1:]:
        if not q or q[0] in ("File Path", "Function Name", "Line No"):
            break
        if q[0] == "" or q[2] != "-":
            continue            # SASS rows: the CUDA row carries their sums
        try:
            v = float(q[samp])
        except ValueError:
            continue
        st = {}
        for k in stalls:
            try:
                st[h[k][6:]] = float(q[k])
            except ValueError:
                pass
        try:
            ni = float(q[inst])
        except ValueError:
            ni = 0.0
        out.append((v, ni, f"{fname}:{q[0]}", q[1].strip(), st))
        total += v
total = total or 1.0
print(f"{'share':>6s} {'inst exec':>11s}  line")
for v, ni, loc, src, st in sorted(out, key=lambda t: -t[0])[:n]:
    top = ", ".join(f"{s}={100 * x / max(v, 1):.0f}%" for s, x in sorted(st.items(), key=lambda t: -t[1])[:3])
    print(f"{100 * v / total:5.1f}% {ni:11.0f}  {loc:18s} {src[:72]:72s} [{top}]")
