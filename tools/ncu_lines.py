"""Warp-stall samples of an ncu report aggregated per CUDA source line, by joining the report's
SASS page (address, samples) with `nvdisasm -g` line info of the same cubin (compiled with
-lineinfo). Usage: python tools/ncu_lines.py report.ncu-rep lib.so kernel-substring [N]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, so, kname = sys.argv[1], sys.argv[2], sys.argv[3]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
samp = h.index("Warp Stall Sampling (All Samples)")
sass = []
for r in rows[hi + 1:]:
    try:
        sass.append((int(r[0], 16), r[1].strip(), float(r[samp])))
    except Exception:
        pass
base = min(a for a, _, _ in sass)
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
cubin = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
# split per function, keep the one whose name contains kname and whose length matches
funcs, cur, name = {}, None, None
for line in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", line)
    if m:
        name = m.group(1)
        funcs[name] = []
        continue
    if name is not None:
        funcs[name].append(line)
best = None
for fn, lines in funcs.items():
    if kname not in fn:
        continue
    offs = [int(m.group(1), 16) for l in lines for m in [re.search(r"/\*([0-9a-f]{4,})\*/", l)] if m]
    if offs and abs(max(offs) - (max(a for a, _, _ in sass) - base)) <= 16:
        best = fn
if best is None:
    sys.exit(f"no function matching {kname} with {len(sass)} instructions")
line_of, curl = {}, None
for l in funcs[best]:
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        curl = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m:
        line_of[int(m.group(1), 16)] = curl
agg = collections.Counter()
tot = 0.0
for a, s, v in sass:
    agg[line_of.get(a - base, "?")] += v
    tot += v
src_cache = {}
print(f"{best}: {len(sass)} SASS, {tot:.0f} samples")
for k, v in agg.most_common(n):
    text = ""
    if k and ":" in k:
        f, ln = k.rsplit(":", 1)
        path = next((os.path.join(d, f) for d in ("paper_2011_13695_b200/csrc", "include") if os.path.exists(os.path.join(d, f))), None)
        if path:
            src_cache.setdefault(path, open(path).read().splitlines())
            text = src_cache[path][int(ln) - 1].strip()[:90]
    print(f"{100 * v / tot:5.1f}%  {k:<18} {text}")
