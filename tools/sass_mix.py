"""Static SASS instruction mix per kernel of librx.so (cuobjdump -sass): total instructions and
the FP32 scalar / packed (FADD2 / FMUL2 / FFMA2, sm_100) / shared-memory / min-max counts.
  python tools/sass_mix.py [librx.so] [kernel-substring ...]"""
import collections
import re
import subprocess
import sys

so = sys.argv[1] if len(sys.argv) > 1 else "paper_2011_13695_b200/librx.so"
keys = sys.argv[2:] or ["k_kk_s1", "k_kk_s2", "k_kk_fe", "k_cfo_spec", "k_cfo_fine", "k_pam_fe", "k_pam_be",
                        "k_lms_segILb1ELi2ELi8ELb0ELi1", "k_lms_segILb0ELi0ELi32ELb0ELi1"]
sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
cur, cnt = None, collections.defaultdict(collections.Counter)
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
    if m and cur and m.group(2) not in ("NOP",):
        cnt[cur][m.group(2)] += 1
cols = ("FADD", "FMUL", "FFMA", "FADD2", "FMUL2", "FFMA2", "FMNMX", "LDS", "STS", "SHFL")
print(f"{'kernel':44s} {'total':>6s} " + " ".join(f"{c:>6s}" for c in cols))
for k, c in cnt.items():
    if any(s in k for s in keys):
        print(f"{k[:44]:44s} {sum(c.values()):6d} " + " ".join(f"{c[x]:6d}" for x in cols))
