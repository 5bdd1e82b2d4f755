"""Digest a profiles/<tag> capture directory on the GPU box (so only text travels back):
launches_summary.txt, ncu_full_summary.jsonl, ncu_stalls_opmix.txt and ncu_traffic.json
(DRAM bytes per launch of the kernel behind each bench kernel class; bench.py reads it)."""
import glob
import json
import os
import subprocess
import sys

d = sys.argv[1]
tools = os.path.dirname(os.path.abspath(__file__))
py = sys.executable


def run(args):
    return subprocess.run([py] + args, capture_output=True, text=True).stdout


if os.path.exists(os.path.join(d, "launches.csv")):
    open(os.path.join(d, "launches_summary.txt"), "w").write(
        run([os.path.join(tools, "launch_summary.py"), os.path.join(d, "launches.csv")]))
reps = sorted(glob.glob(os.path.join(d, "*.ncu-rep")))
summ, stalls = [], []
for r in reps:
    out = run([os.path.join(tools, "ncu_summary.py"), r])
    summ.append(out)
    stalls.append(f"== {os.path.basename(r)[:-8]}\n" + run([os.path.join(tools, "ncu_src.py"), r])
                  + run([os.path.join(tools, "ncu_opmix.py"), r]))
open(os.path.join(d, "ncu_full_summary.jsonl"), "w").write("".join(summ))
open(os.path.join(d, "ncu_stalls_opmix.txt"), "w").write("\n".join(stalls))
# ncu kernel -> the bench.py kernel class whose roofline "traffic" it supplies (bench looks up
# <family>_<class>: prof_kk_* reports come from the C4 KK run, the others from the C2 PAM run)
CLASS = {"k_lms_seg<0": "LMS", "k_lms_seg<1": "LMS", "k_pam_be": "PAM_BE", "k_pam_fe": "PAM_FE",
         "k_pam_theta": "PAM_CLOCK", "k_norm_stats": "NORM", "k_kk_s1": "KK_S1", "k_kk_s2": "KK_S2",
         "k_cfo_spec": "CFO", "k_lms_prefix": "LMS_POST", "k_lms_final": "LMS_POST"}
traffic = {}
for line in "".join(summ).splitlines():
    j = json.loads(line)
    name = j.get("Kernel Name", "")
    norm = name.replace("void ", "").replace("(bool)", "").replace("false", "0").replace("true", "1")
    cls = next((v for k, v in CLASS.items() if norm.startswith(k)), None)
    if not cls:
        continue
    cls = ("KK_" if "prof_kk_" in j.get("report", "") else "PAM_") + cls
    if cls in traffic:
        continue

    def val(key):
        v = j.get(key, "0").split()
        x = float(v[0])
        unit = v[1] if len(v) > 1 else "byte"
        return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    traffic[cls] = {"kernel": name, "dram_bytes_per_launch": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
                    "duration": j.get("gpu__time_duration.sum"), "grid": j.get("launch__grid_size"),
                    "report": j.get("report")}
json.dump(traffic, open(os.path.join(d, "ncu_traffic.json"), "w"), indent=1)
if os.environ.get("KEEP_REPS") != "1":
    for r in reps:
        os.remove(r)
print("digested", len(reps), "reports")
