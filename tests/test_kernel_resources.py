"""Resource guards of the hot kernels in the built librx.so (cuobjdump -res-usage, no GPU needed):
no register spills (stack / local memory) and the register budgets that give the occupancy the
kernels were tuned at (k_kk_s1 5 CTAs / SM, k_kk_s2 4, k_pam_fe 6, k_cfo_spec 3)."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_2011_13695_b200", "librx.so")

# mangled-name prefix -> max registers per thread (None: no budget, spills only)
HOT = {
    "_Z7k_kk_s1": 51, "_Z7k_kk_s2": 64, "_Z10k_cfo_spec": 85, "_Z8k_pam_feILb1": 40, "_Z8k_pam_beILb1": 42,
    "_Z9k_lms_segILb1ELi2ELi8ELb0ELi1": None, "_Z9k_lms_segILb0ELi0ELi32ELb0ELi1": None,
}


def _usage():
    if not os.path.exists(SO) or not shutil.which("cuobjdump"):
        pytest.skip("librx.so not built or cuobjdump missing")
    out = subprocess.run(["cuobjdump", "-res-usage", SO], capture_output=True, text=True).stdout
    res, name = {}, None
    for line in out.splitlines():
        m = re.match(r"\s*Function (\S+):", line)
        if m:
            name = m.group(1)
            continue
        m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", line)
        if m and name:
            res[name] = tuple(int(x) for x in m.groups())
    return res


def test_hot_kernels_do_not_spill_and_fit_their_register_budgets():
    res = _usage()
    for prefix, budget in HOT.items():
        hits = {k: v for k, v in res.items() if k.startswith(prefix)}
        assert hits, prefix
        for k, (reg, stack, _shared, local) in hits.items():
            assert stack == 0 and local == 0, (k, stack, local)
            if budget is not None:
                assert reg <= budget, (k, reg, budget)
