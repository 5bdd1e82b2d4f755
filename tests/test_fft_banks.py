"""Host-side check of the shared-memory layout of the FFT-512 (csrc/fft.cuh): every exchange and
packing access of a 64-thread group costs the ideal 2 wavefronts per warp under the half-warp bank
model (tools/banks.py), and the two layouts are bijections into FFT_PAD_N = 576 elements."""
import os
import re
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import banks  # noqa: E402


def test_fft_exchanges_are_conflict_free():
    w = banks.worst()
    assert all(v == 2 for v in w.values()), w


def test_p8_would_conflict_on_pass2_stores():
    # the reason for the second layout Q (ncu measured 4 wavefronts per pass-2 store under P8)
    idx = [64 * (j >> 3) + (j & 7) + 8 * r for r in (0,) for j in range(32)]
    assert banks.wavefronts([banks.P8(i) for i in idx]) == 4


def test_layouts_fit_the_padded_buffer():
    src = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "paper_2011_13695_b200", "csrc", "fft.cuh")).read()
    n = int(re.search(r"#define FFT_PAD_N (\d+)", src).group(1))
    for lay in (banks.P8, banks.Q, banks.N):
        img = [lay(i) for i in range(512)]
        assert len(set(img)) == 512 and max(img) < n
