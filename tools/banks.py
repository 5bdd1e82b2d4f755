"""Shared-memory bank model for the FFT-512 access patterns of csrc/fft.cuh (8-byte elements).
A warp's 64-bit access is served per half-warp (16 lanes x 2 words over 32 banks): a half-warp
costs the largest number of distinct words any bank holds, the warp the sum of its two halves
(ideal 2). This model reproduces ncu's source view (the pass-2 stores and the mirrored packing loads
under P8 cost 4 wavefronts), which the full-warp model used in round 1 did not.
  python tools/banks.py"""
from collections import defaultdict


def wavefronts(addrs):
    tot = 0
    for h in range(2):
        banks = defaultdict(set)
        for a in addrs[16 * h:16 * h + 16]:
            for w in (2 * a, 2 * a + 1):
                banks[w % 32].add(w)
        tot += max(len(v) for v in banks.values())
    return tot


def P8(i):          # passes 1 -> 2 and the real-FFT packing
    return i + (i >> 4)


def Q(i):           # passes 2 -> 3
    return i + 2 * (i >> 4)


def N(i):           # transform inputs / outputs and the real-FFT packing (natural, unpadded)
    return i


def patterns():
    """(name, layout, logical indices of one warp) for every exchange of fft512_regs and the
    real-FFT packing, both warps of a 64-thread group, r = 0..7."""
    for w in (0, 32):
        js = [w + t for t in range(32)]
        for r in range(8):
            yield "pass-1 store", P8, [8 * j + r for j in js]
            yield "pass-2 load", P8, [j + 64 * r for j in js]
            yield "pass-2 store", Q, [64 * (j >> 3) + (j & 7) + 8 * r for j in js]
            yield "pass-3 load", Q, [j + 64 * r for j in js]
            yield "natural store/load", N, [j + 64 * r for j in js]
            yield "run from any offset (PAM extraction)", N, [(r * 37 + t) % 512 for t in range(32)]
        for r in range(4):
            yield "mirror load / store", N, [(512 - (j + 64 * r)) & 511 for j in js]


def worst():
    out = {}
    for name, lay, idx in patterns():
        out[name] = max(out.get(name, 0), wavefronts([lay(i) for i in idx]))
    return out


if __name__ == "__main__":
    print(worst())
    print("P8 for the pass-2 stores:", max(wavefronts([P8(i) for i in idx]) for n, l, idx in patterns()
                                          if n == "pass-2 store"))
