"""Shared-memory bank model for the FFT access patterns (64-bit elements): prints the worst
wavefront count per pattern for candidate paddings. Used to pick P8(i) = i + i/16."""
import itertools
def wavefronts(word_addrs):
    # each lane accesses 2 consecutive words (8-byte element); cost = max over banks of distinct words
    banks = {}
    for w in word_addrs:
        for ww in (2*w, 2*w+1):
            banks.setdefault(ww % 32, set()).add(ww)
    return max(len(v) for v in banks.values())
def pats():
    for r in range(8):
        yield 'A', [j + 64*r for j in range(32)]
        yield 'A2', [j + 32 + 64*r for j in range(32)]
        yield 'B', [8*j + r for j in range(32)]
        yield 'B2', [8*(j+32) + r for j in range(32)]
        yield 'C', [(j>>3)*64 + (j&7) + 8*r for j in range(32)]
        yield 'C2', [((j+32)>>3)*64 + ((j+32)&7) + 8*r for j in range(32)]
    for r in range(4):
        yield 'D', [(512 - (j + 64*r)) & 511 for j in range(32)]
        yield 'D2', [(512 - (j + 32 + 64*r)) & 511 for j in range(32)]
    yield 'X', [2*j for j in range(32)]      # extraction-like even stride? (loc>>1 consecutive)
for name, pad in [('p8', lambda i: i + (i>>3)), ('p16', lambda i: i + (i>>4)), ('p32', lambda i: i + (i>>5)), ('none', lambda i: i), ('p8x', lambda i: i ^ ((i>>3)&7)), ('p4', lambda i: i + (i>>2))]:
    tot = {}
    worst = 0
    for n, p in pats():
        wf = wavefronts([pad(i) for i in p])
        tot[n] = max(tot.get(n, 0), wf)
    print(name, tot)
