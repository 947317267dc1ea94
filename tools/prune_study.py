"""How fast the data-parallel pruning of k_hull (csrc/k_rows_band.cu,
warp_prune) converges on the C5 image: for a few lines, the number of columns
with a carry above the line, the size of their lower hull, and the survivors
after each round (stride 1 only; strides 1..64 as in the kernel).  Host only
(numpy); output committed as profiles/r02/prune_study.txt."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402

img = workloads.config("c5")
H, W = img.shape


def carries_above(line):
    rows = np.arange(line)[:, None]
    return np.where(img[:line] > 0, rows, -1).max(axis=0)


def hull_size(k, Hv):
    st = []
    for i in range(len(k)):
        while len(st) >= 2:
            a, b = st[-2], st[-1]
            if (Hv[b] - Hv[a]) * (k[i] - k[b]) > (Hv[i] - Hv[b]) * (k[b] - k[a]):
                st.pop()
            else:
                break
        st.append(i)
    return len(st)


def rounds(k, Hv, strides, nrounds):
    out = []
    for _ in range(nrounds):
        n = len(k)
        gone = np.zeros(n, bool)
        for s in strides:
            if n <= 2 * s:
                continue
            a, b, c = slice(0, n - 2 * s), slice(s, n - s), slice(2 * s, n)
            gone[s:n - s] |= (Hv[b] - Hv[a]) * (k[c] - k[b]) > (Hv[c] - Hv[b]) * (k[b] - k[a])
        k, Hv = k[~gone], Hv[~gone]
        out.append(len(k))
    return out


print(f"c5 image {H}x{W}, {int(img.sum())} object pixels")
for line in (4096, 16384, 20000, 30000):
    ca = carries_above(line)
    k = np.nonzero(ca >= 0)[0].astype(np.int64)
    d = (line - ca[k]).astype(np.int64)
    Hv = d * d + k * k
    print(f"line {line}: {len(k)} columns with a carry, lower hull {hull_size(k.tolist(), Hv.tolist())} points")
    print("   stride 1 only, 12 rounds :", rounds(k, Hv, (1,), 12))
    print("   strides 1..64, 6 rounds  :", rounds(k, Hv, (1, 2, 4, 8, 16, 32, 64), 6))
