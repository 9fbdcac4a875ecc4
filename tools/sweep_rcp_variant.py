"""Exhaustive CPU check (oracle only): over every fp16 pair (x, s) with
0 < s finite and |x| <= s, the code from n' = RN32(x * RN32(1/s)) equals the
code from n = RN32(x / s).  Justifies the kernel's division-free normalisation
(DESIGN.md "Exactness").  Prints the mismatch count (expected 0)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import nqkv_oracle as O  # noqa: E402

T = O.thresholds_f32()
allx = np.arange(0, 0x10000, dtype=np.uint32).astype(np.uint16).view(np.float16)
allx = allx[np.isfinite(allx)].astype(np.float32)
order = np.argsort(np.abs(allx), kind="stable")
ax_sorted = np.abs(allx)[order]
xs_sorted = allx[order]
s_all = np.arange(1, 0x7C00, dtype=np.uint16).view(np.float16).astype(np.float32)
mism = 0
pairs = 0
n_diff = 0
for i, s in enumerate(s_all):
    k = np.searchsorted(ax_sorted, s, side="right")
    x = xs_sorted[:k]
    n = x / s
    r = np.float32(1.0) / s
    n2 = x * r
    c1 = np.searchsorted(T, n, side="left")
    c2 = np.searchsorted(T, n2, side="left")
    mism += int(np.count_nonzero(c1 != c2))
    n_diff += int(np.count_nonzero(n != n2))
    pairs += k
print(f"pairs={pairs} code_mismatches={mism} n_differs={n_diff}")
