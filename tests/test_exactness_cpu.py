"""Exhaustive fp16 argument for the kernels' division-free normalisation
(CPU, oracle only).  The method's code is defined on n = RN32(x/s)
(reading R4); the kernels compute n' = RN32(x * RN32(1/s)).  Over
EVERY fp16 pair with 0 < s finite and |x| <= s (1,007,713,278 pairs, both
zeros included) the two give the same code, although n' != n for ~27% of the
pairs.  Because fp16 inputs form a finite domain, this sweep is a proof."""
import numpy as np

from oracle import nqkv_oracle as O


def test_reciprocal_normalisation_gives_identical_codes_for_all_fp16_pairs():
    T = O.thresholds_f32()
    allx = np.arange(0, 0x10000, dtype=np.uint32).astype(np.uint16).view(np.float16)
    allx = allx[np.isfinite(allx)].astype(np.float32)
    order = np.argsort(np.abs(allx), kind="stable")
    ax, xs = np.abs(allx)[order], allx[order]
    s_all = np.arange(1, 0x7C00, dtype=np.uint16).view(np.float16).astype(np.float32)
    pairs = mism = ndiff = 0
    for s in s_all:
        k = np.searchsorted(ax, s, side="right")
        x = xs[:k]
        n = x / s
        n2 = x * (np.float32(1.0) / s)
        mism += int(np.count_nonzero(np.searchsorted(T, n, "left") != np.searchsorted(T, n2, "left")))
        ndiff += int(np.count_nonzero(n != n2))
        pairs += k
    assert pairs == 1007713278
    assert mism == 0
    assert ndiff > 0.25 * pairs     # the normalised values themselves do differ
