"""Writes tests/golden/near_threshold_pairs.txt using ONLY oracle/.

For every positive finite fp16 scale s and every decision threshold T_i, the
fp16 values x bracketing T_i*s are the only ones whose normalised value
n = RN32(x/s) can land within 1 fp32 ulp of T_i; we keep the (x, s) pairs
(and their mirrored negatives) that do, with the oracle's brute-force code.
These are the fp16 inputs most sensitive to the rounding of x/s and of the
thresholds (SURVEY.md 8(c) "near-threshold regression vectors").

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import nqkv_oracle as O  # noqa: E402


def main():
    L = O.nf_levels_f32()
    T = O.thresholds_f32(L)
    s_all = np.arange(1, 0x7C00, dtype=np.uint16).view(np.float16)          # positive finite
    rows = []
    for t in T:
        target = s_all.astype(np.float64) * float(t)
        x0 = target.astype(np.float16)                                     # nearest
        cands = [x0, np.nextafter(x0, np.float16(-np.inf)), np.nextafter(x0, np.float16(np.inf))]
        for x in cands:
            ok = np.isfinite(x) & (np.abs(x.astype(np.float32)) <= s_all.astype(np.float32))
            n = x.astype(np.float32) / s_all.astype(np.float32)
            dist = np.abs(n.astype(np.float64) - float(t)) / np.spacing(np.float32(abs(t)))
            sel = ok & (dist <= 1.0)
            for xv, sv in zip(x[sel], s_all[sel]):
                rows.append((xv, sv))
    pairs = sorted(set((int(np.float16(x).view(np.uint16)), int(np.float16(s).view(np.uint16)))
                       for x, s in rows))
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "near_threshold_pairs.txt")
    with open(path, "w") as f:
        f.write("# x_fp16_hex s_fp16_hex code  -- written by tests/golden/make_golden.py (oracle only)\n")
        f.write("# each pair: block {s, x}; n = RN32(x/s) within 1 fp32 ulp of a threshold T_i\n")
        for xb, sb in pairs:
            x = np.array([xb], np.uint16).view(np.float16)
            s = np.array([sb], np.uint16).view(np.float16)
            _, c = O.quantize_blocks(np.concatenate([s, x]).reshape(1, 2))
            f.write(f"{xb:04x} {sb:04x} {int(c[0, 1])}\n")
    print(len(pairs), "pairs ->", path)


if __name__ == "__main__":
    main()
