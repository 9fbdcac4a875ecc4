"""Development: where does the prefill kernel differ from the oracle?  Prints
per (b, h) and per 32-row band the max error, for each hd/blk case."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_2505_16210_b200 import nqkv as N  # noqa: E402
import test_gpu_parity as T  # noqa: E402

for hd, blk in ((64, 64), (128, 64)):
    lens = [0, 1, 63, 64, 65, 200]
    out, ref = T._prefill_case(N, len(lens), 200, 2, hd, blk, lens, 256, seed=hd + blk)
    e = np.abs(out.astype(np.float64) - ref)
    print("hd", hd, "blk", blk, "max", e.max())
    for b in range(len(lens)):
        for h in range(2):
            bands = [f"{e[b, r:r + 32, h].max():.1e}" for r in range(0, 200, 32)]
            print(f"  b{b} len {lens[b]:3d} h{h}:", " ".join(bands))
    # columns of the worst row
    bb, rr, hh, cc = np.unravel_index(np.argmax(e), e.shape)
    print("  worst b,row,h,col", bb, rr, hh, cc, "cols with err>1e-3:", np.nonzero(e[bb, rr, hh] > 1e-3)[0][:40])
