"""Time the §8(f) row-4 KV-layout decode cases (bench.layouts_config: c5
shard shape, contiguous / paged-256 / gqa-4) and print one JSON line.
NQKV_GQA_NATIVE=0 routes GQA through the per-query-head MHA kernel."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import __graft_entry__  # noqa: E402

__graft_entry__.build()
peak = json.load(open(os.path.join(os.path.dirname(bench.__file__), "MEASURED_PEAKS.json")))["hbm_gbs"]
res = bench.layouts_config(torch.device("cuda"), peak)
print(json.dumps({k: (v["us_per_launch"], round(v["decode_roofline"]["frac"], 3)) for k, v in res.items()
                  if isinstance(v, dict)}))
