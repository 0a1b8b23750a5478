"""Throughput of R independent requests in flight on one GPU vs per-request SM budget."""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2211_02048_b200 as sb  # noqa: E402

m = sb.Model("ddim_stack")
cfg = sb.default_config(dilate_full=5, min_sparse_res=64)
sms = torch.cuda.get_device_properties(0).multi_processor_count
for R, budget in [(1, 0), (4, 0), (4, sms // 4), (4, sms // 2), (8, sms // 8), (8, sms // 4), (8, sms // 2)]:
    r = bench.batched_requests(sb, torch, m, cfg, sb.MATH_F16, R=R, sms=budget or None)
    print(json.dumps(r), flush=True)
    torch.cuda.empty_cache()
