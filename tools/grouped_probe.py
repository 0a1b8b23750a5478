"""Memory and time of grouped config-2 requests (config 5 on one GPU) per group size."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2211_02048_b200 as sb  # noqa: E402

model = sb.Model("ddim_stack")
cfg = sb.default_config(dilate_full=5, min_sparse_res=64)
flush = torch.empty(128 * 1024 * 1024, device="cuda")
for R in [int(a) for a in sys.argv[1:]] or [8, 16, 32]:
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    os_, es_ = zip(*[sb.make_edit_fixture("rect1", 1, 3, 256, 256, 7 + i) for i in range(R)])
    eng = sb.Engine(model, batch=R, math=sb.MATH_F16)
    eng.precompute(torch.cat(os_).cuda())
    x = torch.cat(es_).cuda()
    out = torch.empty(eng.output_shape(), device="cuda")
    for _ in range(3):
        eng.sparse_forward_grouped(x, config=cfg, out=out)
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    ts = []
    for _ in range(10):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.sparse_forward_grouped(x, config=cfg, out=out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sorted(ts)[len(ts) // 2]
    print(json.dumps({"R": R, "gb": round((free0 - free1) / 1e9, 2), "gb_per_request": round((free0 - free1) / 1e9 / R, 3),
                      "ms": round(ms, 3), "edits_per_s": round(R * 1e3 / ms, 1)}), flush=True)
    del eng, x, out
    torch.cuda.empty_cache()
