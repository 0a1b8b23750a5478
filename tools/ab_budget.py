"""Config-2 edit time under Engine.set_sm_budget(B) for B in argv (grid-size experiment)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2211_02048_b200 as sb  # noqa: E402

m = sb.Model("ddim_stack")
o, e = sb.make_edit_fixture("rect1", 1, 3, 256, 256, 7)
flush = torch.empty(128 * 1024 * 1024, device="cuda")
for b in [int(a) for a in sys.argv[1:]]:
    eng = sb.Engine(m, math=sb.MATH_F16)
    eng.set_sm_budget(b)
    eng.precompute(o.cuda())
    cfg = sb.default_config(dilate_full=5, min_sparse_res=64)
    x = e.cuda()
    out = torch.empty(eng.output_shape(), device="cuda")
    for _ in range(5):
        eng.sparse_forward(x, config=cfg, out=out)
    ts = []
    for _ in range(30):
        flush.zero_()
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.sparse_forward(x, config=cfg, out=out)
        c.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(c))
    ts.sort()
    print(f"budget {b}: median {ts[len(ts) // 2]:.4f} ms min {ts[0]:.4f}", flush=True)
    del eng
