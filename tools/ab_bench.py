"""Minimal config-2 edit timing (graph replay, L2 flushed, CUDA events) that
needs only the core entry points — for A/B of library builds from different
commits via SIGE_B200_LIB. Prints one line: label median_ms mean_ms."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2211_02048_b200 as sb  # noqa: E402

label = sys.argv[1] if len(sys.argv) > 1 else "cur"
m = sb.Model("ddim_stack")
o, e = sb.make_edit_fixture("rect1", 1, 3, 256, 256, 7)
eng = sb.Engine(m, math=sb.MATH_F16)
eng.precompute(o.cuda())
cfg = sb.default_config(dilate_full=5, min_sparse_res=64)
x = e.cuda()
out = torch.empty(eng.output_shape(), device="cuda")
for _ in range(5):
    eng.sparse_forward(x, config=cfg, out=out)
flush = torch.empty(128 * 1024 * 1024, device="cuda")
ts = []
for _ in range(40):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    eng.sparse_forward(x, config=cfg, out=out)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ts.sort()
print(f"{label} median {ts[len(ts) // 2]:.4f} mean {sum(ts) / len(ts):.4f} min {ts[0]:.4f}", flush=True)
