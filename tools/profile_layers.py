"""Per-conv-launch timing of one config-2 sparse edit and one dense pass
(CUDA events around every fused conv launch; see Engine.set_profiling)."""
import argparse
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2211_02048_b200 as sb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--math", default="f16")
ap.add_argument("--model", default="ddim_stack")
ap.add_argument("--no-graphs", action="store_true")
args = ap.parse_args()
math = {"f16": sb.MATH_F16, "tf32": sb.MATH_TF32, "exact": sb.MATH_EXACT}[args.math]
m = sb.Model(args.model)
c, h, w = m.in_shape
o, e = sb.make_edit_fixture("rect1", 1, c, h, w, 7)
eng = sb.Engine(m, math=math)
eng.set_graphs(not args.no_graphs)
eng.precompute(o.cuda())
cfg = sb.default_config(dilate_full=5, min_sparse_res=64)
ed = e.cuda()
for _ in range(3):
    eng.sparse_forward(ed, config=cfg)
torch.cuda.synchronize()
flush = torch.empty(128 * 1024 * 1024, device="cuda")
for label, fn in [("sparse", lambda: eng.sparse_forward(ed, config=cfg)), ("dense", lambda: eng.dense_forward(ed))]:
    flush.zero_()
    eng.set_profiling(True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    eng.set_profiling(False)
    torch.cuda.synchronize()
    rows = eng.profile_read().numpy()
    tot = a.elapsed_time(b)
    print(f"== {label}: total {tot:.3f} ms, conv launches {len(rows)}, conv sum {rows[:, 0].sum():.3f} ms, "
          f"flops {rows[:, 1].sum() / 1e9:.2f} GF")
    for i, r in enumerate(rows):
        tf = r[1] / (r[0] * 1e-3) / 1e12 if r[0] > 0 else 0
        print(f"  {i:3d} {r[0] * 1e3:9.1f} us {r[1] / 1e9:9.3f} GF {tf:8.2f} TF/s")
