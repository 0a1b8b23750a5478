"""Active tiles per conv site of one config-2 edit (RunTrace rows) and the
work items they make for the tensor-core conv (T tiles per M=128 MMA)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2211_02048_b200 as sb  # noqa: E402

m = sb.Model("ddim_stack")
o, e = sb.make_edit_fixture("rect1", 1, 3, 256, 256, 7)
eng = sb.Engine(m, math=sb.MATH_F16)
eng.precompute(o.cuda())
cfg = sb.default_config(dilate_full=5, min_sparse_res=64)
eng.sparse_forward(e.cuda(), config=cfg)
tr = eng.trace().numpy()
for i, r in enumerate(tr):
    if r[5] == 1:
        print(f"{i:3d} tiles {r[0]:5d} items(T2) {(r[0] + 1) // 2:5d} per-CTA max {-(-((r[0] + 1) // 2) // 148)}  macs {r[3] / 1e6:8.1f} M")
