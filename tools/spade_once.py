"""Config-3 edits (gaugan_spade, F16, every layer sparse, dilation 1) for an ncu launch list."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2211_02048_b200 as sb  # noqa: E402

m = sb.Model("gaugan_spade")
c, h, w = m.in_shape
o, e = sb.make_seg_fixture(1, c, h, w, 11)
eng = sb.Engine(m, math=sb.MATH_F16)
eng.set_graphs(False)
eng.precompute(o.cuda())
cfg = sb.default_config(dilate_full=1, dilate_scale=1, min_sparse_res=1)
x = e.cuda()
for _ in range(3):
    eng.sparse_forward(x, config=cfg)
torch.cuda.synchronize()
print("launches per edit", eng.last_launch_count())
