"""Run the op-level gather / scatter / difference mask once each at the
ops_hbm workload (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2211_02048_b200 as sb  # noqa: E402

dev = torch.device("cuda", 0)
n, c, h, w, b = 8, 128, 256, 256, 6
g = torch.Generator(device="cpu").manual_seed(11)
orig = torch.rand((n, c, h, w), generator=g).to(dev) * 2 - 1
edited = orig.clone()
side = int(round((0.30 * h * w) ** 0.5))
edited[:, :, 40:40 + side, 60:60 + side] += 0.25
mask = sb.compute_difference_mask(orig, edited, 1e-3)
idx = sb.mask_to_block_indices(sb.dilate_mask(mask, 1), b, n)
out_blocks = torch.rand((int(idx.shape[0]), c, b, b), generator=g).to(dev)
base = orig.clone()
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
for _ in range(2):
    flush.zero_()
    sb.gather(edited, idx, b, 3, 1)
    flush.zero_()
    sb.scatter_inplace(out_blocks, idx, base)
torch.cuda.synchronize()
print("tiles", int(idx.shape[0]))
