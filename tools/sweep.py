"""BASELINE config 4: edit-area sweep (0.5 %-30 %) x block-size sweep on the
DDIM-shaped stack (config 2 model), sparse vs dense B200 pass, F16.
Edits are the reference's rect fixtures for 1.2/5/15/35 % and squares placed
like fixtures.cpp:26-34 for the other areas. One JSON line per point."""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2211_02048_b200 as sb  # noqa: E402


def timed(fn, reps=10):
    flush = torch.empty(128 * 1024 * 1024, device="cuda")
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    m = sb.Model("ddim_stack")
    c, h, w = m.in_shape
    orig, _ = sb.make_edit_fixture("rect1", 1, c, h, w, 7)
    eng = sb.Engine(m, math=sb.MATH_F16)
    eng.precompute(orig.cuda())
    o = orig.cuda()
    dense = timed(lambda: eng.dense_forward(o))
    g = torch.Generator().manual_seed(7)
    for area in [0.005, 0.012, 0.05, 0.10, 0.15, 0.20, 0.30]:
        side = max(1, int(round((area * h * w) ** 0.5)))
        y0 = int(torch.randint(0, h - side + 1, (1,), generator=g))
        x0 = int(torch.randint(0, w - side + 1, (1,), generator=g))
        ed = orig.clone()
        ed[:, :, y0:y0 + side, x0:x0 + side] += 0.3
        edd = ed.cuda()
        for b3, b1 in [(6, 4), (8, 4), (4, 4)]:
            cfg = sb.default_config(dilate_full=5, min_sparse_res=64, block3=b3, block1=b1)
            try:
                t = timed(lambda: eng.sparse_forward(edd, config=cfg))
                tr = eng.trace().numpy()
                macs, dmacs = int(tr[:, 3].sum()), int(tr[:, 4].sum())
                print(json.dumps({"area_pct": round(100 * side * side / (h * w), 2), "block3": b3, "block1": b1,
                                  "sparse_ms": round(t, 4), "dense_ms": round(dense, 4),
                                  "speedup": round(dense / t, 3), "mac_reduction": round(dmacs / max(macs, 1), 3)}),
                      flush=True)
            except Exception as e:  # report the failing point, keep sweeping
                print(json.dumps({"area_pct": round(100 * side * side / (h * w), 2), "block3": b3, "error": str(e)}),
                      flush=True)


if __name__ == "__main__":
    main()
