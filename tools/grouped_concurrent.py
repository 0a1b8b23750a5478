"""64 config-2 requests on one GPU: two grouped engines of 32 run one after the
other (bench.py's schedule) vs concurrently on two streams (SM budget B each)."""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2211_02048_b200 as sb  # noqa: E402

model = sb.Model("ddim_stack")
cfg = sb.default_config(dilate_full=5, min_sparse_res=64)
G, R = int(sys.argv[1]), int(sys.argv[2])
budgets = [0]
runs = []
for gi in range(G):
    fx = [sb.make_edit_fixture("rect1", 1, 3, 256, 256, 7 + gi * R + i) for i in range(R)]
    eng = sb.Engine(model, batch=R, math=sb.MATH_F16)
    eng.precompute(torch.cat([o for o, _ in fx]).cuda())
    x = torch.cat([e for _, e in fx]).cuda()
    runs.append((eng, x, torch.empty(eng.output_shape(), device="cuda"), torch.cuda.Stream()))
flush = torch.empty(128 * 1024 * 1024, device="cuda")


def timed(fn, reps=8):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        for _, _, _, s in runs:
            torch.cuda.current_stream().wait_stream(s)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


def sequential():
    for eng, x, y, _ in runs:
        eng.sparse_forward_grouped(x, config=cfg, out=y)


def concurrent():
    cur = torch.cuda.current_stream()
    for eng, x, y, s in runs:
        s.wait_stream(cur)
        with torch.cuda.stream(s):
            eng.sparse_forward_grouped(x, config=cfg, out=y)


print(json.dumps({"sequential_ms": round(timed(sequential), 3)}), flush=True)
for b in budgets:
    for eng, _, _, _ in runs:
        eng.set_sm_budget(b)
    t = timed(concurrent)
    print(json.dumps({"concurrent_budget": b, "ms": round(t, 3), "edits_per_s": round(G * R * 1e3 / t, 1)}), flush=True)
