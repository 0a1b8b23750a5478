"""Per-conv-launch timing of one grouped config-2 call (R requests in one
engine, Engine.sparse_forward_grouped) with CUDA events around every fused conv
(Engine.set_profiling): where a batched round's time goes."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2211_02048_b200 as sb  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 32
GRAPHS = "--no-graphs" not in sys.argv
model = sb.Model("ddim_stack")
cfg = sb.default_config(dilate_full=5, min_sparse_res=64)
os_, es_ = zip(*[sb.make_edit_fixture("rect1", 1, 3, 256, 256, 7 + i) for i in range(R)])
eng = sb.Engine(model, batch=R, math=sb.MATH_F16)
eng.set_graphs(GRAPHS)
eng.precompute(torch.cat(os_).cuda())
x = torch.cat(es_).cuda()
out = torch.empty(eng.output_shape(), device="cuda")
for _ in range(3):
    eng.sparse_forward_grouped(x, config=cfg, out=out)
torch.cuda.synchronize()
flush = torch.empty(128 * 1024 * 1024, device="cuda")
flush.zero_()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
eng.sparse_forward_grouped(x, config=cfg, out=out)
b.record()
torch.cuda.synchronize()
print(f"graph replay: {a.elapsed_time(b):.3f} ms for {R} requests")
eng.set_profiling(True)
flush.zero_()
a.record()
eng.sparse_forward_grouped(x, config=cfg, out=out)
b.record()
eng.set_profiling(False)
torch.cuda.synchronize()
rows = eng.profile_read().numpy()
print(f"profiled call: {a.elapsed_time(b):.3f} ms, {len(rows)} conv launches, conv sum {rows[:, 0].sum():.3f} ms, "
      f"{rows[:, 1].sum() / 1e9:.1f} GFLOP")
for i, r in enumerate(rows):
    print(f"{i:3d} {r[0] * 1e3:8.1f} us {r[1] / 1e9:8.2f} GFLOP {r[1] / max(r[0], 1e-9) / 1e9:8.1f} TF/s")
