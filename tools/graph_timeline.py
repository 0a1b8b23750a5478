"""Per-launch conv spans and inter-launch gaps of one graph-replayed sparse edit
(config 2, F16); each row names its launch slot ([gtl i] — the library prints
the slot's conv shape and plan to stderr at capture). Needs SIGE_TC_GTL=1 (device-side globaltimer stamps written by
every k_conv_tc launch; see conv_tc.cu debug_conv_timeline)."""
import ctypes as C
import os
import sys

sys.path.insert(0, ".")
os.environ.setdefault("SIGE_TC_GTL", "1")
import torch  # noqa: E402

import paper_2211_02048_b200 as sb  # noqa: E402
from paper_2211_02048_b200 import _capi  # noqa: E402

lib = sb._lib()
lib.sige_debug_conv_timeline.restype = C.c_int
lib.sige_debug_conv_timeline.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
lib.sige_debug_conv_marks.restype = C.c_int
lib.sige_debug_conv_marks.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]

m = sb.Model("ddim_stack")
c, h, w = m.in_shape
o, e = sb.make_edit_fixture("rect1", 1, c, h, w, 7)
eng = sb.Engine(m, math=sb.MATH_F16)
eng.precompute(o.cuda())
cfg = sb.default_config(dilate_full=5, min_sparse_res=64)
ed = e.cuda()
out = torch.empty(eng.output_shape(), device="cuda")
for _ in range(4):
    eng.sparse_forward(ed, config=cfg, out=out)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 3072)()
lib.sige_debug_conv_timeline(buf, 1024)  # reset
flush = torch.empty(128 * 1024 * 1024, device="cuda")
flush.zero_()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
eng.sparse_forward(ed, config=cfg, out=out)
b.record()
torch.cuda.synchronize()
STRIDE = 64 + 3 * 160  # conv_tc.cu kMarkStride
marks = (C.c_ulonglong * (STRIDE * 1024))()
lib.sige_debug_conv_marks(marks, 1024)
n = lib.sige_debug_conv_timeline(buf, 1024)
rows = [(buf[3 * i], buf[3 * i + 1], buf[3 * i + 2], i) for i in range(n) if buf[3 * i + 1]]
t0 = rows[0][0]
print(f"step {a.elapsed_time(b):.3f} ms (events), {len(rows)} conv launches")
print("idx   start(us)  wait_done  end     work=end-wait  handoff=wait-prev_end")
prev_end = None
tot_work = tot_hand = 0.0
for i, (s, en, wd, gi) in enumerate(rows):
    work = (en - wd) / 1e3
    hand = (wd - prev_end) / 1e3 if prev_end else 0.0
    tot_work += work
    tot_hand += hand
    print(f"{i:3d} {(s - t0) / 1e3:9.2f} {(wd - t0) / 1e3:9.2f} {(en - t0) / 1e3:9.2f} {work:8.2f} {hand:8.2f}"
          f"  [gtl {gi}]")
    prev_end = en
print()
print("CTA 0 phases (us): wait->A landed (22-49), MMAs (9-22), acc ready (5-9), epilogue (47-5), "
      "teardown (13-47); reduce-scatter (52-53) when split")


def mk(gi, k):
    v = marks[gi * STRIDE + k]
    return v if v else None


acc = {}
for i, (s_, en, wd, gi) in enumerate(rows):
    m = {k: mk(gi, k) for k in (49, 22, 9, 5, 47, 13, 52, 53)}
    def d(a, b):
        return (m[a] - m[b]) / 1e3 if m[a] and m[b] else float("nan")
    ph = [d(22, 49), d(9, 22), d(5, 9), d(47, 5), d(13, 47), d(52, 53)]
    print(f"{i:3d} " + " ".join(f"{v:6.2f}" for v in ph) + f"  [gtl {gi}]")
    for j, v in enumerate(ph):
        if v == v:
            acc[j] = acc.get(j, 0.0) + v
print("sums " + " ".join(f"{acc.get(j, 0.0):7.1f}" for j in range(6)))
import json
with open(os.environ.get("SIGE_TL_MARKS_OUT", "gpurun_out/tl_marks.json"), "w") as f:
    json.dump([{"slot": gi, "start": s_, "end": en, "wait": wd,
                "marks": {k: marks[gi * STRIDE + k] for k in range(64) if marks[gi * STRIDE + k]},
                "ctas": [[marks[gi * STRIDE + 64 + 3 * c + j] for j in range(3)] for c in range(160)
                         if marks[gi * STRIDE + 64 + 3 * c]]} for (s_, en, wd, gi) in rows], f)
print(f"sum work {tot_work:.1f} us, sum handoff (incl. non-conv kernels) {tot_hand:.1f} us, "
      f"first->last {(rows[-1][1] - t0) / 1e3:.1f} us")
