"""Split-K plans of the tensor-core conv for static tile counts (the dense
pass and the dense-fallback layers): every (N tile, K split over a thread-block
cluster, partials reduce-scattered over DSMEM) the planner may pick must give
the oracle's result. Integer data makes every partial sum exact, so any
summation order is bit-exact; the config-2 run checks the fused
GroupNorm-statistics epilogue under forced splits against the reference within
the north-star tolerance. Plans are pinned with the
SIGE_FORCE_PLAN="nt:ks" hook, read once per process: each plan runs in a child."""
import json
import os
import pathlib
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = pathlib.Path(__file__).resolve().parents[1]

CHILD = r"""
import json, sys
import numpy as np, torch
sys.path[:0] = [".", "tests"]
import oracle
import paper_2211_02048_b200 as sb
from test_gpu_tc import DescBuilder, int_case
O = oracle.orc()
res = []
for (c_in, c_out, k, h, w) in [(512, 512, 3, 8, 8), (256, 512, 3, 16, 16), (512, 256, 1, 16, 16), (256, 256, 3, 32, 32)]:
    rng = np.random.default_rng(c_in * 7 + h)
    orig, edited, wt, bias = int_case(rng, 1, c_in, c_out, k, 1, h, w)
    model = DescBuilder("int_conv", c_in, h, w).conv(wt, bias, 1).build()
    om = O.model(model.desc.contents)
    eng = sb.Engine(model, batch=1, math=sb.MATH_F16)
    eng.precompute(torch.from_numpy(orig).cuda())
    got = eng.dense_forward(torch.from_numpy(edited).cuda()).cpu().numpy()
    res.append(bool(np.array_equal(got, om.dense_forward(edited))))
print(json.dumps(res))
"""


@pytest.mark.parametrize("plan", ["16:1", "32:2", "64:4", "128:8", "64:2", "256:8", "128:4"])
def test_forced_plan_integer_bit_exact(plan):
    env = dict(os.environ, SIGE_FORCE_PLAN=plan)
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert all(res), res


CHILD_C2 = r"""
import json, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
import oracle
import paper_2211_02048_b200 as sb
R = oracle.ref()
os.environ.setdefault("SIGE_THREADS", str(os.cpu_count() or 1))
rm = R.model("ddim_stack")
orig, edited = R.make_edit_fixture("rect1", 1, 3, 256, 256, 7)
mask = R.difference_mask(orig, edited)
cfg = sb.default_config(dilate_full=5, min_sparse_res=64)
cache = rm.precompute(orig)
want, _ = rm.sparse_forward(cache, edited, mask, cfg)
eng = sb.Engine(sb.Model("ddim_stack"), math=sb.MATH_F16)
eng.precompute(torch.from_numpy(orig).cuda())
x = torch.from_numpy(edited).cuda()
outs = [eng.sparse_forward(x, config=cfg).cpu().numpy() for _ in range(3)]
err = float(np.abs(outs[0] - want).max() / np.abs(want).max())
print(json.dumps({"err": err, "replay_same": all(np.array_equal(o, outs[0]) for o in outs)}))
"""


@pytest.mark.skipif(not (ROOT / "oracle" / "_ref" / "libsigeref.so").exists(), reason="reference library not built")
@pytest.mark.parametrize("plan", ["128:8", "64:4"])
def test_forced_plan_config2_tolerance(plan):
    env = dict(os.environ, SIGE_FORCE_PLAN=plan)
    r = subprocess.run([sys.executable, "-c", CHILD_C2], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    print(plan, res)
    assert res["replay_same"] and res["err"] <= 1e-2, res
