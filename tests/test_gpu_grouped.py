"""Grouped independent requests (BASELINE config 5 on one GPU): one engine of
batch R serves R requests — each its own original (precompute), edited input
and difference mask — with per-sample IndexPlans concatenated n-major into
each layer's tile list (one launch per layer for all requests). Every
request's output must equal what the reference's sparse_forward
(graph.cpp:619-901) gives for that request alone: bit-exact in
SIGE_MATH_EXACT (checked against the oracle per request), and equal to R
separate batch-1 engines in the tensor-core mode within the north-star
tolerance. An empty-mask request returns its cached final output."""
import numpy as np
import pytest
import torch

import paper_2211_02048_b200 as sb

pytestmark = pytest.mark.gpu


def requests(orc, name, fixtures, c, h, w):
    origs, edits = [], []
    for fx, seed in fixtures:
        if fx == "none":  # a request whose edit changes nothing
            o, _ = orc.make_edit_fixture("rect5", 1, c, h, w, seed)
            e = o.copy()
        else:
            o, e = orc.make_edit_fixture(fx, 1, c, h, w, seed)
        origs.append(o)
        edits.append(e)
    return np.concatenate(origs), np.concatenate(edits)


@pytest.mark.parametrize("explicit_masks", [False, True])
def test_grouped_exact_matches_per_request_oracle(orc, explicit_masks):
    name = "mini_unet_gn"
    om = orc.model(name)
    fixtures = [("rect5", 3), ("blob5", 4), ("none", 5), ("rect15", 6), ("multi15", 7)]
    orig, edited = requests(orc, name, fixtures, 3, 64, 64)
    R = len(fixtures)
    cfg = sb.default_config(dilate_full=om.required_dilation())
    eng = sb.Engine(sb.Model(name), batch=R, math=sb.MATH_EXACT)
    eng.precompute(torch.from_numpy(orig).cuda())
    masks = np.stack([orc.difference_mask(orig[i:i + 1], edited[i:i + 1]) for i in range(R)])
    out = torch.empty(eng.output_shape(), device="cuda")
    for rep in range(3):  # direct, capture, replay
        eng.sparse_forward_grouped(torch.from_numpy(edited).cuda(),
                                   torch.from_numpy(masks).cuda() if explicit_masks else None, config=cfg, out=out)
        got = out.cpu().numpy()
        for i in range(R):
            cache = om.precompute(orig[i:i + 1])
            want, _ = om.sparse_forward(cache, edited[i:i + 1], masks[i], cfg)
            assert np.array_equal(got[i].view(np.uint32), want[0].view(np.uint32)), (rep, i)
    assert masks[2].sum() == 0  # the no-op request short-circuits to its cached final
    # grouped and shared-mask programs coexist on one engine: the plain call
    # ORs the masks over the batch (compute_difference_mask, mask.cpp:14-32)
    plain = eng.sparse_forward(torch.from_numpy(edited).cuda(), config=cfg).cpu().numpy()
    shared = np.any(masks, axis=0).astype(np.uint8)
    want, _ = om.sparse_forward(om.precompute(orig), edited, shared, cfg)
    assert np.array_equal(plain, want)


def test_grouped_config2_f16_equals_separate_engines(orc):
    """4 config-2 requests (ddim_stack 3x256x256, rect1 seeds 7..10) grouped vs
    one batch-1 engine per request, F16."""
    model = sb.Model("ddim_stack")
    cfg = sb.default_config(dilate_full=5, min_sparse_res=64)
    R = 4
    os_, es_ = [], []
    for i in range(R):
        o, e = sb.make_edit_fixture("rect1", 1, 3, 256, 256, 7 + i)
        os_.append(o)
        es_.append(e)
    orig, edited = torch.cat(os_), torch.cat(es_)
    g = sb.Engine(model, batch=R, math=sb.MATH_F16)
    g.precompute(orig.cuda())
    x = edited.cuda()
    out = torch.empty(g.output_shape(), device="cuda")
    for _ in range(3):
        g.sparse_forward_grouped(x, config=cfg, out=out)
    got = out.cpu().numpy()
    for i in range(R):
        e1 = sb.Engine(model, batch=1, math=sb.MATH_F16)
        e1.precompute(os_[i].cuda())
        want = e1.sparse_forward(es_[i].cuda(), config=cfg).cpu().numpy()[0]
        err = float(np.abs(got[i] - want).max() / np.abs(want).max())
        assert err <= 1e-2, (i, err)
    tr = g.trace().numpy()
    assert int(tr[tr[:, 5] == 1, 0].sum()) > 1132  # every request's tiles in one plan
