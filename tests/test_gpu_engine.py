"""GPU parity of the engine (device ActivationCache + sparse executor).

SIGE_MATH_EXACT must reproduce the oracle's sparse_forward bit for bit (the
oracle is itself bit-identical to the reference, tests/test_oracle_vs_ref.py),
both with the cache uploaded from the CPU precompute and with the device
precompute. SIGE_MATH_TF32 is held to the north-star tolerance (normalised
max error <= 1e-2) with uncovered pixels bit-identical to the cache."""
import numpy as np
import pytest
import torch

import paper_2211_02048_b200 as sb

pytestmark = pytest.mark.gpu


def upload_cache(eng, ocache, entries):
    for kind, key, numel in entries:
        if kind == 0:
            eng.put_tensor(key, ocache.tensor(key))
        else:
            sc, sh = ocache.norm(key)
            eng.put_norm(key, sc, sh)


CASES = [
    # model, fixture, batch, seed, config overrides (dilate_full None = required)
    ("mini_unet_gn", "rect5", 1, 17, {}),
    ("mini_unet_gn", "blob5", 2, 5, {"norm_precompute": 0}),
    ("mini_unet_bn", "rect15", 1, 11, {"dilate_full": 3}),
    ("gaugan_stack_in", "multi15", 1, 3, {}),
    ("ddim_stack_64x32", "rect5", 1, 7, {"dilate_full": 5, "min_sparse_res": 16}),
    ("ddim_stack_64x32", "rect1", 2, 8, {"dilate_full": 2, "min_sparse_res": 8, "block3": 4, "block1": 2}),
    ("ddim_stack_64x32", "rect1", 1, 9, {"dilate_full": 2, "min_sparse_res": 8, "dilate_scale": 0}),
]


def run_case(orc, name, fx, n, seed, over, math, device_precompute):
    om = orc.model(name)
    c, h, w = sb.Model(name).in_shape
    orig, edited = orc.make_edit_fixture(fx, n, c, h, w, seed)
    mask = orc.difference_mask(orig, edited)
    over = dict(over)
    df = over.pop("dilate_full", None)
    cfg = sb.default_config(dilate_full=om.required_dilation() if df is None else df, **over)
    ocache = om.precompute(orig)
    want, wtrace = om.sparse_forward(ocache, edited, mask, cfg)
    eng = sb.Engine(sb.Model(name), batch=n, math=math)
    if device_precompute:
        eng.precompute(torch.from_numpy(orig).cuda())
    else:
        upload_cache(eng, ocache, ocache.entries())
        eng.put_tensor("input", orig)
    got = eng.sparse_forward(torch.from_numpy(edited).cuda(), config=cfg)
    torch.cuda.synchronize()
    return want, got.cpu().numpy(), wtrace, eng.trace().numpy().astype(np.uint64), ocache


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}-{c[1]}-n{c[2]}" for c in CASES])
@pytest.mark.parametrize("device_precompute", [False, True])
def test_exact_engine_bit_exact(orc, case, device_precompute):
    want, got, wtr, gtr, _ = run_case(orc, *case, sb.MATH_EXACT, device_precompute)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), f"max diff {np.abs(got - want).max()}"
    assert np.array_equal(gtr, wtr)


def test_exact_engine_config1_full_size(orc):
    """BASELINE config 1: 1x64x256x256, 3x3 conv, rect1, b=6 — bit-exact."""
    want, got, wtr, gtr, _ = run_case(orc, "single_conv64", "rect1", 1, 7, {"dilate_full": 1}, sb.MATH_EXACT, True)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    assert gtr[0][0] == 36  # 36 active tiles


def test_user_mask_and_empty_mask(orc):
    om = orc.model("mini_unet_gn")
    orig, edited = orc.make_edit_fixture("rect5", 1, 3, 64, 64, 3)
    eng = sb.Engine(sb.Model("mini_unet_gn"), math=sb.MATH_EXACT)
    eng.precompute(torch.from_numpy(orig).cuda())
    cfg = sb.default_config(dilate_full=25)
    mask = orc.difference_mask(orig, edited)
    a = eng.sparse_forward(torch.from_numpy(edited).cuda(), config=cfg).cpu().numpy()
    b = eng.sparse_forward(torch.from_numpy(edited).cuda(), torch.from_numpy(mask).cuda(), config=cfg).cpu().numpy()
    assert np.array_equal(a, b)
    # all-false mask short-circuits to the cached final output (graph.cpp:665-668)
    empty = torch.zeros((64, 64), dtype=torch.uint8, device="cuda")
    c = eng.sparse_forward(torch.from_numpy(edited).cuda(), empty, config=cfg).cpu().numpy()
    ocache = om.precompute(orig)
    assert np.array_equal(c, ocache.tensor("final"))
    # repeated calls (lazy tile restore) stay identical
    d = eng.sparse_forward(torch.from_numpy(edited).cuda(), config=cfg).cpu().numpy()
    assert np.array_equal(a, d)


def test_precompute_matches_oracle_cache_exact(orc):
    om = orc.model("mini_unet_gn")
    orig, _ = orc.make_edit_fixture("rect5", 1, 3, 64, 64, 2)
    ocache = om.precompute(orig)
    eng = sb.Engine(sb.Model("mini_unet_gn"), math=sb.MATH_EXACT)
    eng.precompute(torch.from_numpy(orig).cuda())
    torch.cuda.synchronize()
    for kind, key, numel in ocache.entries():
        if kind == 0:
            want = ocache.tensor(key)
            got = eng.get_tensor(key, want.shape).numpy()
            assert np.array_equal(got, want), key


def test_dense_forward_matches_oracle(orc):
    om = orc.model("mini_unet_gn")
    orig, edited = orc.make_edit_fixture("rect5", 1, 3, 64, 64, 21)
    eng = sb.Engine(sb.Model("mini_unet_gn"), math=sb.MATH_EXACT)
    eng.precompute(torch.from_numpy(orig).cuda())
    got = eng.dense_forward(torch.from_numpy(edited).cuda()).cpu().numpy()
    assert np.array_equal(got, om.dense_forward(edited))
    ocache = om.precompute(orig)
    got = eng.dense_forward(torch.from_numpy(edited).cuda(), reused_stats=True).cpu().numpy()
    assert np.array_equal(got, om.dense_forward(edited, ocache))


def test_errors_like_reference(orc):
    eng = sb.Engine(sb.Model("mini_unet_gn"), math=sb.MATH_EXACT)
    x = torch.zeros((1, 3, 64, 64), device="cuda")
    with pytest.raises(sb.ConfigError, match="precompute required"):
        eng.sparse_forward(x)
    with pytest.raises(sb.ConfigError, match="config: block sizes must be >= 1"):
        eng.sparse_forward(x, config=sb.default_config(block3=0))


@pytest.mark.parametrize("math", [sb.MATH_EXACT, sb.MATH_F16])
def test_graph_replay_identical(orc, math):
    """CUDA-graph replay (default after the first call) gives the same bits as
    direct launches, across repeated calls and a switch of edited input."""
    orig, edited = orc.make_edit_fixture("rect5", 1, 3, 64, 64, 31)
    _, edited2 = orc.make_edit_fixture("blob5", 1, 3, 64, 64, 31)
    cfg = sb.default_config(dilate_full=25)
    outs = {}
    for graphs in (False, True):
        eng = sb.Engine(sb.Model("mini_unet_gn"), math=math)
        eng.set_graphs(graphs)
        eng.precompute(torch.from_numpy(orig).cuda())
        e1, e2 = torch.from_numpy(edited).cuda(), torch.from_numpy(edited2).cuda()
        out = torch.empty(eng.output_shape(), device="cuda")
        res = []
        for x in (e1, e1, e1, e2, e1):
            eng.sparse_forward(x, config=cfg, out=out)
            res.append(out.cpu().numpy().copy())
        outs[graphs] = res
    for a, b in zip(outs[False], outs[True]):
        assert np.array_equal(a, b)
    assert np.array_equal(outs[True][0], outs[True][4])


def test_graph_replay_follows_threshold(orc):
    """Without a mask the threshold is part of the captured call: alternating
    thresholds on the same buffers with graphs on must give the same bits as
    direct launches (compute_difference_mask's strict '>' at each threshold,
    mask.cpp:14-32)."""
    orig, _ = orc.make_edit_fixture("rect5", 1, 3, 64, 64, 41)
    edited = orig.copy()
    edited[:, :, 5:11, 5:11] += 0.1  # below the 0.3 threshold
    edited[:, :, 40:46, 30:36] -= 1.0  # above it
    outs = {}
    for graphs in (False, True):
        eng = sb.Engine(sb.Model("mini_unet_gn"), math=sb.MATH_EXACT)
        eng.set_graphs(graphs)
        eng.precompute(torch.from_numpy(orig).cuda())
        x = torch.from_numpy(edited).cuda()
        out = torch.empty(eng.output_shape(), device="cuda")
        res = []
        for thr in (1e-3, 1e-3, 0.3, 1e-3, 0.3, 0.3, 10.0):
            eng.sparse_forward(x, config=sb.default_config(dilate_full=1, min_sparse_res=1, mask_threshold=thr), out=out)
            res.append(out.cpu().numpy().copy())
        outs[graphs] = res
    for a, b in zip(outs[False], outs[True]):
        assert np.array_equal(a, b)
    m_lo, m_hi = orc.difference_mask(orig, edited, 1e-3), orc.difference_mask(orig, edited, 0.3)
    assert m_hi.sum() < m_lo.sum()
    assert not np.array_equal(outs[True][0], outs[True][2])  # 0.3 drops part of the edit
    om = orc.model("mini_unet_gn")
    ocache = om.precompute(orig)
    for i, thr in ((2, 0.3), (6, 10.0)):
        want, _ = om.sparse_forward(ocache, edited, orc.difference_mask(orig, edited, thr),
                                    sb.default_config(dilate_full=1, min_sparse_res=1))
        assert np.array_equal(outs[True][i], want)


def test_engine_rejects_bad_buffers(orc):
    """Shape / dtype / device of the edited input, the mask and a caller's out
    are checked before any device access (check_inputs, graph.cpp:606-614)."""
    orig, edited = orc.make_edit_fixture("rect5", 1, 3, 64, 64, 2)
    eng = sb.Engine(sb.Model("mini_unet_gn"), math=sb.MATH_EXACT)
    eng.precompute(torch.from_numpy(orig).cuda())
    x = torch.from_numpy(edited).cuda()
    with pytest.raises(sb.ConfigError, match="forward: input channel mismatch"):
        eng.sparse_forward(torch.zeros((1, 4, 64, 64), device="cuda"))
    with pytest.raises(sb.ConfigError, match="engine expects"):
        eng.sparse_forward(torch.zeros((1, 3, 32, 64), device="cuda"))
    with pytest.raises(sb.ConfigError, match="float32"):
        eng.sparse_forward(x.double())
    with pytest.raises(sb.ConfigError, match="forward: mask is 32x64 but input is 64x64"):
        eng.sparse_forward(x, torch.ones((32, 64), dtype=torch.uint8, device="cuda"))
    with pytest.raises(sb.ConfigError, match="uint8"):
        eng.sparse_forward(x, torch.ones((64, 64), dtype=torch.bool, device="cuda"))
    with pytest.raises(sb.ConfigError, match="out must be"):
        eng.sparse_forward(x, out=torch.empty((1, 3, 64, 32), device="cuda"))
    with pytest.raises(sb.ConfigError, match="out must be"):
        eng.sparse_forward(x, out=torch.empty(eng.output_shape(), device="cuda").transpose(2, 3))
    with pytest.raises(sb.ConfigError, match="host tensor"):
        eng.sparse_forward_host(x)
    with pytest.raises(sb.ConfigError, match="forward: input has 4 channels, model expects 3"):
        eng.dense_forward(torch.zeros((1, 4, 64, 64), device="cuda"))
    # a non-contiguous host mask is copied and kept alive across the call
    m = torch.from_numpy(orc.difference_mask(orig, edited)).t().contiguous().t()
    got = eng.sparse_forward_host(torch.from_numpy(edited), m, config=sb.default_config(dilate_full=25))
    want = eng.sparse_forward(x, m.cuda(), config=sb.default_config(dilate_full=25)).cpu()
    assert torch.equal(got, want)


@pytest.mark.parametrize("math", [sb.MATH_EXACT, sb.MATH_F16])
def test_fusion_toggles_do_not_change_the_output(orc, math):
    """RunConfig.elem_fusion / scatter_fusion (graph.cpp:571-582) select the
    reference's ablation schedule, whose output is identical by the reference's
    own tests (test_graph.cpp:215-250, 'fusion toggles do not change the output
    at all'); the device executor always runs the fused schedule, so every
    toggle combination gives the same bits (and, exact mode, the oracle's)."""
    om = orc.model("mini_unet_gn")
    orig, edited = orc.make_edit_fixture("rect5", 1, 3, 64, 64, 19)
    eng = sb.Engine(sb.Model("mini_unet_gn"), math=math)
    eng.precompute(torch.from_numpy(orig).cuda())
    x = torch.from_numpy(edited).cuda()
    outs = []
    for bits in range(4):
        cfg = sb.default_config(dilate_full=om.required_dilation(), elem_fusion=bits & 1, scatter_fusion=(bits >> 1) & 1)
        outs.append(eng.sparse_forward(x, config=cfg).cpu().numpy())
        if math == sb.MATH_EXACT:
            want, _ = om.sparse_forward(om.precompute(orig), edited, orc.difference_mask(orig, edited), cfg)
            assert np.array_equal(outs[-1], want)
    for o in outs[1:]:
        assert np.array_equal(o.view(np.uint32), outs[0].view(np.uint32))


def test_cache_lifecycle_steps_and_model_guard(orc):
    """Multi-step ActivationCache (graph.hpp:116-176): per-step precompute,
    drop_step (graph.cpp:271-274) frees a step, refresh_step (graph.cpp:437-444)
    replaces one from a new original, and a cache declared for another model
    fails like check_cache_model (graph.cpp:596-603)."""
    name = "mini_unet_gn"
    om = orc.model(name)
    a_orig, a_edit = orc.make_edit_fixture("rect5", 1, 3, 64, 64, 61)
    b_orig, b_edit = orc.make_edit_fixture("blob5", 1, 3, 64, 64, 62)
    eng = sb.Engine(sb.Model(name), math=sb.MATH_EXACT)
    eng.precompute(torch.from_numpy(a_orig).cuda(), step=0)
    eng.precompute(torch.from_numpy(b_orig).cuda(), step=1)
    bytes_two = eng.cache_bytes()

    def run(edit, step):
        cfg = sb.default_config(dilate_full=om.required_dilation(), step=step)
        return eng.sparse_forward(torch.from_numpy(edit).cuda(), config=cfg).cpu().numpy()

    def want(orig, edit):
        cfg = sb.default_config(dilate_full=om.required_dilation())
        return om.sparse_forward(om.precompute(orig), edit, orc.difference_mask(orig, edit), cfg)[0]

    assert np.array_equal(run(a_edit, 0), want(a_orig, a_edit))
    assert np.array_equal(run(b_edit, 1), want(b_orig, b_edit))
    eng.drop_step(1)
    assert eng.cache_bytes() < bytes_two
    with pytest.raises(sb.ConfigError, match="precompute required: no cache entry for step 1"):
        run(b_edit, 1)
    assert np.array_equal(run(a_edit, 0), want(a_orig, a_edit))  # step 0 untouched
    eng.refresh_step(torch.from_numpy(b_orig).cuda(), 0)  # step 0 now holds b's activations
    assert np.array_equal(run(b_edit, 0), want(b_orig, b_edit))
    cache_h, model_h = eng.cache_model_hash()
    assert cache_h == model_h == sb.Model(name).structure_hash()
    eng.set_cache_model_hash(sb.Model("mini_unet_bn").structure_hash())
    with pytest.raises(sb.ConfigError, match="cache was precomputed for a different model than 'mini_unet_gn'"):
        run(b_edit, 0)
    eng.set_cache_model_hash(model_h)
    assert np.array_equal(run(b_edit, 0), want(b_orig, b_edit))


COV_CASES = [
    ("mini_unet_gn", "rect5", 1, 3, {}),
    ("mini_unet_gn", "blob5", 2, 4, {"norm_precompute": 0}),
    ("mini_unet_bn", "rect15", 1, 5, {"dilate_full": 3}),
    ("gaugan_stack_in", "multi15", 1, 6, {}),
    ("ddim_stack_64x32", "rect5", 1, 7, {"dilate_full": 5, "min_sparse_res": 16}),
    ("ddim_stack_64x32", "rect1", 1, 8, {"dilate_full": 2, "min_sparse_res": 8, "block3": 4, "block1": 2}),
    ("ddim_stack", "rect1", 1, 7, {"dilate_full": 5, "min_sparse_res": 64}),
    ("mini_unet_gn", "rect5", 1, 9, {"sparse": 0}),
]


@pytest.mark.parametrize("case", COV_CASES, ids=[f"{c[0]}-{c[1]}-{i}" for i, c in enumerate(COV_CASES)])
def test_output_coverage_matches_reference(orc, ref, case):
    """Device output_coverage (graph.cpp:1078-1129) from the executor's own
    on-device IndexPlan == the reference's, for the computed mask and for an
    explicit (empty) mask; and the sparse output differs from the cache only
    inside it."""
    import ctypes as C

    name, fx, n, seed, over = case
    om = orc.model(name)
    c, h, w = sb.Model(name).in_shape
    orig, edited = orc.make_edit_fixture(fx, n, c, h, w, seed)
    over = dict(over)
    df = over.pop("dilate_full", None)
    cfg = sb.default_config(dilate_full=om.required_dilation() if df is None else df, **over)
    eng = sb.Engine(sb.Model(name), batch=n, math=sb.MATH_F16)
    eng.precompute(torch.from_numpy(orig).cuda())
    mask = orc.difference_mask(orig, edited)
    rm = ref.model(name)
    oc, oh, ow = rm.output_shape()
    want = np.zeros((oh, ow), np.uint8)
    hh, ww = C.c_int(), C.c_int()
    assert ref.lib.ref_output_coverage(rm.h, mask.ctypes.data, h, w, n, C.byref(cfg), want.ctypes.data,
                                       C.byref(hh), C.byref(ww)) == 0
    got = eng.output_coverage(torch.from_numpy(edited).cuda(), config=cfg).cpu().numpy()
    assert np.array_equal(got, want)
    got_m = eng.output_coverage(mask=torch.from_numpy(mask).cuda(), config=cfg).cpu().numpy()
    assert np.array_equal(got_m, want)
    empty = eng.output_coverage(mask=torch.zeros((h, w), dtype=torch.uint8, device="cuda"), config=cfg)
    assert int(empty.sum()) == 0
    out = eng.sparse_forward(torch.from_numpy(edited).cuda(), config=cfg).cpu().numpy()
    fin = eng.get_tensor("final", out.shape).numpy()
    outside = np.broadcast_to(want[None, None] == 0, out.shape)
    assert np.array_equal(out[outside], fin[outside])


@pytest.mark.parametrize("math", [sb.MATH_EXACT, sb.MATH_F16])
def test_offload_and_prefetch_steps(orc, math):
    """Multi-step caches with host offload: an offloaded step's
    device memory is freed, a call on it fails like a missing cache entry,
    prefetch_step on a side stream brings it back and the call gives the same
    bits as before; other steps are untouched."""
    name = "mini_unet_gn"
    om = orc.model(name)
    a_orig, a_edit = orc.make_edit_fixture("rect5", 1, 3, 64, 64, 71)
    b_orig, b_edit = orc.make_edit_fixture("blob5", 1, 3, 64, 64, 72)
    eng = sb.Engine(sb.Model(name), math=math)
    eng.precompute(torch.from_numpy(a_orig).cuda(), step=0)
    eng.precompute(torch.from_numpy(b_orig).cuda(), step=1)
    cfg0 = sb.default_config(dilate_full=om.required_dilation(), step=0)
    cfg1 = sb.default_config(dilate_full=om.required_dilation(), step=1)
    xa, xb = torch.from_numpy(a_edit).cuda(), torch.from_numpy(b_edit).cuda()
    want_a = eng.sparse_forward(xa, config=cfg0).cpu()
    want_b = eng.sparse_forward(xb, config=cfg1).cpu()
    full = eng.cache_bytes()
    eng.offload_step(1)
    assert eng.cache_bytes() < full
    with pytest.raises(sb.ConfigError, match="precompute required"):
        eng.sparse_forward(xb, config=cfg1)
    assert torch.equal(eng.sparse_forward(xa, config=cfg0).cpu(), want_a)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        eng.prefetch_step(1)
    torch.cuda.current_stream().wait_stream(side)
    assert eng.cache_bytes() == full
    for _ in range(3):  # direct, capture, replay
        assert torch.equal(eng.sparse_forward(xb, config=cfg1).cpu(), want_b)
    eng.offload_step(1)  # unchanged step: only the device copy goes
    eng.prefetch_step(1)
    assert torch.equal(eng.sparse_forward(xb, config=cfg1).cpu(), want_b)
    with pytest.raises(sb.ConfigError, match="was not offloaded"):
        eng.prefetch_step(5)
    if math == sb.MATH_EXACT:
        cache = om.precompute(b_orig)
        want, _ = om.sparse_forward(cache, b_edit, orc.difference_mask(b_orig, b_edit),
                                    sb.default_config(dilate_full=om.required_dilation()))
        assert np.array_equal(want_b.numpy(), want)


@pytest.mark.parametrize("math", [sb.MATH_EXACT, sb.MATH_F16])
def test_misaligned_edited_input_same_bits(orc, math):
    """The edited input is the caller's tensor: a view at a one-float offset
    (off 16-byte alignment) takes the scalar mask loads and gives the aligned
    tensor's bits."""
    orig, edited = orc.make_edit_fixture("rect5", 1, 3, 64, 64, 43)
    eng = sb.Engine(sb.Model("mini_unet_gn"), math=math)
    eng.precompute(torch.from_numpy(orig).cuda())
    cfg = sb.default_config(dilate_full=1, min_sparse_res=1)
    want = eng.sparse_forward(torch.from_numpy(edited).cuda(), config=cfg).clone()
    flat = torch.from_numpy(np.concatenate([[0.0], edited.ravel()]).astype(np.float32)).cuda()
    xv = flat[1:].view(edited.shape)
    assert xv.data_ptr() % 16 != 0
    assert torch.equal(eng.sparse_forward(xv, config=cfg), want)
