"""BASELINE config 3 through the engine: the GauGAN SPADE generator.

The reference has no SPADE layer, so the checker is the float64
restatement in oracle/spade.py (parity unpinned against the reference itself;
its elementwise pieces are pinned bit for bit in tests/test_spade_ops.py).
`gaugan_spade_mini` is the config-3 generator at 64x128 with nf 8 / nhidden 16 /
8 labels: the same layer sequence (resize, conv, 7 SPADE ResBlocks with five 2x
upsamplings, LeakyReLU, conv_img) at sizes the oracle runs in seconds.

* dense_forward, FP32_FMA and EXACT: normalised max error <= 1e-4 against the
  oracle; TF32 / F16: <= 1e-2 (11-bit significands).
* sparse_forward with a dilation that covers the image equals
  dense_forward(reused_stats=True) (the same cached instance-norm statistics)
  bit for bit in EXACT; with every SPADE block below min_sparse_res it equals
  the fresh-statistics dense_forward bit for bit.
* An empty edit returns the cached output bit for bit; a 1.2 % relabel at the
  model's required dilation equals the cached-statistics dense pass (EXACT,
  bit for bit) and leaves pixels beyond the dilated edit untouched.
"""
import numpy as np
import pytest
import torch

import paper_2211_02048_b200 as sb

pytestmark = pytest.mark.gpu

NAME = "gaugan_spade_mini"


def nerr(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-30))


@pytest.fixture(scope="module")
def fx():
    from oracle import spade as osp

    m = sb.Model(NAME)
    _, label_nc, h, w = (1,) + m.in_shape
    orig, edited = sb.make_seg_fixture(1, label_nc, h, w, 11)
    return dict(m=m, orig=orig, edited=edited, want_o=osp.forward(m.desc, orig.numpy()),
                want_e=osp.forward(m.desc, edited.numpy()))


@pytest.mark.parametrize("math,tol", [(sb.MATH_FP32_FMA, 1e-4), (sb.MATH_EXACT, 1e-4),
                                      (sb.MATH_TF32, 1e-2), (sb.MATH_F16, 1e-2)])
def test_dense_matches_oracle(fx, math, tol):
    eng = sb.Engine(fx["m"], 1, math)
    got = eng.dense_forward(fx["edited"].cuda()).cpu().numpy()
    e = nerr(got, fx["want_e"])
    print(f"math {math}: normalised max error {e:.3g}")
    assert np.isfinite(got).all() and e <= tol


@pytest.mark.parametrize("math", [sb.MATH_EXACT, sb.MATH_F16])
def test_precompute_caches_the_dense_output(fx, math):
    eng = sb.Engine(fx["m"], 1, math)
    eng.precompute(fx["orig"].cuda())
    out = eng.sparse_forward(fx["orig"].cuda(), config=sb.default_config())  # empty edit
    want = eng.dense_forward(fx["orig"].cuda())
    assert torch.equal(out, want)
    assert nerr(want.cpu().numpy(), fx["want_o"]) <= (1e-4 if math == sb.MATH_EXACT else 1e-2)


@pytest.mark.parametrize("math", [sb.MATH_EXACT, sb.MATH_F16])
def test_full_dilation_equals_dense_with_cached_stats(fx, math):
    eng = sb.Engine(fx["m"], 1, math)
    eng.precompute(fx["orig"].cuda())
    x = fx["edited"].cuda()
    cfg = sb.default_config(dilate_full=10**4, dilate_scale=1, min_sparse_res=1)
    got = eng.sparse_forward(x, config=cfg).clone()
    want = eng.dense_forward(x, reused_stats=True)
    if math == sb.MATH_EXACT:
        assert torch.equal(got, want)
    else:
        assert nerr(got.cpu().numpy(), want.cpu().numpy()) <= 1e-2
    # twice in a row (working buffers restored between calls)
    assert torch.equal(eng.sparse_forward(x, config=cfg), got)


def test_dense_fallback_blocks_use_fresh_stats(fx):
    eng = sb.Engine(fx["m"], 1, sb.MATH_EXACT)
    eng.precompute(fx["orig"].cuda())
    x = fx["edited"].cuda()
    got = eng.sparse_forward(x, config=sb.default_config(min_sparse_res=10**4))
    assert torch.equal(got, eng.dense_forward(x))


@pytest.mark.parametrize("math", [sb.MATH_EXACT, sb.MATH_F16])
def test_sparse_edit_at_required_dilation(fx, math):
    """At the model's required dilation every pixel the edit reaches is
    recomputed, so the sparse pass equals the dense pass that reuses the
    cached instance-norm statistics (SIGE's approximation: statistics of the
    original, graph.cpp:745-750); pixels beyond the dilated edit keep the
    cached output bit for bit. The distance to the fresh-statistics dense pass
    over the edit is the approximation itself and is printed."""
    eng = sb.Engine(fx["m"], 1, math)
    eng.precompute(fx["orig"].cuda())
    x = fx["edited"].cuda()
    r = fx["m"].required_dilation()
    cfg = sb.default_config(dilate_full=r, dilate_scale=1, min_sparse_res=1)
    got = eng.sparse_forward(x, config=cfg).cpu().numpy()
    want = eng.dense_forward(x, reused_stats=True).cpu().numpy()
    e = nerr(got, want)
    print(f"math {math}: required dilation {r}: vs dense with cached stats {e:.3g}, "
          f"vs fresh-statistics dense over the edit {nerr(got, fx['want_e']):.3g}")
    if math == sb.MATH_EXACT:
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    else:
        assert e <= 1e-2
    cached = eng.sparse_forward(fx["orig"].cuda(), config=cfg).cpu().numpy()
    diff = np.abs(fx["orig"].numpy() - fx["edited"].numpy()).max(axis=(0, 1)) > 0
    ys, xs = np.nonzero(diff)
    far = np.ones(diff.shape, bool)
    far[max(ys.min() - r, 0):ys.max() + r + 1, max(xs.min() - r, 0):xs.max() + r + 1] = False
    if far.any():
        assert np.array_equal(got[..., far].view(np.uint32), cached[..., far].view(np.uint32))


def test_sparse_edit_default_config(fx):
    """The default RunConfig (dilate_full 1): finite, and the distance to the
    dense pass over the edit printed (quality is the caller's dilation choice)."""
    eng = sb.Engine(fx["m"], 1, sb.MATH_F16)
    eng.precompute(fx["orig"].cuda())
    got = eng.sparse_forward(fx["edited"].cuda(), config=sb.default_config(min_sparse_res=1)).cpu().numpy()
    print(f"default config: vs fresh-statistics dense over the edit {nerr(got, fx['want_e']):.3g}")
    assert np.isfinite(got).all()


def test_output_coverage_rejects_spade(fx):
    eng = sb.Engine(fx["m"], 1, sb.MATH_F16)
    eng.precompute(fx["orig"].cuda())
    with pytest.raises(Exception):
        eng.output_coverage(fx["edited"].cuda())


def test_grouped_requests_equal_separate_engines(fx):
    """Two SPADE requests (different label maps and edits) through one grouped
    engine give each request's own single-engine result bit for bit (EXACT),
    at the required dilation and at the default one."""
    m = fx["m"]
    _, label_nc, h, w = (1,) + m.in_shape
    pairs = [sb.make_seg_fixture(1, label_nc, h, w, s) for s in (11, 12)]
    r = m.required_dilation()
    for cfg in (sb.default_config(dilate_full=r, dilate_scale=1, min_sparse_res=1), sb.default_config(min_sparse_res=1)):
        singles = []
        for o, e in pairs:
            eng = sb.Engine(m, 1, sb.MATH_EXACT)
            eng.precompute(o.cuda())
            singles.append(eng.sparse_forward(e.cuda(), config=cfg).cpu())
        geng = sb.Engine(m, 2, sb.MATH_EXACT)
        geng.precompute(torch.cat([o for o, _ in pairs]).cuda())
        got = geng.sparse_forward_grouped(torch.cat([e for _, e in pairs]).cuda(), config=cfg).cpu()
        for i in range(2):
            assert torch.equal(got[i:i + 1], singles[i])


def test_host_buffer_path_and_graph_replay(fx):
    """The e2e entry point (host buffers, sige_engine_sparse_forward_host) and
    repeated graph-replayed calls give the device call's bits (F16)."""
    eng = sb.Engine(fx["m"], 1, sb.MATH_F16)
    eng.precompute(fx["orig"].cuda())
    cfg = sb.default_config(min_sparse_res=1)
    want = eng.sparse_forward(fx["edited"].cuda(), config=cfg).cpu()
    for _ in range(3):  # direct run, capture, replays
        assert torch.equal(eng.sparse_forward(fx["edited"].cuda(), config=cfg).cpu(), want)
    got = eng.sparse_forward_host(fx["edited"].pin_memory(), config=cfg)
    assert torch.equal(got, want)
