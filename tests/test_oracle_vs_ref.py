"""The C restatement (ORC) against the compiled, unmodified reference (REF),
bit for bit, on seeded random cases modelled on the reference's acceptance
criteria (acceptance.cpp:52-253). Skips when oracle/_ref was not built."""
import numpy as np
import pytest

from paper_2211_02048_b200._capi import default_config


def test_fixtures_and_masks(orc, ref):
    for kind in ["rect1", "rect5", "rect15", "rect35", "blob5", "multi15"]:
        for shape in [(1, 3, 64, 64), (2, 4, 37, 53)]:
            a = orc.make_edit_fixture(kind, *shape, 13)
            b = ref.make_edit_fixture(kind, *shape, 13)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
            m = orc.difference_mask(*a)
            assert np.array_equal(m, ref.difference_mask(*b))


def test_mask_algebra_random(orc, ref):
    rng = np.random.default_rng(8)  # acceptance criterion 8 style
    for _ in range(200):
        h, w = rng.integers(3, 40, 2)
        m = (rng.random((h, w)) < rng.uniform(0, 0.3)).astype(np.uint8)
        r = int(rng.integers(0, 5))
        assert np.array_equal(orc.dilate_mask(m, r), ref.dilate_mask(m, r))
        b, batch = int(rng.integers(1, 9)), int(rng.integers(1, 4))
        ia, ha = orc.mask_to_block_indices(m, b, batch)
        ib, hb = ref.mask_to_block_indices(m, b, batch)
        assert np.array_equal(ia, ib) and ha == hb


def test_ops_random(orc, ref):
    rng = np.random.default_rng(9001)
    for rep in range(40):
        n, c = int(rng.integers(1, 3)), int(rng.integers(1, 7))
        k, s = [(1, 1), (3, 1), (3, 2)][rep % 3]
        h, w = int(rng.integers(6, 30)), int(rng.integers(6, 30))
        x = rng.uniform(-3, 3, (n, c, h, w)).astype(np.float32)
        oh, ow = (h + 2 * ((k - 1) // 2) - k) // s + 1, (w + 2 * ((k - 1) // 2) - k) // s + 1
        b = int(rng.integers(2, 7))
        m = (rng.random((oh, ow)) < 0.2).astype(np.uint8)
        idx, _ = ref.mask_to_block_indices(m, b, n)
        epi = [("ss", rng.uniform(0.5, 1.5, n * c).astype(np.float32), rng.uniform(-0.4, 0.4, n * c).astype(np.float32)),
               ("act", 2 if rep % 2 else 1)]
        ga = orc.gather(x, idx, b, oh, ow, k, s, epi)
        assert np.array_equal(ga.view(np.uint32), ref.gather(x, idx, b, oh, ow, k, s, epi).view(np.uint32))
        wt = rng.uniform(-0.5, 0.5, (5, c, k, k)).astype(np.float32)
        bias = rng.uniform(-0.2, 0.2, 5).astype(np.float32)
        ca = orc.conv_on_blocks(ga, wt, bias, k, s, b)
        assert np.array_equal(ca, ref.conv_on_blocks(ga, wt, bias, k, s, b))
        assert np.array_equal(orc.conv2d(x, wt, bias, k, s), ref.conv2d(x, wt, bias, k, s))
        base = rng.uniform(-1, 1, (n, 5, oh, ow)).astype(np.float32)
        assert np.array_equal(orc.scatter(ca, idx, base), ref.scatter(ca, idx, base))


def test_fused_kernels_random(orc, ref):
    rng = np.random.default_rng(9002)  # acceptance criterion 3 style
    for rep in range(30):
        res, c, n = 2 * int(rng.integers(8, 16)), int(rng.integers(2, 9)), 1 + int(rng.integers(0, 4) == 0)
        base = rng.uniform(-1, 1, (n, c, res, res)).astype(np.float32)
        m = (rng.random((res, res)) < 0.05).astype(np.uint8)
        m = orc.dilate_mask(m, 1)
        im, _ = ref.mask_to_block_indices(m, 6, n)
        is_, _ = ref.mask_to_block_indices(m, 4, n)
        mb = rng.uniform(-1, 1, (len(im), c, 6, 6)).astype(np.float32)
        sb_ = rng.uniform(-1, 1, (len(is_), c, 4, 4)).astype(np.float32)
        epi = [("ss", rng.uniform(0.5, 1.5, c).astype(np.float32), rng.uniform(-0.3, 0.3, c).astype(np.float32)), ("act", 2)]
        a = orc.scatter_gather(mb, im, base, im, 6, res, res, 3, 1, epi)
        b = ref.scatter_gather(mb, im, base, im, 6, res, res, 3, 1, epi)
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
        osc = rng.uniform(-1, 1, base.shape).astype(np.float32)
        for fused in (True, False):
            assert np.array_equal(orc.scatter_with_block_residual(mb, im, sb_, is_, base, osc, fused),
                                  ref.scatter_with_block_residual(mb, im, sb_, is_, base, osc, fused))


@pytest.mark.parametrize("name,fx,n,seed,over", [
    ("mini_unet_gn", "rect5", 1, 17, {}),
    ("mini_unet_gn", "blob5", 2, 5, {"norm_precompute": 0}),
    ("mini_unet_bn", "rect15", 1, 11, {"dilate_full": 3}),
    ("gaugan_stack_in", "multi15", 1, 3, {"block3": 4, "block1": 2}),
    ("ddim_stack_64x32", "rect1", 1, 8, {"dilate_full": 2, "min_sparse_res": 8, "dilate_scale": 0}),
])
def test_executor_bit_exact(orc, ref, name, fx, n, seed, over):
    outs = []
    for impl in (orc, ref):
        m = impl.model(name)
        o, e = impl.make_edit_fixture(fx, n, 3, 64, 64, seed)
        mask = impl.difference_mask(o, e)
        ov = dict(over)
        df = ov.pop("dilate_full", m.required_dilation())
        outs.append(m.sparse_forward(m.precompute(o), e, mask, default_config(dilate_full=df, **ov)))
    assert np.array_equal(outs[0][0].view(np.uint32), outs[1][0].view(np.uint32))
    assert np.array_equal(outs[0][1], outs[1][1])
