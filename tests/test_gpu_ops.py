"""GPU parity of the op-level C-ABI kernels against the oracle (bit-exact).

Cases follow the reference's own unit tests (proj/tests/test_kernels.cpp,
test_mask.cpp) and acceptance criterion 3 (acceptance.cpp:182-253): frozen
windows, fringe clipping, batch OR, epilogue-on-copied-pixels-only, fused ==
unfused, plus seeded random sweeps. Every comparison is np.array_equal on the
raw float32 bits (NaN-free inputs), i.e. bit-exact."""
import numpy as np
import pytest
import torch

import paper_2211_02048_b200 as sb

pytestmark = pytest.mark.gpu


def cu(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def bits_equal(a, b):
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


def rand_epi_np(rng, c, n=1, silu=True, per_sample=False):
    k = n * c if per_sample else c
    sc = rng.uniform(0.5, 1.5, k).astype(np.float32)
    sh = rng.uniform(-0.4, 0.4, k).astype(np.float32)
    steps = [("ss", sc, sh)]
    if silu:
        steps.append(("act", sb.ACT_SILU))
    return steps


def to_dev_epi(steps):
    e = sb.Epilogue()
    for st in steps:
        if st[0] == "ss":
            e.add_scale_shift(torch.from_numpy(st[1]), torch.from_numpy(st[2]))
        else:
            e.add_activation(st[1])
    return e


# ----------------------------------------------------------- masks -------

def test_difference_mask_threshold_strict_and_batch_or(orc):
    # test_mask.cpp:33-51
    o = np.zeros((1, 2, 3, 3), np.float32)
    e = o.copy()
    e[0, 1, 2, 2] = 0.5
    e[0, 0, 0, 0] = 1e-3
    m = host(sb.compute_difference_mask(cu(o), cu(e), 1e-3))
    assert m.sum() == 1 and m[2, 2] == 1 and m[0, 0] == 0
    o = np.zeros((2, 1, 2, 2), np.float32)
    e = o.copy()
    e[0, 0, 0, 0] = 1
    e[1, 0, 1, 1] = 1
    m = host(sb.compute_difference_mask(cu(o), cu(e), 0.1))
    assert m[0, 0] == 1 and m[1, 1] == 1 and m.sum() == 2


@pytest.mark.parametrize("kind,n,c,h,w,seed", [("rect1", 1, 64, 256, 256, 7), ("blob5", 2, 3, 64, 48, 3),
                                                ("multi15", 1, 5, 37, 53, 9), ("rect35", 3, 2, 31, 17, 4)])
def test_difference_mask_matches_oracle(orc, kind, n, c, h, w, seed):
    o, e = orc.make_edit_fixture(kind, n, c, h, w, seed)
    want = orc.difference_mask(o, e, 1e-3)
    got = host(sb.compute_difference_mask(cu(o), cu(e), 1e-3))
    assert np.array_equal(got, want)
    # inputs at a one-float offset (off 16-byte alignment): the scalar path, same mask
    ov = cu(np.concatenate([[0.0], o.ravel()]).astype(np.float32))[1:].view(o.shape)
    ev = cu(np.concatenate([[0.0], e.ravel()]).astype(np.float32))[1:].view(e.shape)
    assert np.array_equal(host(sb.compute_difference_mask(ov, ev, 1e-3)), want)


def test_difference_mask_golden_hash(orc):
    o, e = orc.make_edit_fixture("rect1", 1, 64, 256, 256, 7)
    m = host(sb.compute_difference_mask(cu(o), cu(e), 1e-3))
    assert orc.fnv1a64(m) == 0x938A3A322907C793
    assert int(m.sum()) == 784


def test_dilate_and_downsample_match_oracle(orc):
    rng = np.random.default_rng(11)
    for rep in range(30):
        h, w = rng.integers(4, 40, 2)
        m = (rng.random((h, w)) < 0.1).astype(np.uint8)
        r = int(rng.integers(0, 4))
        assert np.array_equal(host(sb.dilate_mask(cu(m), r)), orc.dilate_mask(m, r))
    m = (rng.random((48, 64)) < 0.05).astype(np.uint8)
    for oh, ow in [(24, 32), (12, 16), (48, 8), (1, 1)]:
        assert np.array_equal(host(sb.downsample_mask(cu(m), oh, ow)), orc.downsample_mask(m, oh, ow))
    with pytest.raises(sb.ConfigError, match="non-integer scale factor"):
        sb.downsample_mask(cu(m), 7, 7)


def test_block_indices_match_oracle_and_golden(orc):
    rng = np.random.default_rng(41)
    for rep in range(40):
        h, w = rng.integers(5, 70, 2)
        b = int(rng.integers(1, 9))
        batch = int(rng.integers(1, 4))
        m = (rng.random((h, w)) < rng.uniform(0.0, 0.2)).astype(np.uint8)
        want, _ = orc.mask_to_block_indices(m, b, batch)
        got = host(sb.mask_to_block_indices(cu(m), b, batch))
        assert np.array_equal(got, want), (h, w, b, batch)
    # golden: 36 tiles at b=6 after two radius-1 dilations
    o, e = orc.make_edit_fixture("rect1", 1, 64, 256, 256, 7)
    m = sb.compute_difference_mask(cu(o), cu(e), 1e-3)
    d = sb.dilate_mask(sb.dilate_mask(m, 1), 1)
    idx = host(sb.mask_to_block_indices(d, 6, 1))
    assert len(idx) == 36
    assert orc.lib.orc_index_set_hash(idx.ctypes.data, 36, 6, 256, 256) == 0xCCBB614A2A613105


# ---------------------------------------------------------- blocks -------

def test_gather_frozen_windows():
    # test_kernels.cpp:61-92
    x = np.arange(16, dtype=np.float32).reshape(1, 1, 4, 4)
    g = host(sb.gather(cu(x), cu(np.array([[0, 0, 0]], np.int32)), 2, 3, 1))
    assert g.ravel().tolist() == [0, 0, 0, 0, 0, 0, 1, 2, 0, 4, 5, 6, 0, 8, 9, 10]
    g = host(sb.gather(cu(x), cu(np.array([[0, 2, 2]], np.int32)), 2, 3, 1))
    assert g.ravel().tolist() == [5, 6, 7, 0, 9, 10, 11, 0, 13, 14, 15, 0, 0, 0, 0, 0]
    g = host(sb.gather(cu(x), cu(np.array([[0, 2, 2]], np.int32)), 2, 1, 1))
    assert g.ravel().tolist() == [10, 11, 14, 15]
    x8 = np.arange(64, dtype=np.float32).reshape(1, 1, 8, 8)
    g = host(sb.gather(cu(x8), cu(np.array([[0, 2, 2]], np.int32)), 2, 3, 2))
    assert g.shape[-1] == 5 and g[0, 0, 0, 0] == x8[0, 0, 3, 3] and g[0, 0, 4, 4] == x8[0, 0, 7, 7]


def test_gather_errors_like_reference():
    x = cu(np.zeros((1, 1, 8, 8), np.float32))
    i = cu(np.zeros((1, 3), np.int32))
    with pytest.raises(sb.ConfigError, match="gather: kernel size must be 1 or 3"):
        sb.gather(x, i, 2, 5, 1)
    with pytest.raises(sb.ConfigError, match="gather: stride must be 1 or 2"):
        sb.gather(x, i, 2, 3, 3)
    with pytest.raises(sb.ConfigError, match="gather: index set lives at"):
        sb.gather(x, i, 2, 3, 1, idx_hw=(4, 4))


@pytest.mark.parametrize("k,s", [(3, 1), (1, 1), (3, 2)])
def test_gather_with_epilogue_matches_oracle(orc, k, s):
    rng = np.random.default_rng(71 + k + s)
    for rep in range(6):
        n, c = int(rng.integers(1, 3)), int(rng.integers(1, 9))
        h, w = int(rng.integers(6, 40)), int(rng.integers(6, 40))
        x = rng.uniform(-3, 3, (n, c, h, w)).astype(np.float32)
        oh, ow = (h + 2 * ((k - 1) // 2) - k) // s + 1, (w + 2 * ((k - 1) // 2) - k) // s + 1
        b = int(rng.integers(2, 8))
        m = (rng.random((oh, ow)) < 0.15).astype(np.uint8)
        idx, _ = orc.mask_to_block_indices(m, b, n)
        epi = rand_epi_np(rng, c, n, silu=rep % 2 == 0, per_sample=rep % 3 == 0)
        want = orc.gather(x, idx, b, oh, ow, k, s, epi)
        got = host(sb.gather(cu(x), cu(idx), b, k, s, to_dev_epi(epi)))
        assert bits_equal(got, want)


@pytest.mark.parametrize("k,b,w,offset", [(3, 6, 64, 0), (1, 8, 40, 0), (3, 6, 48, 1)])
def test_gather_wide_rows_match_oracle(orc, k, b, w, offset):
    """8-wide window rows with w % 8 == 0 take the 256-bit-load kernel (every
    phase 0-7 of the window start, fringe windows at both image edges); a base
    pointer off 32-byte alignment (offset 1) takes the 16-byte-load kernel."""
    rng = np.random.default_rng(w + b + offset)
    n, c, h = 2, 5, 29
    flat = rng.uniform(-3, 3, n * c * h * w + offset).astype(np.float32)
    x = flat[offset:].reshape(n, c, h, w)
    m = (rng.random((h, w)) < 0.3).astype(np.uint8)
    m[:, 0] = m[:, -1] = m[0, :] = m[-1, :] = 1
    idx, _ = orc.mask_to_block_indices(m, b, n)
    for epi in ([], rand_epi_np(rng, c, n, silu=True, per_sample=True)):
        want = orc.gather(np.ascontiguousarray(x), idx, b, h, w, k, 1, epi)
        xd = cu(flat)[offset:].view(n, c, h, w)
        got = host(sb.gather(xd, cu(idx), b, k, 1, to_dev_epi(epi)))
        assert bits_equal(got, want)


def test_silu_relu_epilogue_zero_fill_untouched(orc):
    # test_kernels.cpp:94-112
    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, (2, 3, 9, 9)).astype(np.float32)
    idx = np.array([[0, 0, 0], [0, 3, 3], [1, 6, 6]], np.int32)
    epi = rand_epi_np(rng, 3)
    got = host(sb.gather(cu(x), cu(idx), 3, 3, 1, to_dev_epi(epi)))
    assert got[0, 0, 0, 0] == 0.0
    assert bits_equal(got, orc.gather(x, idx, 3, 9, 9, 3, 1, epi))
    epi = [("act", sb.ACT_RELU)]
    x[0, 0, 1, 1] = -0.0
    assert bits_equal(host(sb.gather(cu(x), cu(idx), 3, 3, 1, to_dev_epi(epi))), orc.gather(x, idx, 3, 9, 9, 3, 1, epi))


def test_scatter_family_matches_oracle(orc):
    rng = np.random.default_rng(81)
    for rep in range(12):
        n, c, h, w = int(rng.integers(1, 3)), int(rng.integers(1, 6)), int(rng.integers(5, 30)), int(rng.integers(5, 30))
        b = int(rng.integers(1, 7))
        m = (rng.random((h, w)) < 0.1).astype(np.uint8)
        idx, _ = orc.mask_to_block_indices(m, b, n)
        blocks = rng.uniform(-1, 1, (len(idx), c, b, b)).astype(np.float32)
        base = rng.uniform(-1, 1, (n, c, h, w)).astype(np.float32)
        assert bits_equal(host(sb.scatter(cu(blocks), cu(idx), cu(base))), orc.scatter(blocks, idx, base))
        tb = cu(base)
        sb.scatter_add_inplace(cu(blocks), cu(idx), tb)
        assert bits_equal(host(tb), orc.scatter_add_inplace(blocks, idx, base.copy()))


@pytest.mark.parametrize("n,c,hw,b,dens", [
    (2, 256, 128, 4, 1.0),   # ~1400 (tiles x channels) items: the persistent kernel alternates its two buffers
    (2, 96, 70, 6, 0.3),     # ragged chunks and channel slices, fringe tiles
    (1, 2, 170, 80, 1.0),    # 80x80 blocks exceed a staging buffer: the single-buffered kernel
])
def test_scatter_pipeline_sizes_match_oracle(orc, n, c, hw, b, dens):
    rng = np.random.default_rng(hw + b)
    m = (rng.random((hw, hw)) < dens).astype(np.uint8)
    idx, _ = orc.mask_to_block_indices(m, b, n)
    blocks = rng.uniform(-1, 1, (len(idx), c, b, b)).astype(np.float32)
    base = rng.uniform(-1, 1, (n, c, hw, hw)).astype(np.float32)
    assert bits_equal(host(sb.scatter(cu(blocks), cu(idx), cu(base))), orc.scatter(blocks, idx, base))
    tb = cu(base)
    sb.scatter_add_inplace(cu(blocks), cu(idx), tb)
    assert bits_equal(host(tb), orc.scatter_add_inplace(blocks, idx, base.copy()))


def test_scatter_misaligned_tensors_match_oracle(orc):
    """Block stacks and bases that start off 16- / 8-byte alignment (views at a
    one-float offset) take the scalar paths and give the same bits."""
    rng = np.random.default_rng(5)
    n, c, hw, b = 2, 12, 40, 6
    m = (rng.random((hw, hw)) < 0.4).astype(np.uint8)
    idx, _ = orc.mask_to_block_indices(m, b, n)
    blocks = rng.uniform(-1, 1, (len(idx), c, b, b)).astype(np.float32)
    base = rng.uniform(-1, 1, (n, c, hw, hw)).astype(np.float32)
    bl = cu(np.concatenate([[0.0], blocks.ravel()]).astype(np.float32))[1:].view(blocks.shape)
    tb = cu(np.concatenate([[0.0], base.ravel()]).astype(np.float32))[1:].view(base.shape)
    sb.scatter_inplace(bl, cu(idx), tb)
    assert bits_equal(host(tb), orc.scatter(blocks, idx, base))
    tb2 = cu(np.concatenate([[0.0], base.ravel()]).astype(np.float32))[1:].view(base.shape)
    sb.scatter_add_inplace(bl, cu(idx), tb2)
    assert bits_equal(host(tb2), orc.scatter_add_inplace(blocks, idx, base.copy()))


def test_scatter_clips_fringe_tiles():
    # test_kernels.cpp:136-145
    base = cu(np.zeros((1, 1, 5, 5), np.float32))
    sb.scatter_inplace(cu(np.full((1, 1, 4, 4), 3.0, np.float32)), cu(np.array([[0, 4, 4]], np.int32)), base)
    out = host(base)
    assert out[0, 0, 4, 4] == 3.0 and (out != 0).sum() == 1


def test_scatter_map_and_scatter_gather_match_oracle(orc):
    rng = np.random.default_rng(93)
    for rep in range(10):
        h, c, n = 12 + rep, 3, 2
        pm = np.zeros((h, h), np.uint8)
        for _ in range(3):
            pm[rng.integers(0, h), rng.integers(0, h)] = 1
        prod, _ = orc.mask_to_block_indices(pm, 4, n)
        blocks = rng.uniform(-1, 1, (len(prod), c, 4, 4)).astype(np.float32)
        base = rng.uniform(-1, 1, (n, c, h, h)).astype(np.float32)
        cm = np.zeros((h, h), np.uint8)
        cm[0, 0] = 1
        cm[rng.integers(0, h), rng.integers(0, h)] = 1
        cons, _ = orc.mask_to_block_indices(cm, 4, n)
        want_map, want_bps = orc.build_scatter_map(prod, 4, h, h)
        got_map, got_bps = sb.build_scatter_map(cu(prod), 4, h, h)
        assert got_bps == want_bps
        assert np.array_equal(host(got_map).view(np.uint8).ravel(), want_map.view(np.uint8).ravel())
        epi = rand_epi_np(rng, c) if rep % 2 == 0 else []
        k = 1 if rep % 3 == 0 else 3
        want = orc.scatter_gather(blocks, prod, base, cons, 4, h, h, k, 1, epi)
        got = host(sb.scatter_gather(cu(blocks), cu(base), (got_map, got_bps), cu(cons), 4, k, 1, to_dev_epi(epi)))
        assert bits_equal(got, want)


def test_scatter_map_rejects_batch_pattern_mismatch():
    idx = cu(np.array([[0, 0, 0], [1, 4, 4]], np.int32))
    with pytest.raises(sb.ConfigError, match="tile pattern differs across batch"):
        sb.build_scatter_map(idx, 4, 8, 8)


def test_block_residual_fused_equals_unfused_and_oracle(orc):
    # test_kernels.cpp:250-286
    rng = np.random.default_rng(103)
    for rep in range(8):
        h, c, n = 16, 4, 1 + rep % 2
        s_ = rng.uniform(-1, 1, (n, c, h, h)).astype(np.float32)
        osc = rng.uniform(-1, 1, (n, c, h, h)).astype(np.float32)
        mm = np.zeros((h, h), np.uint8)
        smk = np.zeros((h, h), np.uint8)
        for _ in range(3):
            mm[rng.integers(0, h), rng.integers(0, h)] = 1
            smk[rng.integers(0, h), rng.integers(0, h)] = 1
        mi, _ = orc.mask_to_block_indices(orc.dilate_mask(mm, 1), 6, n)
        si, _ = orc.mask_to_block_indices(smk, 4, n)
        mb = rng.uniform(-1, 1, (len(mi), c, 6, 6)).astype(np.float32)
        pb = rng.uniform(-1, 1, (len(si), c, 4, 4)).astype(np.float32)
        want = orc.scatter_with_block_residual(mb, mi, pb, si, s_, osc, True)
        assert bits_equal(want, orc.scatter_with_block_residual(mb, mi, pb, si, s_, osc, False))
        f = host(sb.scatter_with_block_residual(cu(mb), cu(mi), cu(pb), cu(si), cu(s_), cu(osc)))
        u = host(sb.scatter_with_block_residual_unfused(cu(mb), cu(mi), cu(pb), cu(si), cu(s_), cu(osc)))
        assert bits_equal(f, want) and bits_equal(u, want)


def test_block_arithmetic_and_epilogue_on_blocks(orc):
    rng = np.random.default_rng(139)
    a = np.arange(8, dtype=np.float32).reshape(2, 1, 2, 2)
    b = np.full_like(a, 10.0)
    assert host(sb.add_blocks(cu(a), cu(b))).ravel()[3] == 13.0
    assert host(sb.subtract_blocks(cu(a), cu(b))).ravel()[3] == -7.0
    idx = np.array([[0, 0, 0], [1, 4, 4]], np.int32)
    s = rng.uniform(-1, 1, (2, 3, 4, 4)).astype(np.float32)
    epi = rand_epi_np(rng, 3, n=2, per_sample=True)
    t = cu(s)
    sb.apply_epilogue_on_blocks(t, cu(idx), to_dev_epi(epi))
    assert bits_equal(host(t), orc.apply_epilogue_on_blocks(s, idx, 8, 8, epi))


@pytest.mark.parametrize("math", [sb.MATH_EXACT, sb.MATH_FP32_FMA])
def test_conv_on_blocks_and_conv2d(orc, math):
    # test_kernels.cpp:288-351: conv_on_blocks over a whole-canvas tile == conv2d
    rng = np.random.default_rng(113)
    for k in (1, 3):
        for s in (1, 2):
            x = rng.uniform(-1, 1, (2, 3, 8, 8)).astype(np.float32)
            wt = rng.uniform(-0.5, 0.5, (5, 3, k, k)).astype(np.float32)
            bias = rng.uniform(-0.2, 0.2, 5).astype(np.float32)
            oh = (8 + 2 * ((k - 1) // 2) - k) // s + 1
            idx = np.array([[0, 0, 0], [1, 0, 0]], np.int32)
            g = orc.gather(x, idx, oh, oh, oh, k, s)
            want_blocks = orc.conv_on_blocks(g, wt, bias, k, s, oh)
            want_dense = orc.conv2d(x, wt, bias, k, s)
            got_blocks = host(sb.conv_on_blocks(cu(g), cu(wt), cu(bias), s, oh, math=math))
            got_dense = host(sb.conv2d(cu(x), cu(wt), cu(bias), s, math=math))
            if math == sb.MATH_EXACT:
                assert bits_equal(got_blocks, want_blocks) and bits_equal(got_dense, want_dense)
                assert bits_equal(want_blocks.transpose(1, 0, 2, 3).reshape(5, 2, oh, oh), want_dense.transpose(1, 0, 2, 3))
            else:
                assert np.abs(got_dense - want_dense).max() <= 1e-4 * np.abs(want_dense).max()


def test_conv_on_blocks_geometry_error():
    with pytest.raises(sb.ConfigError, match="conv_on_blocks: window 8 with k=3 s=1 yields 6, expected block 5"):
        sb.conv_on_blocks(cu(np.zeros((1, 2, 8, 8), np.float32)), cu(np.zeros((2, 2, 3, 3), np.float32)), None, 1, 5)


@pytest.mark.parametrize("b", [1, 6, 13])
def test_gather_scatter_long_runs_chunk_and_slice_edges(orc, b):
    # Dense masks: row runs longer than one CTA chunk (256 columns), channel
    # counts that split into several slices with a ragged last one, tiles at
    # the fringe. Exercises the (channel, row, tile, column) walk of
    # k_gather / k_scatter against the oracle bit for bit.
    rng = np.random.default_rng(1000 + b)
    for k, s in [(3, 1), (3, 2), (1, 1)]:
        n, c, h, w = 2, 37, 61, 301
        x = rng.uniform(-2, 2, (n, c, h, w)).astype(np.float32)
        oh, ow = (h + 2 * ((k - 1) // 2) - k) // s + 1, (w + 2 * ((k - 1) // 2) - k) // s + 1
        m = (rng.random((oh, ow)) < 0.6).astype(np.uint8)
        idx, _ = orc.mask_to_block_indices(m, b, n)
        epi = rand_epi_np(rng, c, n, silu=True, per_sample=True)
        want = orc.gather(x, idx, b, oh, ow, k, s, epi)
        assert bits_equal(host(sb.gather(cu(x), cu(idx), b, k, s, to_dev_epi(epi))), want)
    m = (rng.random((h, w)) < 0.6).astype(np.uint8)
    idx, _ = orc.mask_to_block_indices(m, b, n)
    blocks = rng.uniform(-1, 1, (len(idx), c, b, b)).astype(np.float32)
    base = rng.uniform(-1, 1, (n, c, h, w)).astype(np.float32)
    assert bits_equal(host(sb.scatter(cu(blocks), cu(idx), cu(base))), orc.scatter(blocks, idx, base))
    tb = cu(base)
    sb.scatter_add_inplace(cu(blocks), cu(idx), tb)
    assert bits_equal(host(tb), orc.scatter_add_inplace(blocks, idx, base.copy()))


@pytest.mark.parametrize("math", [sb.MATH_TF32, sb.MATH_F16], ids=["tf32", "f16"])
def test_conv_tensor_core_op_level(orc, math):
    """conv_on_blocks / conv2d (kernels.cpp:391-421, conv.cpp:83-102) on the
    tcgen05 path: integer data is exact in any summation order (bit-exact vs the
    oracle), real data within the north-star 1e-2 normalised max error."""
    rng = np.random.default_rng(151)
    for k, s, cin, cout, b, hw in [(3, 1, 64, 96, 6, 20), (1, 1, 128, 64, 4, 16), (3, 2, 32, 40, 6, 26),
                                  (3, 1, 3, 16, 6, 14)]:
        oh = (hw + 2 * ((k - 1) // 2) - k) // s + 1
        for integer in (True, False):
            if integer:
                x = rng.integers(-2, 3, (2, cin, hw, hw)).astype(np.float32)
                wt = rng.integers(-2, 3, (cout, cin, k, k)).astype(np.float32)
                bias = rng.integers(-3, 4, cout).astype(np.float32)
            else:
                x = rng.uniform(-1, 1, (2, cin, hw, hw)).astype(np.float32)
                wt = rng.uniform(-0.2, 0.2, (cout, cin, k, k)).astype(np.float32)
                bias = rng.uniform(-0.1, 0.1, cout).astype(np.float32)
            m = (rng.random((oh, oh)) < 0.3).astype(np.uint8)
            idx, _ = orc.mask_to_block_indices(m, b, 2)
            g = orc.gather(x, idx, b, oh, oh, k, s)
            want_b = orc.conv_on_blocks(g, wt, bias, k, s, b)
            want_d = orc.conv2d(x, wt, bias, k, s)
            got_b = host(sb.conv_on_blocks(cu(g), cu(wt), cu(bias), s, b, math=math))
            got_d = host(sb.conv2d(cu(x), cu(wt), cu(bias), s, math=math))
            if integer:
                assert bits_equal(got_b, want_b) and bits_equal(got_d, want_d), (k, s, cin, cout)
            else:
                for got, want in ((got_b, want_b), (got_d, want_d)):
                    assert np.abs(got - want).max() <= 1e-2 * np.abs(want).max(), (k, s, cin, cout)


def test_conv_rejects_unknown_math_mode():
    g = cu(np.zeros((1, 2, 8, 8), np.float32))
    w = cu(np.zeros((2, 2, 3, 3), np.float32))
    with pytest.raises(sb.ConfigError, match="conv_on_blocks: unknown math mode 7"):
        sb.conv_on_blocks(g, w, None, 1, 6, math=7)
    with pytest.raises(sb.ConfigError, match="conv2d: unknown math mode -1"):
        sb.conv2d(g, w, None, math=-1)


def test_scatter_rejects_incompatible_indices_like_reference():
    """require_scatter_compatible (kernels.cpp:18-35) / require_join_compatible
    (:276-287) messages; the kernels themselves never write outside the tensor."""
    base = cu(np.zeros((1, 2, 12, 12), np.float32))
    blocks = cu(np.ones((2, 2, 6, 6), np.float32))
    bad_n = cu(np.array([[0, 0, 0], [1, 6, 6]], np.int32))
    with pytest.raises(sb.ConfigError, match="scatter: block sample out of range"):
        sb.scatter_inplace(blocks, bad_n, base)
    with pytest.raises(sb.ConfigError, match="scatter_add: block sample out of range"):
        sb.scatter_add_inplace(blocks, bad_n, base)
    with pytest.raises(sb.ConfigError, match="scatter: channel mismatch"):
        sb.scatter(cu(np.ones((2, 3, 6, 6), np.float32)), cu(np.zeros((2, 3), np.int32)), base)
    with pytest.raises(sb.ConfigError, match=r"scatter: index resolution 6x6 does not match tensor \(1, 2, 12, 12\)"):
        sb.scatter(blocks, cu(np.zeros((2, 3), np.int32)), base, idx_hw=(6, 6))
    with pytest.raises(sb.ConfigError, match=r"block_residual\(main\): block sample out of range"):
        sb.scatter_with_block_residual(blocks, bad_n, blocks, cu(np.zeros((2, 3), np.int32)), base, base)
    # straight through the ABI (no wrapper checks): the out-of-range block is skipped
    t = cu(np.zeros((1, 2, 12, 12), np.float32))
    assert sb._lib().sige_scatter_inplace(blocks.data_ptr(), 2, 2, 6, bad_n.data_ptr(), t.data_ptr(), 1, 2, 12, 12,
                                          torch.cuda.current_stream().cuda_stream) == 0
    got = host(t)
    assert got[0, :, :6, :6].min() == 1.0 and got[0, :, 6:, 6:].max() == 0.0


@pytest.mark.parametrize("win_b,n,c,h,w", [(6, 2, 70, 36, 44), (2, 1, 5, 16, 12), (6, 1, 33, 20, 20)])
def test_gather_tma_boxes_match_oracle(orc, win_b, n, c, h, w):
    """Gather at the shapes of the (measured slower and removed) TMA-box
    variant — 8x8 / 4x4 windows, W % 4 == 0: ragged channel slices, tiles at
    every fringe (negative window origins zero-filled), per-sample epilogue
    with SiLU on in-canvas cells only — bit-exact vs the oracle, with and
    without the epilogue."""
    rng = np.random.default_rng(win_b * 1000 + c)
    x = rng.uniform(-3, 3, (n, c, h, w)).astype(np.float32)
    b = win_b
    m = np.zeros((h, w), np.uint8)
    m[0, 0] = m[-1, -1] = m[0, -1] = m[-1, 0] = 1
    m[h // 2, w // 2] = 1
    m |= (rng.random((h, w)) < 0.05).astype(np.uint8)
    idx, _ = orc.mask_to_block_indices(m, b, n)
    for epi in ([], rand_epi_np(rng, c, n, silu=True, per_sample=True)):
        want = orc.gather(x, idx, b, h, w, 3, 1, epi)
        got = host(sb.gather(cu(x), cu(idx), b, 3, 1, to_dev_epi(epi) if epi else None))
        assert bits_equal(got, want)
