"""SPADE ops for BASELINE config 3 (GauGAN SPADE ResBlocks at 256x512).

The reference has no SPADE API (per-pixel gamma/beta exceed its
per-channel Epilogue, and it has no label-map resample), so parity here is
anchored on the C restatement (orc_gather_spade / orc_resize_nearest), which is
itself checked against an independent numpy statement of the same arithmetic
(float32, one rounding per operation) and against the reference's own gather()
when gamma = beta = 0 (then the modulation is the identity).
CPU tests pin the oracle; GPU tests call the CUDA kernels through the C ABI
and compare bit for bit."""
import numpy as np
import pytest
import torch

import paper_2211_02048_b200 as sb


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def bits_equal(a, b):
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


def to_dev_epi(steps):
    e = sb.Epilogue()
    for st in steps:
        if st[0] == "ss":
            e.add_scale_shift(torch.from_numpy(st[1]), torch.from_numpy(st[2]))
        else:
            e.add_activation(st[1])
    return e


def _np_gather_spade(x, gamma, beta, idx, b, k, s, sc, sh, act):
    n, c, h, w = x.shape
    win, pad = s * b + k - s, (k - 1) // 2
    out = np.zeros((len(idx), c, win, win), np.float32)
    for i, (bn, r, cc) in enumerate(idx):
        y0, x0 = r * s - pad, cc * s - pad
        for wy in range(win):
            sy = y0 + wy
            if not 0 <= sy < h:
                continue
            for wx in range(win):
                sx = x0 + wx
                if not 0 <= sx < w:
                    continue
                v = x[bn, :, sy, sx]
                v = (sc * v).astype(np.float32) + sh
                v = (v * (np.float32(1) + gamma[bn, :, sy, sx])).astype(np.float32)
                v = (v + beta[bn, :, sy, sx]).astype(np.float32)
                if act == sb.ACT_RELU:
                    v = np.where(v > 0, v, np.float32(0))
                elif act == sb.ACT_LEAKY_RELU:
                    v = np.where(v > 0, v, (np.float32(0.2) * v).astype(np.float32))
                out[i, :, wy, wx] = v
    return out


def _case(rng, n=2, c=5, h=23, w=31, b=4, k=3, s=1, p=0.2):
    x = rng.uniform(-2, 2, (n, c, h, w)).astype(np.float32)
    gamma = rng.uniform(-0.5, 0.5, x.shape).astype(np.float32)
    beta = rng.uniform(-0.5, 0.5, x.shape).astype(np.float32)
    oh, ow = (h + 2 * ((k - 1) // 2) - k) // s + 1, (w + 2 * ((k - 1) // 2) - k) // s + 1
    return x, gamma, beta, oh, ow


@pytest.mark.parametrize("act", [0, 1, 3])
@pytest.mark.parametrize("k,s", [(3, 1), (1, 1), (3, 2)])
def test_oracle_gather_spade_matches_numpy(orc, act, k, s):
    rng = np.random.default_rng(10 * act + k + s)
    x, gamma, beta, oh, ow = _case(rng, k=k, s=s)
    m = (rng.random((oh, ow)) < 0.2).astype(np.uint8)
    idx, _ = orc.mask_to_block_indices(m, 4, 2)
    sc = rng.uniform(0.5, 1.5, 5).astype(np.float32)
    sh = rng.uniform(-0.3, 0.3, 5).astype(np.float32)
    got = orc.gather_spade(x, gamma, beta, idx, 4, oh, ow, k, s, [("ss", sc, sh)], act)
    want = _np_gather_spade(x, gamma, beta, np.asarray(idx).reshape(-1, 3), 4, k, s, sc, sh, act)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_oracle_gather_spade_identity_modulation_is_reference_gather(orc, ref):
    rng = np.random.default_rng(4)
    x, _, _, oh, ow = _case(rng)
    z = np.zeros_like(x)
    m = (rng.random((oh, ow)) < 0.3).astype(np.uint8)
    idx, _ = orc.mask_to_block_indices(m, 4, 2)
    epi = [("ss", rng.uniform(0.5, 1.5, 5).astype(np.float32), rng.uniform(-0.3, 0.3, 5).astype(np.float32)),
           ("act", sb.ACT_SILU)]
    got = orc.gather_spade(x, z, z, idx, 4, oh, ow, 3, 1, epi[:1], sb.ACT_SILU)
    want = ref.gather(x, idx, 4, oh, ow, 3, 1, epi)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_oracle_resize_nearest(orc):
    rng = np.random.default_rng(2)
    lab = rng.integers(0, 35, (1, 3, 16, 32)).astype(np.float32)
    up = orc.resize_nearest(lab, 64, 64)
    assert np.array_equal(up, lab.repeat(4, 2).repeat(2, 3))
    down = orc.resize_nearest(lab, 4, 8)
    assert np.array_equal(down, lab[:, :, ::4, ::4])
    t = torch.nn.functional.interpolate(torch.from_numpy(lab), size=(64, 128), mode="nearest").numpy()
    assert np.array_equal(orc.resize_nearest(lab, 64, 128), t)
    with pytest.raises(Exception, match="resize_nearest: non-integer scale"):
        orc.resize_nearest(lab, 12, 32)


@pytest.mark.gpu
@pytest.mark.parametrize("act", [0, 1, 2, 3])
@pytest.mark.parametrize("k,s", [(3, 1), (1, 1), (3, 2)])
def test_gpu_gather_spade_bit_exact(orc, act, k, s):
    rng = np.random.default_rng(100 + 10 * act + k + s)
    for rep in range(3):
        b = int(rng.integers(2, 7))
        x, gamma, beta, oh, ow = _case(rng, n=2, c=int(rng.integers(1, 9)), h=int(rng.integers(8, 40)),
                                       w=int(rng.integers(8, 40)), k=k, s=s)
        m = (rng.random((oh, ow)) < 0.25).astype(np.uint8)
        idx, _ = orc.mask_to_block_indices(m, b, 2)
        c = x.shape[1]
        norm = [("ss", rng.uniform(0.5, 1.5, 2 * c).astype(np.float32), rng.uniform(-0.3, 0.3, 2 * c).astype(np.float32))]
        want = orc.gather_spade(x, gamma, beta, idx, b, oh, ow, k, s, norm, act)
        got = host(sb.gather_spade(cu(x), cu(gamma), cu(beta), cu(np.asarray(idx, np.int32).reshape(-1, 3)), b, k, s,
                                   to_dev_epi(norm), act))
        assert bits_equal(got, want)


@pytest.mark.gpu
def test_gpu_resize_nearest_and_config3_shape(orc):
    rng = np.random.default_rng(9)
    lab = rng.integers(0, 35, (1, 8, 32, 64)).astype(np.float32)
    for oh, ow in [(256, 512), (128, 256), (16, 32), (32, 64)]:
        assert np.array_equal(host(sb.resize_nearest(cu(lab), oh, ow)), orc.resize_nearest(lab, oh, ow))
    with pytest.raises(sb.ConfigError, match="resize_nearest: non-integer scale"):
        sb.resize_nearest(cu(lab), 48, 64)


def test_spade_oracle_matches_torch_functional():
    """oracle/spade.py (numpy float64) against an independent statement of the
    published SPADE generator in torch.nn.functional (conv2d, instance_norm,
    interpolate nearest, leaky_relu), on the config-3 mini generator."""
    import torch.nn.functional as F

    from oracle import spade as osp

    m = sb.Model("gaugan_spade_mini")
    c, h, w = m.in_shape
    orig, _ = sb.make_seg_fixture(1, c, h, w, 5)
    d = m.desc.contents

    def cw(cd):
        wt, b, s = osp.conv_weights(cd)
        return torch.from_numpy(wt), None if b is None else torch.from_numpy(b), s

    def conv(x, cd):
        wt, b, s = cw(cd)
        return F.conv2d(x, wt, b, stride=s, padding=(wt.shape[-1] - 1) // 2)

    def spade(x, seg, sd):
        segk = F.interpolate(seg, size=x.shape[2:], mode="nearest")
        a = F.relu(conv(segk, sd.shared))
        return F.instance_norm(x, eps=sd.eps) * (1 + conv(a, sd.gamma)) + conv(a, sd.beta)

    seg = orig.double()
    x = seg
    for i in range(d.num_layers):
        L = d.layers[i]
        if L.kind == osp.LAYER_RESIZE:
            x = F.interpolate(seg, size=(L.resize_h, L.resize_w), mode="nearest")
        elif L.kind == osp.LAYER_CONV:
            x = conv(x, L.conv)
        elif L.kind == osp.LAYER_UP:
            x = F.interpolate(x, scale_factor=2, mode="nearest")
        elif L.kind == osp.LAYER_ACT:
            x = F.leaky_relu(x, 0.2)
        else:
            assert L.kind == osp.LAYER_SPADE
            sp = L.spade
            dx = conv(F.leaky_relu(spade(x, seg, sp[0]), 0.2), L.conv)
            dx = conv(F.leaky_relu(spade(dx, seg, sp[1]), 0.2), L.conv2)
            xs = conv(spade(x, seg, sp[2]), L.shortcut) if L.has_shortcut else x
            x = xs + dx
    want = x.numpy()
    got = osp.forward(m.desc, orig.numpy())
    assert got.shape == (1, 3, h, w)
    assert np.abs(got - want).max() <= 1e-9 * np.abs(want).max()
