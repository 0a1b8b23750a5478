"""GPU tests of the tcgen05 (kind::tf32) fused conv path.

1. Indexing exactness: with small-integer activations and weights every
   product and partial sum is exact in TF32/FP32, so the tensor-core result
   must equal the oracle bit for bit — this pins the implicit-GEMM data
   movement (window staging, tap descriptor shifts, stride-2 phase planes,
   multi-tile M packing, N tiling, fringe clipping) independent of rounding.
2. Real data: normalised max error <= 1e-2 (north-star tolerance, SURVEY
   §8(c)) on the toy models, config 1 and a reduced config 2, with pixels
   outside the touched tiles bit-identical to the cache.
"""
import ctypes as C

import numpy as np
import pytest
import torch

import paper_2211_02048_b200 as sb
from paper_2211_02048_b200 import _capi

pytestmark = pytest.mark.gpu


class DescBuilder:
    """Build a sige_model_desc from numpy weights (kept alive by this object)."""

    def __init__(self, name, c, h, w):
        self.keep = []
        self.layers = []
        self.name = name.encode()
        self.shape = (c, h, w)

    def _arr(self, a):
        a = np.ascontiguousarray(a, np.float32)
        self.keep.append(a)
        return a.ctypes.data

    def conv(self, wt, bias, stride):
        L = _capi.LayerDesc()
        L.kind = _capi.LAYER_DOWNSAMPLE if stride == 2 else _capi.LAYER_CONV
        L.policy_sparse = 1
        L.min_resolution = 1
        L.conv = _capi.ConvDesc(wt.shape[1], wt.shape[0], wt.shape[2], stride, self._arr(wt),
                                self._arr(bias) if bias is not None else None)
        self.layers.append(L)
        return self

    def build(self):
        arr = (_capi.LayerDesc * len(self.layers))(*self.layers)
        self.keep.append(arr)
        d = _capi.ModelDesc(self.name, *self.shape, len(self.layers), arr)
        self.keep.append(d)
        return sb.Model(C.pointer(d), owner=self)


def int_case(rng, n, c_in, c_out, k, s, h, w):
    orig = rng.integers(-2, 3, (n, c_in, h, w)).astype(np.float32)
    edited = orig.copy()
    y0, x0 = rng.integers(0, h - 3), rng.integers(0, w - 3)
    edited[:, :, y0:y0 + 3, x0:x0 + 3] = rng.integers(-2, 3, (n, c_in, 3, 3))
    edited[:, 0, y0, x0] = orig[:, 0, y0, x0] + 1.0
    wt = rng.integers(-2, 3, (c_out, c_in, k, k)).astype(np.float32)
    bias = rng.integers(-3, 4, c_out).astype(np.float32)
    return orig, edited, wt, bias


GEOMS = [  # n, c_in, c_out, k, s, h, w, block
    (1, 3, 16, 3, 1, 64, 64, 6),
    (1, 64, 64, 3, 1, 64, 48, 6),
    (2, 32, 48, 3, 1, 40, 40, 6),
    (1, 128, 256, 3, 1, 32, 32, 6),
    (1, 256, 128, 1, 1, 32, 32, 4),
    (1, 64, 64, 3, 2, 64, 64, 6),
    (1, 40, 24, 3, 2, 50, 38, 6),
    (1, 16, 3, 3, 1, 33, 29, 4),
    (1, 96, 96, 3, 1, 48, 48, 8),
    (1, 512, 512, 3, 1, 16, 16, 6),
]


@pytest.mark.parametrize("g", GEOMS, ids=[f"n{g[0]}c{g[1]}-{g[2]}k{g[3]}s{g[4]}_{g[5]}x{g[6]}b{g[7]}" for g in GEOMS])
@pytest.mark.parametrize("math", [sb.MATH_TF32, sb.MATH_F16], ids=["tf32", "f16"])
def test_tc_conv_integer_bit_exact(orc, g, math):
    n, c_in, c_out, k, s, h, w, b = g
    rng = np.random.default_rng(hash(g) % 2**32)
    orig, edited, wt, bias = int_case(rng, n, c_in, c_out, k, s, h, w)
    db = DescBuilder("int_conv", c_in, h, w).conv(wt, bias, s)
    model = db.build()
    om = orc.model(model.desc.contents)
    mask = orc.difference_mask(orig, edited)
    cfg = sb.default_config(dilate_full=1, block3=b, block1=b, min_sparse_res=1)
    ocache = om.precompute(orig)
    want, _ = om.sparse_forward(ocache, edited, mask, cfg)
    for precompute_on_device in (False, True):
        eng = sb.Engine(model, batch=n, math=math)
        if precompute_on_device:
            eng.precompute(torch.from_numpy(orig).cuda())
            # the dense pass also runs on tensor cores: integer data keeps it exact
            assert np.array_equal(eng.get_tensor("L0.out", ocache.tensor("L0.out").shape).numpy(),
                                  ocache.tensor("L0.out"))
        else:
            eng.put_tensor("L0.out", ocache.tensor("L0.out"))
            eng.put_tensor("final", ocache.tensor("final"))
            eng.put_tensor("input", orig)
        got = eng.sparse_forward(torch.from_numpy(edited).cuda(), config=cfg)
        torch.cuda.synchronize()
        got = got.cpu().numpy()
        assert np.array_equal(got, want), f"max diff {np.abs(got - want).max()}"
        dense = eng.dense_forward(torch.from_numpy(edited).cuda()).cpu().numpy()
        assert np.array_equal(dense, om.dense_forward(edited))


def norm_err(got, want):
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-30))


CASES = [
    ("mini_unet_gn", "rect5", 1, 17, {}),
    ("mini_unet_bn", "rect15", 1, 11, {"dilate_full": 3}),
    ("gaugan_stack_in", "multi15", 1, 3, {}),
    ("ddim_stack_64x32", "rect5", 1, 7, {"dilate_full": 5, "min_sparse_res": 16}),
    ("ddim_stack_64x32", "blob5", 2, 8, {"dilate_full": 2, "min_sparse_res": 8}),
]


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}-{c[1]}-n{c[2]}" for c in CASES])
@pytest.mark.parametrize("math", [sb.MATH_TF32, sb.MATH_F16], ids=["tf32", "f16"])
def test_tc_engine_tolerance(orc, case, math):
    name, fx, n, seed, over = case
    om = orc.model(name)
    c, h, w = sb.Model(name).in_shape
    orig, edited = orc.make_edit_fixture(fx, n, c, h, w, seed)
    mask = orc.difference_mask(orig, edited)
    over = dict(over)
    df = over.pop("dilate_full", None)
    cfg = sb.default_config(dilate_full=om.required_dilation() if df is None else df, **over)
    ocache = om.precompute(orig)
    want, _ = om.sparse_forward(ocache, edited, mask, cfg)
    eng = sb.Engine(sb.Model(name), batch=n, math=math)
    # cache from the CPU precompute isolates the sparse path's own error
    for kind, key, numel in ocache.entries():
        if kind == 0:
            eng.put_tensor(key, ocache.tensor(key))
        else:
            eng.put_norm(key, *ocache.norm(key))
    eng.put_tensor("input", orig)
    got = eng.sparse_forward(torch.from_numpy(edited).cuda(), config=cfg).cpu().numpy()
    err = norm_err(got, want)
    assert err <= 1e-2, err
    # pixels outside the sparse footprint (reference output_coverage,
    # graph.cpp:1078-1129) equal the cached output exactly
    import oracle

    if oracle.ref_available():
        R = oracle.ref()
        rm = R.model(om.desc.contents)
        cov = np.zeros((h, w), np.uint8)
        oh, ow = C.c_int(), C.c_int()
        rc = R.lib.ref_output_coverage(rm.h, np.ascontiguousarray(mask).ctypes.data, h, w, n, C.byref(cfg),
                                       cov.ctypes.data, C.byref(oh), C.byref(ow))
        assert rc == 0
        fin = ocache.tensor("final")
        outside = np.broadcast_to(cov[None, None] == 0, fin.shape)
        assert outside.any() and np.array_equal(got[outside], fin[outside])
    # and with the device precompute
    eng2 = sb.Engine(sb.Model(name), batch=n, math=math)
    eng2.precompute(torch.from_numpy(orig).cuda())
    got2 = eng2.sparse_forward(torch.from_numpy(edited).cuda(), config=cfg).cpu().numpy()
    assert norm_err(got2, want) <= 1e-2


@pytest.mark.parametrize("math", [sb.MATH_TF32, sb.MATH_F16], ids=["tf32", "f16"])
def test_tc_config1_full_size(orc, math):
    om = orc.model("single_conv64")
    orig, edited = orc.make_edit_fixture("rect1", 1, 64, 256, 256, 7)
    mask = orc.difference_mask(orig, edited)
    cfg = sb.default_config(dilate_full=1)
    ocache = om.precompute(orig)
    want, _ = om.sparse_forward(ocache, edited, mask, cfg)
    eng = sb.Engine(sb.Model("single_conv64"), math=math)
    eng.precompute(torch.from_numpy(orig).cuda())
    got = eng.sparse_forward(torch.from_numpy(edited).cuda(), config=cfg).cpu().numpy()
    assert norm_err(got, want) <= 1e-2
    assert int(eng.trace()[0][0]) == 36
