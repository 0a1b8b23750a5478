"""On-disk exchange formats (io.hpp:12-36) through the library's C ABI against
the reference's own io.cpp (compiled into oracle/_ref when nlohmann/json is
available): files written by either side load in the other, the bytes are
identical, and malformed files fail with the reference's ConfigError text.
Host-only — runs without a GPU."""
import ctypes as C

import numpy as np
import pytest
import torch

import paper_2211_02048_b200 as sb

_i, _vp, _sz = C.c_int, C.c_void_p, C.c_size_t


@pytest.fixture(scope="module")
def refio(ref):
    L = ref.lib
    if not hasattr(L, "ref_io_save_tensor"):
        pytest.skip("reference io.cpp not built (nlohmann/json absent)")
    L.ref_io_save_tensor.argtypes = [C.c_char_p, _vp, _i, _i, _i, _i]
    L.ref_io_load_tensor.argtypes = [C.c_char_p, _vp, _sz, C.POINTER(_i)]
    L.ref_io_save_mask_pbm.argtypes = [C.c_char_p, _vp, _i, _i]
    L.ref_io_load_mask_pbm.argtypes = [C.c_char_p, _vp, _sz, C.POINTER(_i), C.POINTER(_i)]
    L.ref_io_save_block_stack.argtypes = [C.c_char_p, _vp, _i, _i, _i, _i, _i, _i, _i, _vp]
    L.ref_io_load_block_stack.argtypes = [C.c_char_p, _vp, _sz, _vp, _sz, C.POINTER(_i)]
    for f in ("save_tensor", "load_tensor", "save_mask_pbm", "load_mask_pbm", "save_block_stack", "load_block_stack"):
        getattr(L, "ref_io_" + f).restype = _i
    L.ref_last_error.restype = C.c_char_p
    return L


def _ok(L, rc):
    assert rc == 0, L.ref_last_error().decode()


def test_tensor_bytes_and_cross_load(refio, tmp_path):
    rng = np.random.default_rng(3)
    x = rng.standard_normal((2, 3, 5, 7)).astype(np.float32)
    x[0, 0, 0, :3] = [np.float32(-0.0), np.inf, np.float32(1e-40)]  # sign, inf, subnormal bits survive
    ours, theirs = tmp_path / "ours.sigt", tmp_path / "theirs.sigt"
    sb.save_tensor(str(ours), torch.from_numpy(x))
    _ok(refio, refio.ref_io_save_tensor(str(theirs).encode(), x.ctypes.data, *x.shape))
    assert ours.read_bytes() == theirs.read_bytes()
    got = sb.load_tensor(str(theirs)).numpy()
    assert np.array_equal(got.view(np.uint32), x.view(np.uint32))
    back = np.empty_like(x)
    dims = (_i * 4)()
    _ok(refio, refio.ref_io_load_tensor(str(ours).encode(), back.ctypes.data, back.size, dims))
    assert tuple(dims) == x.shape and np.array_equal(back.view(np.uint32), x.view(np.uint32))


def test_tensor_errors_match_reference(refio, tmp_path):
    x = np.ones((1, 1, 2, 2), np.float32)
    good = tmp_path / "g.sigt"
    sb.save_tensor(str(good), torch.from_numpy(x))
    raw = good.read_bytes()
    cases = {
        "badmagic": b"XIGT" + raw[4:],
        "version": raw[:4] + (2).to_bytes(4, "little") + raw[8:],
        "trunc": raw[:-3],
        "trailing": raw + b"\0",
        "zero": raw[:8] + (0).to_bytes(4, "little") + raw[12:24],
    }
    for name, data in cases.items():
        p = tmp_path / f"{name}.sigt"
        p.write_bytes(data)
        dims = (_i * 4)()
        buf = np.empty(16, np.float32)
        assert refio.ref_io_load_tensor(str(p).encode(), buf.ctypes.data, buf.size, dims) != 0
        want = refio.ref_last_error().decode()
        with pytest.raises(sb.ConfigError) as ei:
            sb.load_tensor(str(p))
        assert str(ei.value) == want, name
    with pytest.raises(sb.ConfigError, match="cannot open"):
        sb.load_tensor(str(tmp_path / "missing.sigt"))


def test_pbm_bytes_and_cross_load(refio, tmp_path):
    rng = np.random.default_rng(5)
    m = (rng.random((9, 13)) < 0.3).astype(np.uint8)
    ours, theirs = tmp_path / "ours.pbm", tmp_path / "theirs.pbm"
    sb.save_mask_pbm(str(ours), torch.from_numpy(m))
    _ok(refio, refio.ref_io_save_mask_pbm(str(theirs).encode(), m.ctypes.data, *m.shape))
    assert ours.read_bytes() == theirs.read_bytes()
    assert np.array_equal(sb.load_mask_pbm(str(theirs)).numpy(), m)
    # comments and digits packed without whitespace (io.cpp:138-156)
    packed = tmp_path / "packed.pbm"
    packed.write_text("P1\n# a comment\n13 9\n" + "\n".join("".join(str(v) for v in row) for row in m) + "\n")
    assert np.array_equal(sb.load_mask_pbm(str(packed)).numpy(), m)
    h, w = _i(), _i()
    back = np.empty(m.size, np.uint8)
    _ok(refio, refio.ref_io_load_mask_pbm(str(packed).encode(), back.ctypes.data, back.size, C.byref(h), C.byref(w)))
    assert np.array_equal(back.reshape(m.shape), m)


@pytest.mark.parametrize("text", ["P1 #c 9\n3 2 # w h\n1 0 1\n# mid-payload comment 1 1\n0 1 0\n",
                                  "P1\n3 2\n101#x\n010", "#lead\nP1\n3\n2\n1\t0 1 0 1 0 1 1 1",
                                  "P1\n3 2 101010"])
def test_pbm_grammar_matches_reference(refio, tmp_path, text):
    """Header comments, payload comments, packed / tab-separated bits, a missing
    final newline and trailing extra bits load the same as the reference's."""
    p = tmp_path / "g.pbm"
    p.write_text(text)
    h, w = _i(), _i()
    want = np.empty(6, np.uint8)
    _ok(refio, refio.ref_io_load_mask_pbm(str(p).encode(), want.ctypes.data, want.size, C.byref(h), C.byref(w)))
    assert (h.value, w.value) == (2, 3)
    assert np.array_equal(sb.load_mask_pbm(str(p)).numpy().reshape(-1), want)


@pytest.mark.parametrize("text", ["P2\n2 2\n0 1 1 0\n", "P1\n2 2\n0 1 1\n", "P1\n2 2\n0 1 x 0\n", "P1\n0 2\n",
                                  "P1\n2", "# only a comment\n", "P1\n2 2\n0 1 # 1 0\n"])
def test_pbm_errors_match_reference(refio, tmp_path, text):
    p = tmp_path / "bad.pbm"
    p.write_text(text)
    h, w = _i(), _i()
    buf = np.empty(16, np.uint8)
    assert refio.ref_io_load_mask_pbm(str(p).encode(), buf.ctypes.data, buf.size, C.byref(h), C.byref(w)) != 0
    want = refio.ref_last_error().decode()
    with pytest.raises(sb.ConfigError) as ei:
        sb.load_mask_pbm(str(p))
    assert str(ei.value) == want


@pytest.mark.parametrize("count,block,overlap", [(0, 6, 2), (1, 4, 0), (37, 6, 2)])
def test_block_stack_bytes_and_cross_load(refio, orc, tmp_path, count, block, overlap):
    rng = np.random.default_rng(7 + count)
    h = w = 64
    m = np.zeros((h, w), np.uint8)
    if count:
        m[rng.integers(0, h, count), rng.integers(0, w, count)] = 1
    idx, _ = orc.mask_to_block_indices(m, block, 2)
    g = len(idx)
    bh = block + overlap
    blocks = rng.standard_normal((g, 5, bh, bh)).astype(np.float32)
    ours, theirs = tmp_path / "ours", tmp_path / "theirs"
    sb.save_block_stack(str(ours), torch.from_numpy(blocks), torch.from_numpy(np.asarray(idx, np.int32).reshape(-1, 3)),
                        block, overlap, (h, w))
    ii = np.ascontiguousarray(np.asarray(idx, np.int32).reshape(-1, 3))
    _ok(refio, refio.ref_io_save_block_stack(str(theirs).encode(), blocks.ctypes.data, g, 5, block, overlap, block, h, w,
                                             ii.ctypes.data))
    for ext in (".sigt", ".json"):
        assert (tmp_path / ("ours" + ext)).read_bytes() == (tmp_path / ("theirs" + ext)).read_bytes(), ext
    r = sb.load_block_stack(str(theirs))
    assert r["block"] == block and r["overlap"] == overlap and r["origin_hw"] == (h, w) and r["origin_block"] == block
    assert np.array_equal(r["idx"].numpy(), ii) and np.array_equal(r["blocks"].numpy(), blocks)
    meta = (_i * 7)()
    back = np.empty(max(blocks.size, 1), np.float32)
    bi = np.empty(max(ii.size, 1), np.int32)
    _ok(refio, refio.ref_io_load_block_stack(str(ours).encode(), back.ctypes.data, back.size, bi.ctypes.data, bi.size,
                                             meta))
    assert list(meta) == [g, 5 if g else 0, block, overlap, block, h, w] or list(meta)[0] == 0


def test_block_stack_errors_match_reference(refio, tmp_path):
    blocks = np.ones((2, 1, 8, 8), np.float32)
    idx = np.array([[0, 0, 0], [0, 0, 6]], np.int32)
    base = tmp_path / "s"
    sb.save_block_stack(str(base), torch.from_numpy(blocks), torch.from_numpy(idx), 6, 2, (12, 12))
    js = (tmp_path / "s.json").read_text()
    cases = {
        "format": js.replace("sige_blocks_v1", "sige_blocks_v2"),
        "count": js.replace("[0,0,6]", "[0,0,6],\n    [0,6,0]"),
        "geometry": js.replace('"overlap": 2', '"overlap": 1'),
    }
    for name, text in cases.items():
        (tmp_path / "s.json").write_text(text)
        meta = (_i * 7)()
        assert refio.ref_io_load_block_stack(str(base).encode(), None, 0, None, 0, meta) != 0
        want = refio.ref_last_error().decode()
        with pytest.raises(sb.ConfigError) as ei:
            sb.load_block_stack(str(base))
        assert str(ei.value) == want, name
