"""The oracle (oracle/sige_oracle.c, a C restatement of the reference) pinned
against the reference's own known answers and the golden vectors generated
from the compiled reference (tests/golden/make_golden.py). CPU only."""
import json
import pathlib

import numpy as np
import pytest

from paper_2211_02048_b200._capi import default_config

GOLD = pathlib.Path(__file__).resolve().parent / "golden"
META = json.loads((GOLD / "golden.json").read_text())
ARR = np.load(GOLD / "golden.npz")


def content_hash(orc, t):  # Tensor::content_hash (tensor.cpp:28-32)
    return orc.fnv1a64(t, orc.fnv1a64(np.array(t.shape, np.int32)))


def test_rng_is_mt19937(orc):
    u, _ = orc.rng_stream(5489, 10000)
    assert int(u[-1]) == 4123659995  # the C++ standard's required 10000th mt19937 output (seed 5489)


def test_survey_appendix_b_chain(orc):
    o, e = orc.make_edit_fixture("rect1", 1, 64, 256, 256, 7)
    assert content_hash(orc, o) == 0x12DECF015379559B == META["rect1_64x256_original_hash"]
    assert content_hash(orc, e) == 0x1414A628CDF89474 == META["rect1_64x256_edited_hash"]
    m = orc.difference_mask(o, e, 1e-3)
    assert orc.fnv1a64(m) == 0x938A3A322907C793 == META["rect1_mask_hash"]
    assert int(m.sum()) == 784
    ys, xs = np.nonzero(m)
    assert (ys.min(), ys.max(), xs.min(), xs.max()) == (209, 236, 14, 41)
    d = orc.dilate_mask(orc.dilate_mask(m, 1), 1)
    idx6, h6 = orc.mask_to_block_indices(d, 6, 1)
    assert len(idx6) == 36 and h6 == 0xCCBB614A2A613105 == META["rect1_idx6_hash"]
    assert idx6[0].tolist() == [0, 204, 12] and idx6[-1].tolist() == [0, 234, 42]
    assert np.array_equal(idx6, ARR["rect1_idx6"])
    assert len(orc.mask_to_block_indices(d, 4, 1)[0]) == 72 == META["rect1_idx4_count"]
    g = orc.gather(e, idx6, 6, 256, 256, 3, 1)
    assert g.size == 147456 and orc.fnv1a64(g) == 0x7A0D773D8E4FE522 == META["rect1_gather_hash"]
    epi = [("ss", ARR["silu_scale"], ARR["silu_shift"]), ("act", 2)]
    assert np.array_equal(orc.gather(e, idx6[:8], 6, 256, 256, 3, 1, epi), ARR["rect1_gather_silu"])


@pytest.mark.parametrize("name,whash,dil", [
    ("conv3x3_128", 18144649916616864714, 1),  # test_graph.cpp:151-166
    ("mini_unet_gn", 1307337009021890759, 25),
    ("mini_unet_bn", 6248356019700358048, 25),
    ("gaugan_stack_in", 16716000267166235036, 16),
    ("single_conv64", None, 1),
    ("ddim_stack", None, 822),
    ("ddim_stack_64x32", None, 822),
])
def test_model_weights_frozen(orc, name, whash, dil):
    m = orc.model(name)
    assert m.weight_hash() == META[f"weight_hash_{name}"]
    if whash is not None:
        assert m.weight_hash() == whash
    assert m.required_dilation() == dil == META[f"required_dilation_{name}"]


def test_cache_accounting(orc):
    # test_graph.cpp:314-333: mini_unet_gn, rect5 seed 7 -> 991584 floats, 31 entries
    m = orc.model("mini_unet_gn")
    o, _ = orc.make_edit_fixture("rect5", 1, 3, 64, 64, 7)
    c = m.precompute(o)
    assert c.total_elements() == 991584
    ents = c.entries()
    assert len(ents) == 31
    conv = sum(n for k, key, n in ents if k == 0 and (key.endswith(".out") and "shortcut" not in key))
    extras = sum(n for k, key, n in ents if k == 0 and (key.endswith(".sum") or key.endswith("shortcut.out")))
    assert conv == 552960 and extras == 425984
    assert sum(n for k, key, n in ents if key == "final") == 12288
    assert sum(2 * n for k, key, n in ents if k == 1) == 352


GOLDEN_CASES = [k[: -len("_config")] for k in META if k.endswith("_config")]


@pytest.mark.parametrize("tag", GOLDEN_CASES)
def test_sparse_forward_golden(orc, tag):
    cfgm = META[f"{tag}_config"]
    m = orc.model(cfgm["model"])
    o, e = orc.make_edit_fixture(cfgm["fixture"], cfgm["batch"], 3, 64, 64, cfgm["seed"])
    mask = orc.difference_mask(o, e)
    over = {k: v for k, v in cfgm.items() if k not in ("model", "fixture", "batch", "seed")}
    cache = m.precompute(o)
    out, trace = m.sparse_forward(cache, e, mask, default_config(**over))
    assert np.array_equal(out.view(np.uint32), ARR[f"{tag}_out"].view(np.uint32))
    assert np.array_equal(trace, ARR[f"{tag}_trace"])
    assert cache.total_elements() == META[f"{tag}_cache_total_elements"]


# ---- frozen cases of the reference's unit tests (restated)

def test_frozen_gather_windows(orc):
    x = np.arange(16, dtype=np.float32).reshape(1, 1, 4, 4)  # test_kernels.cpp:61-92
    g = orc.gather(x, np.array([[0, 0, 0]], np.int32), 2, 4, 4, 3, 1)
    assert g.ravel().tolist() == [0, 0, 0, 0, 0, 0, 1, 2, 0, 4, 5, 6, 0, 8, 9, 10]
    g = orc.gather(x, np.array([[0, 2, 2]], np.int32), 2, 4, 4, 3, 1)
    assert g.ravel().tolist() == [5, 6, 7, 0, 9, 10, 11, 0, 13, 14, 15, 0, 0, 0, 0, 0]
    assert orc.gather(x, np.array([[0, 2, 2]], np.int32), 2, 4, 4, 1, 1).ravel().tolist() == [10, 11, 14, 15]


def test_frozen_masks(orc):
    m = np.zeros((8, 8), np.uint8)  # test_mask.cpp:53-120
    m[5, 5] = 1
    d = orc.downsample_mask(m, 4, 4)
    assert d.sum() == 1 and d[2, 2] == 1
    c = np.zeros((5, 5), np.uint8)
    c[0, 0] = 1
    assert orc.dilate_mask(c, 2).sum() == 9
    m = np.zeros((10, 10), np.uint8)
    m[9, 9] = 1
    idx, _ = orc.mask_to_block_indices(m, 4, 1)
    assert idx.tolist() == [[0, 8, 8]]
    full = np.ones((12, 12), np.uint8)
    i2, _ = orc.mask_to_block_indices(full, 6, 2)
    assert len(i2) == 8 and i2[4, 0] == 1


def test_config_errors(orc):
    import oracle

    with pytest.raises(oracle.OracleError, match="downsample_mask: non-integer scale factor"):
        orc.downsample_mask(np.zeros((8, 8), np.uint8), 3, 3)
    with pytest.raises(oracle.OracleError, match="gather: kernel size must be 1 or 3"):
        orc.gather(np.zeros((1, 1, 8, 8), np.float32), np.zeros((1, 3), np.int32), 2, 8, 8, 5, 1)
