"""CPU checks of the C-ABI library (no GPU needed): it loads, exports every
symbol include/sige_b200.h declares, and its host-side code (synthetic
inputs, model builders, validation) agrees with the oracle / reference."""
import ctypes as C
import pathlib
import re
import subprocess

import numpy as np
import pytest

import paper_2211_02048_b200 as sb
from paper_2211_02048_b200 import _capi

ROOT = pathlib.Path(__file__).resolve().parents[1]


def test_library_exports_every_header_symbol():
    hdr = (ROOT / "include" / "sige_b200.h").read_text()
    declared = set(re.findall(r"\b(sige_[a-z0-9_]+)\s*\(", hdr))
    L = _capi.lib()
    assert declared, "no symbols parsed"
    missing = sorted(s for s in declared if not hasattr(L, s))
    assert not missing, missing
    assert declared == set(_capi.SYMBOLS), declared ^ set(_capi.SYMBOLS)
    out = subprocess.run(["nm", "-D", "--defined-only", str(_capi.LIB_PATH)], capture_output=True, text=True).stdout
    for s in declared:
        assert re.search(rf"\bT {s}\b", out), s


def test_library_has_sm100a_code():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_capi.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", str(_capi.LIB_PATH)], capture_output=True, text=True).stdout
    for mnemonic in ("UTCHMMA", "LDTM", "UTMALDG"):  # tcgen05.mma / tcgen05.ld / TMA load
        assert mnemonic in sass, mnemonic


def test_run_config_defaults():
    c = _capi.RunConfig()
    _capi.lib().sige_run_config_default(C.byref(c))
    ref = sb.default_config()
    for f, _ in _capi.RunConfig._fields_:
        assert getattr(c, f) == pytest.approx(getattr(ref, f)), f
    assert (c.block3, c.block1, c.dilate_full, c.min_sparse_res) == (6, 4, 1, -1)


@pytest.mark.parametrize("kind", ["rect1", "rect5", "blob5", "multi15", "rect35"])
def test_fixtures_match_oracle(orc, kind):
    o, e = sb.make_edit_fixture(kind, 2, 3, 48, 40, 21)
    o2, e2 = orc.make_edit_fixture(kind, 2, 3, 48, 40, 21)
    assert np.array_equal(o.numpy(), o2) and np.array_equal(e.numpy(), e2)


@pytest.mark.parametrize("name", ["conv3x3_128", "mini_unet_gn", "mini_unet_bn", "gaugan_stack_in",
                                  "single_conv64", "ddim_stack", "ddim_stack_64x32"])
def test_models_match_oracle(orc, name):
    m = sb.Model(name)
    om = orc.model(name)
    assert m.weight_hash() == om.weight_hash()
    assert m.required_dilation() == om.required_dilation()


def test_host_errors_are_config_errors():
    with pytest.raises(sb.ConfigError, match="unknown model"):
        sb.Model("nope")
    with pytest.raises(sb.ConfigError, match="unknown edit fixture"):
        sb.make_edit_fixture("bogus", 1, 1, 8, 8, 1)
    assert _capi.lib().sige_last_error().decode().startswith("unknown edit fixture")


def test_ddim_stack_structure():
    """Config 2: 51 layers, 80 conv sites, 128-512 channels."""
    model = sb.Model("ddim_stack")  # keep alive: desc points into its storage
    d = model.desc.contents
    assert d.num_layers == 51
    convs = 0
    chans = set()
    for i in range(d.num_layers):
        L = d.layers[i]
        if L.kind in (_capi.LAYER_CONV, _capi.LAYER_DOWNSAMPLE):
            convs += 1
            chans.add(L.conv.c_out)
        elif L.kind == _capi.LAYER_RESBLOCK:
            convs += 2 + L.has_shortcut
            chans.add(L.conv2.c_out)
    assert convs == 80
    assert chans == {3, 128, 256, 512}


def test_structure_hash_matches_reference(ref):
    """ModelSpec::structure_hash (graph.cpp:89-127) — the cache/model guard key —
    restated in models.cpp equals the reference's for every model (host only)."""
    import ctypes as C

    import paper_2211_02048_b200 as sb

    ref.lib.ref_model_structure_hash.restype = C.c_uint64
    ref.lib.ref_model_structure_hash.argtypes = [C.c_void_p]
    for name in ("mini_unet_gn", "mini_unet_bn", "gaugan_stack_in", "conv3x3_128", "single_conv64", "ddim_stack",
                 "ddim_stack_64x32"):
        m = sb.Model(name)
        rm = ref.model(name)
        assert m.structure_hash() == ref.lib.ref_model_structure_hash(rm.h), name
