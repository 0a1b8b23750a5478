"""ctypes mirror of include/sige_b200.h (the C-ABI boundary).

The structures here are shared by the product wrapper (`paper_2211_02048_b200`)
and by the test-only oracle bindings (`oracle/`). Loading the CUDA library is
done lazily by :func:`lib`; a missing or unbuildable library raises instead of
falling back to anything.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib

PKG_DIR = pathlib.Path(__file__).resolve().parent
# SIGE_B200_LIB: developer override (A/B against another build of the same ABI).
LIB_PATH = pathlib.Path(os.environ.get("SIGE_B200_LIB", PKG_DIR / "lib" / "libsige_b200.so"))

SIGE_OK = 0
SIGE_ERR_CONFIG = 2
SIGE_ERR_CUDA = 3
SIGE_ERR_INTERNAL = 4

ACT_NONE, ACT_RELU, ACT_SILU = 0, 1, 2
EPI_SCALE_SHIFT, EPI_ACTIVATION = 0, 1
MAX_EPI_STEPS = 4
NORM_GROUP, NORM_INSTANCE, NORM_BATCH = 0, 1, 2
LAYER_CONV, LAYER_NORM, LAYER_ACTIVATION, LAYER_RESBLOCK, LAYER_DOWNSAMPLE, LAYER_UPSAMPLE = range(6)
LAYER_SPADE_RESBLOCK, LAYER_RESIZE = 6, 7
ACT_LEAKY_RELU = 3
MATH_EXACT, MATH_TF32, MATH_FP32_FMA, MATH_F16 = 0, 1, 2, 3

FloatP = C.POINTER(C.c_float)


class EpilogueStep(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("act", C.c_int),
        ("nparams", C.c_int),
        ("scale", C.c_void_p),
        ("shift", C.c_void_p),
    ]


class Epilogue(C.Structure):
    _fields_ = [("num_steps", C.c_int), ("steps", EpilogueStep * MAX_EPI_STEPS)]


class ConvDesc(C.Structure):
    _fields_ = [
        ("c_in", C.c_int),
        ("c_out", C.c_int),
        ("k", C.c_int),
        ("stride", C.c_int),
        ("weight", C.c_void_p),
        ("bias", C.c_void_p),
    ]


class NormDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("groups", C.c_int),
        ("channels", C.c_int),
        ("eps", C.c_float),
        ("gamma", C.c_void_p),
        ("beta", C.c_void_p),
        ("running_mean", C.c_void_p),
        ("running_var", C.c_void_p),
    ]


class SpadeDesc(C.Structure):
    _fields_ = [("eps", C.c_float), ("shared", ConvDesc), ("gamma", ConvDesc), ("beta", ConvDesc)]


class LayerDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("policy_sparse", C.c_int),
        ("min_resolution", C.c_int),
        ("conv", ConvDesc),
        ("norm", NormDesc),
        ("act", C.c_int),
        ("conv2", ConvDesc),
        ("has_shortcut", C.c_int),
        ("shortcut", ConvDesc),
        ("spade", C.POINTER(SpadeDesc)),
        ("resize_h", C.c_int),
        ("resize_w", C.c_int),
    ]


class ModelDesc(C.Structure):
    _fields_ = [
        ("name", C.c_char_p),
        ("in_channels", C.c_int),
        ("in_h", C.c_int),
        ("in_w", C.c_int),
        ("num_layers", C.c_int),
        ("layers", C.POINTER(LayerDesc)),
    ]


class RunConfig(C.Structure):
    _fields_ = [
        ("step", C.c_int),
        ("mask_threshold", C.c_float),
        ("dilate_full", C.c_int),
        ("dilate_scale", C.c_int),
        ("block3", C.c_int),
        ("block1", C.c_int),
        ("min_sparse_res", C.c_int),
        ("sparse", C.c_int),
        ("norm_precompute", C.c_int),
        ("elem_fusion", C.c_int),
        ("scatter_fusion", C.c_int),
        ("seed", C.c_uint32),
    ]


def default_config(**over) -> RunConfig:
    """RunConfig with the reference defaults (graph.hpp:87-101)."""
    cfg = RunConfig(0, 1e-3, 1, 1, 6, 4, -1, 1, 1, 1, 1, 42)
    for k, v in over.items():
        setattr(cfg, k, v)
    return cfg


class ScatterEntry(C.Structure):
    _fields_ = [("block", C.c_int32), ("dy", C.c_int16), ("dx", C.c_int16)]


_LIB = None


def lib() -> C.CDLL:
    """Load the in-tree CUDA library (fails loudly if it is not built)."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        _LIB = C.CDLL(str(LIB_PATH), mode=os.RTLD_GLOBAL if hasattr(os, "RTLD_GLOBAL") else 0)
        _declare(_LIB)
    return _LIB


# C-ABI symbol table: name -> (restype, argtypes). Every symbol declared in
# include/sige_b200.h appears here; tests check the .so exports all of them.
_vp, _i, _f, _sz, _u32, _u64 = C.c_void_p, C.c_int, C.c_float, C.c_size_t, C.c_uint32, C.c_uint64
SYMBOLS = {
    "sige_last_error": (C.c_char_p, []),
    "sige_version": (C.c_char_p, []),
    "sige_kernel_launch_count": (_u64, []),
    "sige_run_config_default": (None, [C.POINTER(RunConfig)]),
    "sige_compute_difference_mask": (_i, [_vp, _vp, _i, _i, _i, _i, _f, _vp, _vp]),
    "sige_downsample_mask": (_i, [_vp, _i, _i, _i, _i, _vp, _vp]),
    "sige_dilate_mask": (_i, [_vp, _i, _i, _i, _vp, _vp]),
    "sige_mask_to_block_indices_async": (_i, [_vp, _i, _i, _i, _i, _vp, _i, _vp, _vp]),
    "sige_mask_to_block_indices": (_i, [_vp, _i, _i, _i, _i, _vp, _i, C.POINTER(_i), _vp]),
    "sige_gather": (_i, [_vp, _i, _i, _i, _i, _vp, _i, _i, _i, _i, _i, _i, C.POINTER(Epilogue), _vp, _vp]),
    "sige_scatter_inplace": (_i, [_vp, _i, _i, _i, _vp, _vp, _i, _i, _i, _i, _vp]),
    "sige_scatter": (_i, [_vp, _i, _i, _i, _vp, _vp, _vp, _i, _i, _i, _i, _vp]),
    "sige_scatter_add_inplace": (_i, [_vp, _i, _i, _i, _vp, _vp, _i, _i, _i, _i, _vp]),
    "sige_build_scatter_map": (_i, [_vp, _i, _i, _i, _i, _vp, C.POINTER(_i), _vp]),
    "sige_scatter_gather": (
        _i,
        [_vp, _i, _i, _vp, _i, _i, _i, _i, _vp, _i, _vp, _i, _i, _i, _i, _i, _i, C.POINTER(Epilogue), _vp, _vp],
    ),
    "sige_scatter_with_block_residual": (
        _i,
        [_vp, _i, _i, _vp, _vp, _i, _i, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _vp],
    ),
    "sige_scatter_with_block_residual_unfused": (
        _i,
        [_vp, _i, _i, _vp, _vp, _i, _i, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _vp],
    ),
    "sige_combine_blocks": (_i, [_vp, _vp, _f, _sz, _vp, _vp]),
    "sige_apply_epilogue_on_blocks": (_i, [_vp, _i, _i, _i, _vp, C.POINTER(Epilogue), _vp]),
    "sige_conv_on_blocks": (_i, [_vp, _i, _i, C.POINTER(ConvDesc), _i, _i, _vp, _i, _vp]),
    "sige_conv2d": (_i, [_vp, _i, _i, _i, _i, C.POINTER(ConvDesc), _i, _i, _vp, _vp]),
    "sige_engine_create": (_i, [C.POINTER(ModelDesc), _i, _i, C.POINTER(_vp)]),
    "sige_engine_destroy": (None, [_vp]),
    "sige_engine_precompute": (_i, [_vp, _vp, _i, _vp]),
    "sige_engine_put_tensor": (_i, [_vp, _i, C.c_char_p, _vp, _sz]),
    "sige_engine_put_norm": (_i, [_vp, _i, C.c_char_p, _vp, _vp, _sz]),
    "sige_engine_get_tensor": (_i, [_vp, _i, C.c_char_p, _vp, _sz]),
    "sige_engine_get_norm": (_i, [_vp, _i, C.c_char_p, _vp, _vp, _sz]),
    "sige_engine_sparse_forward": (_i, [_vp, _vp, _vp, C.POINTER(RunConfig), _vp, _vp]),
    "sige_engine_sparse_forward_host": (_i, [_vp, _vp, _vp, C.POINTER(RunConfig), _vp, _vp]),
    "sige_engine_sparse_forward_grouped": (_i, [_vp, _vp, _vp, C.POINTER(RunConfig), _vp, _vp]),
    "sige_engine_dense_forward": (_i, [_vp, _vp, _i, _i, _vp, _vp]),
    "sige_engine_output_shape": (_i, [_vp, C.POINTER(_i), C.POINTER(_i), C.POINTER(_i), C.POINTER(_i)]),
    "sige_engine_last_launch_count": (_i, [_vp]),
    "sige_engine_trace": (_i, [_vp, _vp, _i, C.POINTER(_i), _vp]),
    "sige_engine_cache_bytes": (_sz, [_vp]),
    "sige_engine_set_profiling": (_i, [_vp, _i]),
    "sige_engine_set_graphs": (_i, [_vp, _i]),
    "sige_engine_set_sm_budget": (_i, [_vp, _i]),
    "sige_engine_profile_read": (_i, [_vp, _vp, _i, C.POINTER(_i), _vp]),
    "sige_engine_set_timeline": (_i, [_vp, _i]),
    "sige_engine_drop_step": (_i, [_vp, _i]),
    "sige_engine_offload_step": (_i, [_vp, _i, _vp]),
    "sige_engine_prefetch_step": (_i, [_vp, _i, _vp]),
    "sige_engine_output_coverage": (_i, [_vp, _vp, _vp, C.POINTER(RunConfig), _vp, C.POINTER(_i), C.POINTER(_i), _vp]),
    "sige_engine_refresh_step": (_i, [_vp, _vp, _i, _vp]),
    "sige_engine_cache_model_hash": (_i, [_vp, C.POINTER(_u64), C.POINTER(_u64)]),
    "sige_engine_set_cache_model_hash": (_i, [_vp, _u64]),
    "sige_model_structure_hash": (_u64, [_vp]),
    "sige_block_index_hash": (_i, [_vp, _i, _i, _i, _i, C.POINTER(_u64), _vp]),
    "sige_scatter_map_cache_get": (_i, [_vp, _i, _i, _i, _i, C.POINTER(_vp), C.POINTER(_i), C.POINTER(_u64), _vp]),
    "sige_scatter_map_cache_size": (_sz, []),
    "sige_scatter_map_cache_clear": (None, []),
    "sige_engine_timeline_read": (_i, [_vp, _vp, _i, C.POINTER(_i)]),
    "sige_engine_cache_entries": (_i, [_vp, _i, C.c_char_p, _sz, C.POINTER(_sz)]),
    "sige_make_edit_fixture": (_i, [C.c_char_p, _i, _i, _i, _i, _u32, _vp, _vp]),
    "sige_make_seg_fixture": (_i, [_i, _i, _i, _i, _u32, _vp, _vp]),
    "sige_gather_spade": (_i, [_vp, _vp, _vp, _i, _i, _i, _i, _vp, _i, _i, _i, _i, _i, _i, C.POINTER(Epilogue), _i, _vp, _vp]),
    "sige_resize_nearest": (_i, [_vp, _i, _i, _i, _i, _i, _i, _vp, _vp]),
    "sige_save_tensor": (_i, [C.c_char_p, _vp, _i, _i, _i, _i]),
    "sige_load_tensor": (_i, [C.c_char_p, _vp, C.c_size_t, C.POINTER(_i)]),
    "sige_save_mask_pbm": (_i, [C.c_char_p, _vp, _i, _i]),
    "sige_load_mask_pbm": (_i, [C.c_char_p, _vp, C.c_size_t, C.POINTER(_i), C.POINTER(_i)]),
    "sige_save_block_stack": (_i, [C.c_char_p, _vp, _i, _i, _i, _i, _i, _i, _i, _vp]),
    "sige_load_block_stack": (_i, [C.c_char_p, _vp, C.c_size_t, _vp, C.c_size_t, C.POINTER(_i)]),
    "sige_model_build": (_i, [C.c_char_p, C.POINTER(C.POINTER(ModelDesc))]),
    "sige_model_free": (None, [C.POINTER(ModelDesc)]),
    "sige_model_required_dilation": (_i, [C.POINTER(ModelDesc), C.POINTER(_i)]),
    "sige_model_weight_hash": (_u64, [C.POINTER(ModelDesc)]),
}


def _declare(L: C.CDLL) -> None:
    override = "SIGE_B200_LIB" in os.environ  # an older build may lack newer entry points
    for name, (res, args) in SYMBOLS.items():
        if override and not hasattr(L, name):
            continue
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
