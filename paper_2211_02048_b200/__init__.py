"""SIGE spatially sparse update path on B200 (sm_100a).

Python mirror of the reference's C++ operator API (``proj/include/sige/*.hpp``,
namespace ``sige``) over the C-ABI library ``lib/libsige_b200.so``: the same
function names, argument meaning and error behaviour (``ConfigError`` with the
reference's messages), on CUDA tensors. Device memory and streams come from
PyTorch; every computation runs in this package's own sm_100a kernels.

Layouts follow the reference: tensors NCHW float32, masks uint8 (H, W), index
sets int32 (G, 3) rows {n, r, c}, block stacks (G, C, bh, bw).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import torch

from . import _capi
from ._capi import (  # noqa: F401  (re-exported constants)
    ACT_NONE,
    ACT_RELU,
    ACT_SILU,
    MATH_EXACT,
    MATH_F16,
    MATH_FP32_FMA,
    MATH_TF32,
    RunConfig,
    default_config,
)

__all__ = [
    "ConfigError", "Epilogue", "Model", "Engine", "RunConfig", "default_config",
    "compute_difference_mask", "downsample_mask", "dilate_mask", "mask_to_block_indices",
    "gather", "scatter", "scatter_inplace", "scatter_add_inplace", "build_scatter_map",
    "scatter_gather", "scatter_with_block_residual", "scatter_with_block_residual_unfused",
    "add_blocks", "subtract_blocks", "apply_epilogue_on_blocks", "conv_on_blocks", "conv2d",
    "make_edit_fixture", "kernel_launch_count", "ScatterMapCache", "block_index_hash",
]


class ConfigError(ValueError):
    """The reference's sige::ConfigError (proj/include/sige/common.hpp:14-17)."""


class SigeCudaError(RuntimeError):
    pass


def _lib():
    return _capi.lib()


def _check(rc: int) -> None:
    if rc == _capi.SIGE_OK:
        return
    msg = _lib().sige_last_error().decode()
    if rc == _capi.SIGE_ERR_CONFIG:
        raise ConfigError(msg)
    raise SigeCudaError(msg)


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _dev(t: torch.Tensor, dtype, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ConfigError(f"{name}: expected a CUDA tensor")
    if t.dtype != dtype:
        raise ConfigError(f"{name}: expected {dtype}, got {t.dtype}")
    return t.contiguous()


def kernel_launch_count() -> int:
    """How many kernels of libsige_b200 have launched in this process."""
    return int(_lib().sige_kernel_launch_count())


@dataclass
class Epilogue:
    """Deferred element-wise chain (proj/include/sige/eltwise.hpp:30-59)."""

    steps: list = field(default_factory=list)

    def add_scale_shift(self, scale: torch.Tensor, shift: torch.Tensor) -> "Epilogue":
        self.steps.append(("ss", scale.float().contiguous().cuda(), shift.float().contiguous().cuda()))
        return self

    def add_activation(self, kind: int) -> "Epilogue":
        if kind != ACT_NONE:  # eltwise.cpp:99-105
            self.steps.append(("act", int(kind)))
        return self

    def struct(self) -> _capi.Epilogue:
        e = _capi.Epilogue()
        e.num_steps = len(self.steps)
        for k, st in enumerate(self.steps):
            if st[0] == "ss":
                e.steps[k].kind = _capi.EPI_SCALE_SHIFT
                e.steps[k].nparams = st[1].numel()
                e.steps[k].scale = st[1].data_ptr()
                e.steps[k].shift = st[2].data_ptr()
            else:
                e.steps[k].kind = _capi.EPI_ACTIVATION
                e.steps[k].act = st[1]
        return e


def _epi(e: Epilogue | None) -> _capi.Epilogue:
    return (e or Epilogue()).struct()


# ------------------------------------------------------------ masks ------

def compute_difference_mask(original: torch.Tensor, edited: torch.Tensor, threshold: float) -> torch.Tensor:
    """mask.hpp:31-32 — (H, W) uint8, 1 where max_{n,c} |edited - original| > threshold."""
    o = _dev(original, torch.float32, "compute_difference_mask")
    e = _dev(edited, torch.float32, "compute_difference_mask")
    if o.shape != e.shape or o.dim() != 4:
        raise ConfigError(f"compute_difference_mask: shape mismatch {tuple(o.shape)} vs {tuple(e.shape)}")
    n, c, h, w = o.shape
    m = torch.empty((h, w), dtype=torch.uint8, device=o.device)
    _check(_lib().sige_compute_difference_mask(o.data_ptr(), e.data_ptr(), n, c, h, w, threshold, m.data_ptr(), _stream()))
    return m


def downsample_mask(mask: torch.Tensor, out_h: int, out_w: int) -> torch.Tensor:
    m = _dev(mask, torch.uint8, "downsample_mask")
    out = torch.empty((max(out_h, 1), max(out_w, 1)), dtype=torch.uint8, device=m.device)
    _check(_lib().sige_downsample_mask(m.data_ptr(), m.shape[0], m.shape[1], out_h, out_w, out.data_ptr(), _stream()))
    return out


def dilate_mask(mask: torch.Tensor, radius: int) -> torch.Tensor:
    m = _dev(mask, torch.uint8, "dilate_mask")
    out = torch.empty_like(m)
    _check(_lib().sige_dilate_mask(m.data_ptr(), m.shape[0], m.shape[1], radius, out.data_ptr(), _stream()))
    return out


def mask_to_block_indices(mask: torch.Tensor, block_size: int, batch: int = 1) -> torch.Tensor:
    """mask.hpp:62-63 — (G, 3) int32 {n, r, c}, tiles row-major then n-major."""
    m = _dev(mask, torch.uint8, "mask_to_block_indices")
    h, w = m.shape
    b = max(block_size, 1)
    cap = ((h + b - 1) // b) * ((w + b - 1) // b) * max(batch, 1)
    idx = torch.empty((max(cap, 1), 3), dtype=torch.int32, device=m.device)
    cnt = C.c_int(0)
    _check(_lib().sige_mask_to_block_indices(m.data_ptr(), h, w, block_size, batch, idx.data_ptr(), cap, C.byref(cnt), _stream()))
    return idx[: cnt.value]


# ----------------------------------------------------------- blocks ------

def _conv_out(n: int, k: int, s: int) -> int:
    return (n + 2 * ((k - 1) // 2) - k) // s + 1


def gather(x: torch.Tensor, idx: torch.Tensor, block_size: int, k: int, stride: int,
           epilogue: Epilogue | None = None, idx_hw: tuple[int, int] | None = None) -> torch.Tensor:
    """kernels.hpp:48-49 — (G, C, win, win), win = s*b + k - s."""
    x = _dev(x, torch.float32, "gather")
    idx = _dev(idx, torch.int32, "gather")
    n, c, h, w = x.shape
    ih, iw = idx_hw or (_conv_out(h, k, stride), _conv_out(w, k, stride))
    win = stride * block_size + k - stride
    out = torch.empty((idx.shape[0], c, max(win, 1), max(win, 1)), dtype=torch.float32, device=x.device)
    e = _epi(epilogue)
    _check(_lib().sige_gather(x.data_ptr(), n, c, h, w, idx.data_ptr(), idx.shape[0], block_size, ih, iw, k, stride, C.byref(e), out.data_ptr(), _stream()))
    return out


ACT_LEAKY_RELU = 3  # SPADE blocks only (include/sige_b200.h)


def gather_spade(x: torch.Tensor, gamma: torch.Tensor, beta: torch.Tensor, idx: torch.Tensor, block_size: int,
                 k: int, stride: int, norm: Epilogue | None = None, act: int = 0,
                 idx_hw: tuple[int, int] | None = None) -> torch.Tensor:
    """SPADE modulation gather (config 3; not a reference function, restated in
    orc_gather_spade): window cells -> norm chain -> v * (1 + gamma) + beta -> act."""
    x = _dev(x, torch.float32, "gather_spade")
    gamma = _dev(gamma, torch.float32, "gather_spade")
    beta = _dev(beta, torch.float32, "gather_spade")
    if gamma.shape != x.shape or beta.shape != x.shape:
        raise ConfigError("gather_spade: gamma/beta must have the shape of x")
    idx = _dev(idx, torch.int32, "gather_spade")
    n, c, h, w = x.shape
    ih, iw = idx_hw or (_conv_out(h, k, stride), _conv_out(w, k, stride))
    win = stride * block_size + k - stride
    out = torch.empty((idx.shape[0], c, max(win, 1), max(win, 1)), dtype=torch.float32, device=x.device)
    e = _epi(norm)
    _check(_lib().sige_gather_spade(x.data_ptr(), gamma.data_ptr(), beta.data_ptr(), n, c, h, w, idx.data_ptr(),
                                    idx.shape[0], block_size, ih, iw, k, stride, C.byref(e), act, out.data_ptr(),
                                    _stream()))
    return out


def resize_nearest(x: torch.Tensor, out_h: int, out_w: int) -> torch.Tensor:
    """Nearest resample by integer factors (config 3 label maps)."""
    x = _dev(x, torch.float32, "resize_nearest")
    n, c, h, w = x.shape
    out = torch.empty((n, c, out_h, out_w), dtype=torch.float32, device=x.device)
    _check(_lib().sige_resize_nearest(x.data_ptr(), n, c, h, w, out_h, out_w, out.data_ptr(), _stream()))
    return out


def _check_scatter(op: str, blocks: torch.Tensor, idx: torch.Tensor, base: torch.Tensor, idx_hw) -> None:
    """require_scatter_compatible (kernels.cpp:18-35): channels, index
    resolution (when the caller states it) and every block's sample in range."""
    n, c, h, w = base.shape
    if blocks.dim() != 4 or blocks.shape[2] != blocks.shape[3]:
        raise ConfigError(f"{op}: blocks must be overlap-free output tiles")
    if blocks.shape[1] != c:
        raise ConfigError(f"{op}: channel mismatch")
    if idx_hw is not None and tuple(idx_hw) != (h, w):
        raise ConfigError(f"{op}: index resolution {idx_hw[0]}x{idx_hw[1]} does not match tensor ({n}, {c}, {h}, {w})")
    if idx.shape[0]:
        lo, hi = int(idx[:, 0].min()), int(idx[:, 0].max())
        if lo < 0 or hi >= n:
            raise ConfigError(f"{op}: block sample out of range")


def scatter_inplace(blocks: torch.Tensor, idx: torch.Tensor, base: torch.Tensor, idx_hw=None) -> None:
    """kernels.hpp:54 — idx_hw: the index set's resolution (BlockIndexSet::h, w), checked when given."""
    b = _dev(blocks, torch.float32, "scatter")
    i = _dev(idx, torch.int32, "scatter")
    if not base.is_contiguous():
        raise ConfigError("scatter: base must be contiguous")
    _check_scatter("scatter", b, i, base, idx_hw)
    _check(_lib().sige_scatter_inplace(b.data_ptr(), i.shape[0], b.shape[1], b.shape[2], i.data_ptr(), base.data_ptr(), *base.shape, _stream()))


def scatter(blocks: torch.Tensor, idx: torch.Tensor, base: torch.Tensor, idx_hw=None) -> torch.Tensor:
    """kernels.hpp:53."""
    out = torch.empty_like(_dev(base, torch.float32, "scatter"))
    b = _dev(blocks, torch.float32, "scatter")
    i = _dev(idx, torch.int32, "scatter")
    _check_scatter("scatter", b, i, base, idx_hw)
    _check(_lib().sige_scatter(b.data_ptr(), i.shape[0], b.shape[1], b.shape[2], i.data_ptr(), base.contiguous().data_ptr(), out.data_ptr(), *out.shape, _stream()))
    return out


def scatter_add_inplace(blocks: torch.Tensor, idx: torch.Tensor, base: torch.Tensor, idx_hw=None) -> None:
    """kernels.hpp:57."""
    b = _dev(blocks, torch.float32, "scatter_add")
    i = _dev(idx, torch.int32, "scatter_add")
    if not base.is_contiguous():
        raise ConfigError("scatter_add: base must be contiguous")
    _check_scatter("scatter_add", b, i, base, idx_hw)
    _check(_lib().sige_scatter_add_inplace(b.data_ptr(), i.shape[0], b.shape[1], b.shape[2], i.data_ptr(), base.data_ptr(), *base.shape, _stream()))


def build_scatter_map(idx: torch.Tensor, block_size: int, h: int, w: int):
    """kernels.hpp:77 — ((H, W, 2) int32 view of {block, dy|dx<<16}, blocks_per_sample)."""
    i = _dev(idx, torch.int32, "build_scatter_map")
    m = torch.empty((h, w, 2), dtype=torch.int32, device=i.device)
    bps = C.c_int(0)
    _check(_lib().sige_build_scatter_map(i.data_ptr(), i.shape[0], block_size, h, w, m.data_ptr(), C.byref(bps), _stream()))
    return m, bps.value


def block_index_hash(idx: torch.Tensor, block_size: int, h: int, w: int) -> int:
    """BlockIndexSet::content_hash (mask.cpp:91-101) of a device index set."""
    i = _dev(idx, torch.int32, "content_hash")
    out = C.c_uint64(0)
    _check(_lib().sige_block_index_hash(i.data_ptr(), i.shape[0], block_size, h, w, C.byref(out), _stream()))
    return out.value


class DeviceScatterMap:
    """A cache-owned device scatter map (valid until ScatterMapCache.clear());
    unpacks like build_scatter_map's (map, blocks_per_sample)."""

    def __init__(self, ptr: int, bps: int, key: int, h: int, w: int):
        self.ptr, self.bps, self.key, self.h, self.w = ptr, bps, key, h, w

    def data_ptr(self) -> int:
        return self.ptr

    def __iter__(self):
        return iter((self, self.bps))


class ScatterMapCache:
    """ScatterMapCache (kernels.hpp:80-91): process-wide memo of device scatter
    maps keyed by the index set's content hash."""

    _inst = None

    @classmethod
    def instance(cls) -> "ScatterMapCache":
        if cls._inst is None:
            cls._inst = cls()
        return cls._inst

    def get(self, idx: torch.Tensor, block_size: int, h: int, w: int) -> DeviceScatterMap:
        i = _dev(idx, torch.int32, "ScatterMapCache::get")
        p, bps, key = C.c_void_p(), C.c_int(0), C.c_uint64(0)
        _check(_lib().sige_scatter_map_cache_get(i.data_ptr(), i.shape[0], block_size, h, w, C.byref(p),
                                                 C.byref(bps), C.byref(key), _stream()))
        return DeviceScatterMap(p.value, bps.value, key.value, h, w)

    def size(self) -> int:
        return int(_lib().sige_scatter_map_cache_size())

    def clear(self) -> None:
        _lib().sige_scatter_map_cache_clear()


def scatter_gather(blocks: torch.Tensor, original_out: torch.Tensor, scatter_map, consumer_idx: torch.Tensor,
                   consumer_block: int, k: int, stride: int, epilogue: Epilogue | None = None) -> torch.Tensor:
    """kernels.hpp:98-100."""
    b = _dev(blocks, torch.float32, "scatter_gather")
    o = _dev(original_out, torch.float32, "scatter_gather")
    ci = _dev(consumer_idx, torch.int32, "scatter_gather")
    m, bps = scatter_map
    n, c, h, w = o.shape
    win = stride * consumer_block + k - stride
    out = torch.empty((ci.shape[0], c, win, win), dtype=torch.float32, device=o.device)
    e = _epi(epilogue)
    _check(_lib().sige_scatter_gather(b.data_ptr(), b.shape[0], b.shape[2], o.data_ptr(), n, c, h, w, m.data_ptr(), bps,
                                      ci.data_ptr(), ci.shape[0], consumer_block, _conv_out(h, k, stride), _conv_out(w, k, stride),
                                      k, stride, C.byref(e), out.data_ptr(), _stream()))
    return out


def _residual(fn, main_blocks, main_idx, shortcut_blocks, shortcut_idx, precomputed_sum, original_shortcut):
    mb = _dev(main_blocks, torch.float32, "block_residual")
    sb = _dev(shortcut_blocks, torch.float32, "block_residual")
    mi = _dev(main_idx, torch.int32, "block_residual")
    si = _dev(shortcut_idx, torch.int32, "block_residual")
    s = _dev(precomputed_sum, torch.float32, "block_residual")
    o = _dev(original_shortcut, torch.float32, "block_residual")
    # require_join_compatible (kernels.cpp:276-287)
    _check_scatter("block_residual(main)", mb, mi, s, None)
    _check_scatter("block_residual(shortcut)", sb, si, s, None)
    if s.shape != o.shape:
        raise ConfigError("block_residual: shape mismatch")
    out = torch.empty_like(s)
    _check(fn(mb.data_ptr(), mi.shape[0], mb.shape[2], mi.data_ptr(), sb.data_ptr(), si.shape[0], sb.shape[2], si.data_ptr(),
              s.data_ptr(), o.data_ptr(), out.data_ptr(), *s.shape, _stream()))
    return out


def scatter_with_block_residual(main_blocks, main_idx, shortcut_blocks, shortcut_idx, precomputed_sum, original_shortcut):
    """kernels.hpp:107-110."""
    return _residual(_lib().sige_scatter_with_block_residual, main_blocks, main_idx, shortcut_blocks, shortcut_idx, precomputed_sum, original_shortcut)


def scatter_with_block_residual_unfused(main_blocks, main_idx, shortcut_blocks, shortcut_idx, precomputed_sum, original_shortcut):
    """kernels.hpp:115-118."""
    return _residual(_lib().sige_scatter_with_block_residual_unfused, main_blocks, main_idx, shortcut_blocks, shortcut_idx, precomputed_sum, original_shortcut)


def _combine(a, b, sign):
    a = _dev(a, torch.float32, "combine_blocks")
    b = _dev(b, torch.float32, "combine_blocks")
    if a.shape != b.shape:
        raise ConfigError("add_blocks: block stack geometry mismatch" if sign > 0 else "subtract_blocks: block stack geometry mismatch")
    out = torch.empty_like(a)
    _check(_lib().sige_combine_blocks(a.data_ptr(), b.data_ptr(), sign, a.numel(), out.data_ptr(), _stream()))
    return out


def add_blocks(a, b):
    return _combine(a, b, 1.0)


def subtract_blocks(a, b):
    return _combine(a, b, -1.0)


def apply_epilogue_on_blocks(blocks: torch.Tensor, idx: torch.Tensor, epilogue: Epilogue) -> None:
    b = _dev(blocks, torch.float32, "apply_epilogue_on_blocks")
    i = _dev(idx, torch.int32, "apply_epilogue_on_blocks")
    e = _epi(epilogue)
    _check(_lib().sige_apply_epilogue_on_blocks(b.data_ptr(), b.shape[0], b.shape[1], b.shape[2], i.data_ptr(), C.byref(e), _stream()))
    if b.data_ptr() != blocks.data_ptr():
        blocks.copy_(b)


def _conv_desc(weight: torch.Tensor, bias: torch.Tensor | None, stride: int):
    w = _dev(weight, torch.float32, "conv")
    b = _dev(bias, torch.float32, "conv") if bias is not None else None
    cd = _capi.ConvDesc(w.shape[1], w.shape[0], w.shape[2], stride, w.data_ptr(), b.data_ptr() if b is not None else None)
    return cd, (w, b)


def conv_on_blocks(blocks: torch.Tensor, weight: torch.Tensor, bias: torch.Tensor | None, stride: int, block: int,
                   with_bias: bool = True, math: int = MATH_EXACT) -> torch.Tensor:
    """kernels.hpp:130-131."""
    x = _dev(blocks, torch.float32, "conv_on_blocks")
    cd, keep = _conv_desc(weight, bias, stride)
    out = torch.empty((x.shape[0], cd.c_out, block, block), dtype=torch.float32, device=x.device)
    _check(_lib().sige_conv_on_blocks(x.data_ptr(), x.shape[0], x.shape[2], C.byref(cd), int(with_bias), math, out.data_ptr(), block, _stream()))
    return out


def conv2d(x: torch.Tensor, weight: torch.Tensor, bias: torch.Tensor | None, stride: int = 1,
           with_bias: bool = True, math: int = MATH_EXACT) -> torch.Tensor:
    """conv.hpp:35 — zero padding (k-1)/2."""
    x = _dev(x, torch.float32, "conv2d")
    cd, keep = _conv_desc(weight, bias, stride)
    n, c, h, w = x.shape
    out = torch.empty((n, cd.c_out, _conv_out(h, cd.k, stride), _conv_out(w, cd.k, stride)), dtype=torch.float32, device=x.device)
    _check(_lib().sige_conv2d(x.data_ptr(), n, c, h, w, C.byref(cd), int(with_bias), math, out.data_ptr(), _stream()))
    return out


# ----------------------------------------------------------- inputs ------

def make_edit_fixture(kind: str, n: int, c: int, h: int, w: int, seed: int):
    """fixtures.hpp:23-24 — (original, edited) host float32 tensors."""
    o = torch.empty((n, c, h, w), dtype=torch.float32)
    e = torch.empty((n, c, h, w), dtype=torch.float32)
    _check(_lib().sige_make_edit_fixture(kind.encode(), n, c, h, w, seed, o.data_ptr(), e.data_ptr()))
    return o, e


def make_seg_fixture(n: int, label_nc: int, h: int, w: int, seed: int):
    """Config 3: one-hot segmentation map and its edit (a relabelled 1.2 % square), host float32."""
    o = torch.empty((n, label_nc, h, w), dtype=torch.float32)
    e = torch.empty((n, label_nc, h, w), dtype=torch.float32)
    _check(_lib().sige_make_seg_fixture(n, label_nc, h, w, seed, o.data_ptr(), e.data_ptr()))
    return o, e


# ------------------------------------------------ on-disk formats (io.hpp) --

def save_tensor(path: str, t: torch.Tensor) -> None:
    """io.hpp:14 — SIGT v1 file of a 4-D float32 tensor (host copy taken)."""
    t = t.detach().to("cpu", torch.float32).contiguous()
    if t.dim() != 4:
        raise ConfigError("save_tensor: expected a 4-D tensor")
    _check(_lib().sige_save_tensor(str(path).encode(), t.data_ptr(), *t.shape))


def load_tensor(path: str) -> torch.Tensor:
    """io.hpp:15 — host float32 (n, c, h, w) tensor."""
    dims = (C.c_int * 4)()
    _check(_lib().sige_load_tensor(str(path).encode(), None, 0, dims))
    t = torch.empty(tuple(dims), dtype=torch.float32)
    _check(_lib().sige_load_tensor(str(path).encode(), t.data_ptr(), t.numel(), dims))
    return t


def save_mask_pbm(path: str, mask: torch.Tensor) -> None:
    """io.hpp:18 — plain PBM (P1) of an (h, w) uint8 mask."""
    m = mask.detach().to("cpu", torch.uint8).contiguous()
    _check(_lib().sige_save_mask_pbm(str(path).encode(), m.data_ptr(), *m.shape))


def load_mask_pbm(path: str) -> torch.Tensor:
    """io.hpp:19 — host (h, w) uint8 mask."""
    h, w = C.c_int(0), C.c_int(0)
    _check(_lib().sige_load_mask_pbm(str(path).encode(), None, 0, C.byref(h), C.byref(w)))
    m = torch.empty((h.value, w.value), dtype=torch.uint8)
    _check(_lib().sige_load_mask_pbm(str(path).encode(), m.data_ptr(), m.numel(), C.byref(h), C.byref(w)))
    return m


def save_block_stack(prefix: str, blocks: torch.Tensor, idx: torch.Tensor, block: int, overlap: int,
                     origin_hw: tuple[int, int], origin_block: int | None = None) -> None:
    """io.hpp:33 — <prefix>.sigt + <prefix>.json (sige_blocks_v1)."""
    b = blocks.detach().to("cpu", torch.float32).contiguous()
    i = idx.detach().to("cpu", torch.int32).contiguous()
    g = int(i.shape[0])
    ch = int(b.shape[1]) if b.dim() == 4 else 0
    _check(_lib().sige_save_block_stack(str(prefix).encode(), b.data_ptr(), g, ch, block, overlap,
                                        block if origin_block is None else origin_block, origin_hw[0],
                                        origin_hw[1], i.data_ptr()))


def load_block_stack(prefix: str) -> dict:
    """io.hpp:34 — {blocks (G, C, bh, bh), idx (G, 3), block, overlap, origin_block, origin_hw}."""
    meta = (C.c_int * 7)()
    _check(_lib().sige_load_block_stack(str(prefix).encode(), None, 0, None, 0, meta))
    g, ch, block, overlap = meta[0], meta[1], meta[2], meta[3]
    bh = block + overlap
    blocks = torch.empty((g, ch, bh, bh), dtype=torch.float32)
    idx = torch.empty((g, 3), dtype=torch.int32)
    _check(_lib().sige_load_block_stack(str(prefix).encode(), blocks.data_ptr(), blocks.numel(), idx.data_ptr(),
                                        idx.numel(), meta))
    return {"blocks": blocks, "idx": idx, "block": block, "overlap": overlap, "origin_block": meta[4],
            "origin_hw": (meta[5], meta[6])}


class Model:
    """A model description (graph.hpp:63-71): a named synthetic model or a
    ModelDesc pointer supplied by the caller (kept alive by ``owner``)."""

    def __init__(self, name_or_desc, owner=None):
        self._own = False
        if isinstance(name_or_desc, str):
            p = C.POINTER(_capi.ModelDesc)()
            _check(_lib().sige_model_build(name_or_desc.encode(), C.byref(p)))
            self.desc = p
            self._own = True
        else:
            self.desc = name_or_desc
        self.owner = owner

    def __del__(self):
        try:
            if self._own:
                _lib().sige_model_free(self.desc)
        except Exception:
            pass

    @property
    def name(self) -> str:
        return self.desc.contents.name.decode()

    @property
    def in_shape(self):
        d = self.desc.contents
        return d.in_channels, d.in_h, d.in_w

    def weight_hash(self) -> int:
        return int(_lib().sige_model_weight_hash(self.desc))

    def structure_hash(self) -> int:
        """ModelSpec::structure_hash (graph.cpp:89-127)."""
        return int(_lib().sige_model_structure_hash(self.desc))

    def required_dilation(self) -> int:
        v = C.c_int(0)
        _check(_lib().sige_model_required_dilation(self.desc, C.byref(v)))
        return v.value


class Engine:
    """Device ActivationCache + sparse executor (graph.hpp:116-226)."""

    def __init__(self, model: Model, batch: int = 1, math: int = MATH_TF32):
        self.model = model
        self.batch = batch
        self.math = math
        h = C.c_void_p()
        _check(_lib().sige_engine_create(model.desc, batch, math, C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h:
                _lib().sige_engine_destroy(self.h)
        except Exception:
            pass

    def output_shape(self):
        n, c, h, w = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(_lib().sige_engine_output_shape(self.h, C.byref(n), C.byref(c), C.byref(h), C.byref(w)))
        return n.value, c.value, h.value, w.value

    def precompute(self, original: torch.Tensor, step: int = 0) -> None:
        o = self._check_input(original, "precompute")
        _check(_lib().sige_engine_precompute(self.h, o.data_ptr(), step, _stream()))

    def output_coverage(self, edited: torch.Tensor | None = None, mask: torch.Tensor | None = None,
                        config: RunConfig | None = None) -> torch.Tensor:
        """output_coverage (graph.cpp:1078-1129) of an edit on the device: (out_h, out_w) uint8."""
        e = self._check_input(edited, "output_coverage") if edited is not None else None
        m = self._check_mask(mask, "output_coverage") if mask is not None else None
        _, oc, oh, ow = self.output_shape()
        dev = (e if e is not None else m).device
        out = torch.empty((oh, ow), dtype=torch.uint8, device=dev)
        h, w = C.c_int(0), C.c_int(0)
        cfg = config or default_config()
        _check(_lib().sige_engine_output_coverage(self.h, e.data_ptr() if e is not None else None,
                                                  m.data_ptr() if m is not None else None, C.byref(cfg),
                                                  out.data_ptr(), C.byref(h), C.byref(w), _stream()))
        return out

    def offload_step(self, step: int) -> None:
        """Move one step's cache entries to pinned host memory, freeing their device memory."""
        _check(_lib().sige_engine_offload_step(self.h, step, _stream()))

    def prefetch_step(self, step: int) -> None:
        """Upload an offloaded step again, asynchronously on the current stream."""
        _check(_lib().sige_engine_prefetch_step(self.h, step, _stream()))

    def drop_step(self, step: int) -> None:
        """ActivationCache::drop_step (graph.cpp:271-274): erase (and free) one step's entries."""
        _check(_lib().sige_engine_drop_step(self.h, step))

    def refresh_step(self, original: torch.Tensor, step: int) -> None:
        """refresh_step (graph.cpp:437-444): replace one step's entries from a new original."""
        o = self._check_input(original, "precompute")
        _check(_lib().sige_engine_refresh_step(self.h, o.data_ptr(), step, _stream()))

    def cache_model_hash(self) -> tuple[int, int]:
        """(hash of the model the cache was built for, hash of the engine's model)."""
        c, m = C.c_uint64(0), C.c_uint64(0)
        _check(_lib().sige_engine_cache_model_hash(self.h, C.byref(c), C.byref(m)))
        return c.value, m.value

    def set_cache_model_hash(self, h: int) -> None:
        """Declare the producer model of an imported cache (ActivationCache::set_model_hash)."""
        _check(_lib().sige_engine_set_cache_model_hash(self.h, C.c_uint64(h)))

    def put_tensor(self, key: str, host_nchw, step: int = 0) -> None:
        t = torch.as_tensor(host_nchw, dtype=torch.float32).contiguous().cpu()
        _check(_lib().sige_engine_put_tensor(self.h, step, key.encode(), t.data_ptr(), t.numel()))

    def put_norm(self, key: str, scale, shift, step: int = 0) -> None:
        s = torch.as_tensor(scale, dtype=torch.float32).contiguous().cpu()
        t = torch.as_tensor(shift, dtype=torch.float32).contiguous().cpu()
        _check(_lib().sige_engine_put_norm(self.h, step, key.encode(), s.data_ptr(), t.data_ptr(), s.numel()))

    def get_tensor(self, key: str, shape, step: int = 0) -> torch.Tensor:
        out = torch.empty(shape, dtype=torch.float32)
        _check(_lib().sige_engine_get_tensor(self.h, step, key.encode(), out.data_ptr(), out.numel()))
        return out

    def get_norm(self, key: str, count: int, step: int = 0):
        sc = torch.empty(count, dtype=torch.float32)
        sh = torch.empty(count, dtype=torch.float32)
        _check(_lib().sige_engine_get_norm(self.h, step, key.encode(), sc.data_ptr(), sh.data_ptr(), count))
        return sc, sh

    def _in_shape(self):
        c, h, w = self.model.in_shape
        return (self.batch, c, h, w)

    def _check_input(self, x: torch.Tensor, name: str, device: bool = True) -> torch.Tensor:
        """check_inputs / dense_walk (graph.cpp:348-352,606-614): the edited
        input must be (batch, in_channels, H, W) float32."""
        if not isinstance(x, torch.Tensor):
            raise ConfigError(f"{name}: expected a tensor")
        if device and not x.is_cuda:
            raise ConfigError(f"{name}: expected a CUDA tensor")
        if not device and x.is_cuda:
            raise ConfigError(f"{name}: expected a host tensor")
        if x.dtype != torch.float32:
            raise ConfigError(f"{name}: expected torch.float32, got {x.dtype}")
        want = self._in_shape()
        if x.dim() != 4:
            raise ConfigError(f"{name}: expected a 4-D (n, c, h, w) tensor")
        if x.shape[1] != want[1]:
            if name in ("precompute", "dense_forward"):  # dense_walk (graph.cpp:348-352)
                raise ConfigError(f"forward: input has {x.shape[1]} channels, model expects {want[1]}")
            raise ConfigError("forward: input channel mismatch")  # check_inputs (graph.cpp:606-609)
        if tuple(x.shape) != want:
            raise ConfigError(f"{name}: input is {tuple(x.shape)}, engine expects {want}")
        return x.contiguous()

    def _check_mask(self, m: torch.Tensor | None, name: str, device: bool = True) -> torch.Tensor | None:
        if m is None:
            return None
        if not isinstance(m, torch.Tensor) or m.is_cuda != device:
            raise ConfigError(f"{name}: mask must be a {'CUDA' if device else 'host'} tensor")
        if m.dtype != torch.uint8:
            raise ConfigError(f"{name}: mask must be torch.uint8, got {m.dtype}")
        _, _, h, w = self._in_shape()
        if m.dim() != 2 or tuple(m.shape) != (h, w):
            mh, mw = (tuple(m.shape) + (0, 0))[:2]
            raise ConfigError(f"forward: mask is {mh}x{mw} but input is {h}x{w}")
        return m.contiguous()

    def _check_out(self, out: torch.Tensor | None, like: torch.Tensor, name: str) -> torch.Tensor:
        shape = self.output_shape()
        if out is None:
            return torch.empty(shape, dtype=torch.float32, device=like.device)
        if (not isinstance(out, torch.Tensor) or out.dtype != torch.float32 or tuple(out.shape) != shape
                or out.device != like.device or not out.is_contiguous()):
            raise ConfigError(f"{name}: out must be a contiguous float32 tensor of shape {shape} on {like.device}")
        return out

    def sparse_forward(self, edited: torch.Tensor, mask: torch.Tensor | None = None,
                       config: RunConfig | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
        """sparse_forward (graph.hpp:224-226) on device buffers."""
        e = self._check_input(edited, "sparse_forward")
        m = self._check_mask(mask, "sparse_forward")
        if m is not None and m.device != e.device:
            raise ConfigError("sparse_forward: mask and input on different devices")
        out = self._check_out(out, e, "sparse_forward")
        cfg = config or default_config()
        _check(_lib().sige_engine_sparse_forward(self.h, e.data_ptr(), m.data_ptr() if m is not None else None,
                                                 C.byref(cfg), out.data_ptr(), _stream()))
        return out

    def sparse_forward_grouped(self, edited: torch.Tensor, masks: torch.Tensor | None = None,
                               config: RunConfig | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
        """Independent requests, one per batch sample (own original, edit and
        mask; masks: (batch, H, W) uint8 or None), served by one launch per layer."""
        e = self._check_input(edited, "sparse_forward_grouped")
        m = None
        if masks is not None:
            _, _, h, w = self._in_shape()
            if (not isinstance(masks, torch.Tensor) or not masks.is_cuda or masks.dtype != torch.uint8
                    or tuple(masks.shape) != (self.batch, h, w)):
                raise ConfigError(f"sparse_forward_grouped: masks must be a CUDA uint8 tensor of shape "
                                  f"{(self.batch, h, w)}")
            m = masks.contiguous()
        out = self._check_out(out, e, "sparse_forward_grouped")
        cfg = config or default_config()
        _check(_lib().sige_engine_sparse_forward_grouped(self.h, e.data_ptr(), m.data_ptr() if m is not None else None,
                                                         C.byref(cfg), out.data_ptr(), _stream()))
        return out

    def sparse_forward_host(self, edited_host: torch.Tensor, mask_host: torch.Tensor | None = None,
                            config: RunConfig | None = None, out_host: torch.Tensor | None = None) -> torch.Tensor:
        """The host-buffer entry point (H2D, sparse_forward, D2H, synchronise)."""
        e = self._check_input(edited_host, "sparse_forward_host", device=False)
        m = self._check_mask(mask_host, "sparse_forward_host", device=False)  # kept alive across the call
        shape = self.output_shape()
        if out_host is None:
            out_host = torch.empty(shape, dtype=torch.float32)
        elif (out_host.is_cuda or out_host.dtype != torch.float32 or tuple(out_host.shape) != shape
              or not out_host.is_contiguous()):
            raise ConfigError(f"sparse_forward_host: out_host must be a contiguous host float32 tensor of shape {shape}")
        cfg = config or default_config()
        _check(_lib().sige_engine_sparse_forward_host(self.h, e.data_ptr(), m.data_ptr() if m is not None else None,
                                                      C.byref(cfg), out_host.data_ptr(), _stream()))
        return out_host

    def dense_forward(self, x: torch.Tensor, reused_stats: bool = False, step: int = 0) -> torch.Tensor:
        x = self._check_input(x, "dense_forward")
        out = torch.empty(self.output_shape(), dtype=torch.float32, device=x.device)
        _check(_lib().sige_engine_dense_forward(self.h, x.data_ptr(), int(reused_stats), step, out.data_ptr(), _stream()))
        return out

    def last_launch_count(self) -> int:
        return int(_lib().sige_engine_last_launch_count(self.h))

    def trace(self, cap: int = 1024):
        rows = torch.zeros((cap, 6), dtype=torch.int64)
        n = C.c_int(0)
        _check(_lib().sige_engine_trace(self.h, rows.data_ptr(), cap, C.byref(n), _stream()))
        return rows[: n.value].clone()

    def set_sm_budget(self, sms: int) -> None:
        """Launch grids sized for `sms` SMs (0 = all): several engines in flight share the GPU."""
        _check(_lib().sige_engine_set_sm_budget(self.h, int(sms)))

    def set_graphs(self, on: bool) -> None:
        _check(_lib().sige_engine_set_graphs(self.h, int(on)))

    def set_profiling(self, on: bool) -> None:
        _check(_lib().sige_engine_set_profiling(self.h, int(on)))

    def profile_read(self, cap: int = 4096):
        """[(ms, flops, tensor_core)] of the fused conv launches since the last read."""
        rows = torch.zeros((cap, 3), dtype=torch.float64)
        n = C.c_int(0)
        _check(_lib().sige_engine_profile_read(self.h, rows.data_ptr(), cap, C.byref(n), _stream()))
        return rows[: n.value].clone()

    def set_timeline(self, on: bool) -> None:
        """Device %globaltimer stamps of every tensor-core conv launch (inside replayed graphs)."""
        _check(_lib().sige_engine_set_timeline(self.h, int(on)))

    def timeline_read(self, cap: int = 1024):
        """[(start_ns, end_ns, wait_ns, flops, sparse)] of the last call's conv launches, then reset."""
        rows = torch.zeros((cap, 5), dtype=torch.float64)
        n = C.c_int(0)
        _check(_lib().sige_engine_timeline_read(self.h, rows.data_ptr(), cap, C.byref(n)))
        return rows[: min(n.value, cap)].clone()

    def cache_entries(self, step: int = 0):
        """[("T", key, (n, c, h, w)) | ("N", key, count)] of the device cache."""
        need = C.c_size_t(0)
        _check(_lib().sige_engine_cache_entries(self.h, step, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        _check(_lib().sige_engine_cache_entries(self.h, step, buf, need.value, C.byref(need)))
        out = []
        for line in buf.value.decode().splitlines():
            f = line.split()
            if f[0] == "T":
                out.append(("T", f[1], tuple(int(v) for v in f[2:6])))
            else:
                out.append(("N", f[1], int(f[2])))
        return out

    def cache_bytes(self) -> int:
        return int(_lib().sige_engine_cache_bytes(self.h))
