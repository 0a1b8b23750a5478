"""TEST INFRASTRUCTURE ONLY — parity oracles for the SIGE sparse-update path.

Two checkers with one Python face:

* ``ORC``  — ``oracle/_build/liboracle.so``, the plain-C restatement of the
  reference (``oracle/sige_oracle.c``; every function cites the reference
  file:line it follows).
* ``REF``  — ``oracle/_ref/libsigeref.so``, the UNMODIFIED reference library
  compiled from ``/root/reference/proj/src`` by ``oracle/Makefile`` (with an
  extern "C" veneer, ``oracle/ref_shim.cpp``). Present wherever ``build()``
  ran with ``/root/reference`` mounted; the prebuilt .so travels to the GPU box.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package. The product path never does.
"""
from __future__ import annotations

import ctypes as C
import pathlib

import numpy as np

from paper_2211_02048_b200._capi import (
    ConvDesc,
    Epilogue,
    ModelDesc,
    RunConfig,
    ScatterEntry,
    default_config,
)

HERE = pathlib.Path(__file__).resolve().parent
ORC_PATH = HERE / "_build" / "liboracle.so"
REF_PATH = HERE / "_ref" / "libsigeref.so"

_vp, _i, _f, _sz, _u32, _u64 = C.c_void_p, C.c_int, C.c_float, C.c_size_t, C.c_uint32, C.c_uint64


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _ptr(a) -> int:
    if a is None:
        return None
    return a.ctypes.data


def epilogue_struct(steps, keep: list) -> Epilogue:
    """steps: list of ("ss", scale, shift) | ("act", kind). Host (numpy) params."""
    e = Epilogue()
    e.num_steps = len(steps)
    for k, st in enumerate(steps):
        if st[0] == "ss":
            sc = np.ascontiguousarray(st[1], dtype=np.float32)
            sh = np.ascontiguousarray(st[2], dtype=np.float32)
            keep += [sc, sh]
            e.steps[k].kind = 0
            e.steps[k].nparams = sc.size
            e.steps[k].scale = sc.ctypes.data
            e.steps[k].shift = sh.ctypes.data
        else:
            e.steps[k].kind = 1
            e.steps[k].act = int(st[1])
    return e


def conv_struct(weight, bias, k, stride, keep: list) -> ConvDesc:
    w = np.ascontiguousarray(weight, dtype=np.float32)
    keep.append(w)
    b = None
    if bias is not None:
        b = np.ascontiguousarray(bias, dtype=np.float32)
        keep.append(b)
    c_out, c_in = w.shape[0], w.shape[1]
    return ConvDesc(c_in, c_out, k, stride, w.ctypes.data, b.ctypes.data if b is not None else None)


class _Impl:
    """Uniform numpy API over liboracle (prefix orc_) or libsigeref (ref_)."""

    def __init__(self, path: pathlib.Path, prefix: str):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (run __graft_entry__.build())")
        self.lib = C.CDLL(str(path))
        self.p = prefix
        L, p = self.lib, prefix
        sig = {
            "last_error": (C.c_char_p, []),
            "fnv1a64": (_u64, [_vp, _sz, _u64]),
            "rng_stream": (_i, [_u32, _i, _vp, _vp, _f, _f]),
            "expf": (_f, [_f]),
            "make_edit_fixture": (_i, [C.c_char_p, _i, _i, _i, _i, _u32, _vp, _vp]),
            "compute_difference_mask": (_i, [_vp, _vp, _i, _i, _i, _i, _f, _vp]),
            "downsample_mask": (_i, [_vp, _i, _i, _i, _i, _vp]),
            "dilate_mask": (_i, [_vp, _i, _i, _i, _vp]),
            "mask_to_block_indices": (_i, [_vp, _i, _i, _i, _i, _vp, _i, C.POINTER(_i), C.POINTER(_u64)]),
            "gather": (_i, [_vp, _i, _i, _i, _i, _vp, _i, _i, _i, _i, _i, _i, C.POINTER(Epilogue), _vp]),
            "scatter": (_i, [_vp, _i, _i, _i, _vp, _vp, _vp, _i, _i, _i, _i]),
            "scatter_add_inplace": (_i, [_vp, _i, _i, _i, _vp, _vp, _i, _i, _i, _i]),
            "build_scatter_map": (_i, [_vp, _i, _i, _i, _i, _vp, C.POINTER(_i)]),
            "scatter_gather": (
                _i,
                [_vp, _i, _i, _vp, _vp, _i, _i, _i, _i, _vp, _i, _i, _i, _i, _i, _i, C.POINTER(Epilogue), _vp],
            ),
            "scatter_with_block_residual": (
                _i,
                [_vp, _i, _i, _vp, _vp, _i, _i, _vp, _vp, _vp, _vp, _i, _i, _i, _i, _i],
            ),
            "apply_epilogue_on_blocks": (_i, [_vp, _i, _i, _i, _vp, _i, _i, C.POINTER(Epilogue)]),
            "conv_on_blocks": (_i, [_vp, _i, _i, C.POINTER(ConvDesc), _i, _vp, _i]),
            "conv2d": (_i, [_vp, _i, _i, _i, _i, C.POINTER(ConvDesc), _i, _vp]),
            "group_norm_fold": (_i, [_vp, _i, _i, _i, _i, _i, _f, _vp, _vp, _vp, _vp]),
            "model_free": (None, [_vp]),
            "model_weight_hash": (_u64, [_vp]),
            "model_required_dilation": (_i, [_vp]),
            "model_output_shape": (_i, [_vp, C.POINTER(_i), C.POINTER(_i), C.POINTER(_i)]),
            "cache_precompute": (_vp, [_vp, _vp, _i, _i, _i, _i] + ([_i] if prefix == "ref_" else [])),
            "cache_free": (None, [_vp]),
            "cache_tensor": (_i, [_vp, _i, C.c_char_p, _vp, _sz, C.POINTER(_i * 4)]),
            "cache_norm": (_i, [_vp, _i, C.c_char_p, _vp, _vp, _sz, C.POINTER(_i)]),
            "cache_total_elements": (_u64, [_vp]),
            "sparse_forward": (
                _i,
                [_vp, _vp, _vp, _i, _i, _i, _i, _vp, C.POINTER(RunConfig), _vp, _vp, _i, C.POINTER(_i)],
            ),
            "dense_forward": (_i, [_vp, _vp, _i, _i, _i, _i, _vp]),
            "dense_forward_reused_stats": (_i, [_vp, _vp, _i, _i, _i, _i, _vp, _i, _vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, p + name)
            fn.restype = res
            fn.argtypes = args
        if prefix == "orc_":
            L.orc_model_build.restype = C.POINTER(ModelDesc)
            L.orc_model_build.argtypes = [C.c_char_p]
            L.orc_model_clone.restype = C.POINTER(ModelDesc)
            L.orc_model_clone.argtypes = [C.POINTER(ModelDesc)]
            L.orc_index_set_hash.restype = _u64
            L.orc_index_set_hash.argtypes = [_vp, _i, _i, _i, _i]
            L.orc_combine_blocks.restype = _i
            L.orc_combine_blocks.argtypes = [_vp, _vp, _f, _sz, _vp]
        else:
            L.ref_model_build.restype = _vp
            L.ref_model_build.argtypes = [C.c_char_p]
            L.ref_model_from_desc.restype = _vp
            L.ref_model_from_desc.argtypes = [C.POINTER(ModelDesc)]
            L.ref_expf_digest.restype = _u64
            L.ref_expf_digest.argtypes = [_u32, _u32]
            L.ref_output_coverage.restype = _i
            L.ref_output_coverage.argtypes = [_vp, _vp, _i, _i, _i, C.POINTER(RunConfig), _vp, C.POINTER(_i), C.POINTER(_i)]

    def fn(self, name):
        return getattr(self.lib, self.p + name)

    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self.fn("last_error")().decode())

    # ---- basics
    def fnv1a64(self, data: bytes | np.ndarray, seed: int = 1469598103934665603) -> int:
        a = np.frombuffer(bytes(data), dtype=np.uint8) if isinstance(data, (bytes, bytearray)) else np.ascontiguousarray(data)
        return int(self.fn("fnv1a64")(a.ctypes.data, a.nbytes, seed))

    def rng_stream(self, seed, count, lo=0.0, hi=1.0):
        u = np.zeros(count, np.uint32)
        f = np.zeros(count, np.float32)
        self.fn("rng_stream")(seed, count, u.ctypes.data, f.ctypes.data, lo, hi)
        return u, f

    def expf(self, x: float) -> float:
        return float(self.fn("expf")(x))

    def make_edit_fixture(self, kind, n, c, h, w, seed):
        o = np.zeros((n, c, h, w), np.float32)
        e = np.zeros((n, c, h, w), np.float32)
        self._check(self.fn("make_edit_fixture")(kind.encode(), n, c, h, w, seed, _ptr(o), _ptr(e)))
        return o, e

    # ---- masks
    def difference_mask(self, o, e, thr=1e-3):
        o = np.ascontiguousarray(o, np.float32)
        e = np.ascontiguousarray(e, np.float32)
        n, c, h, w = o.shape
        m = np.zeros((h, w), np.uint8)
        self._check(self.fn("compute_difference_mask")(_ptr(o), _ptr(e), n, c, h, w, thr, _ptr(m)))
        return m

    def downsample_mask(self, m, oh, ow):
        m = np.ascontiguousarray(m, np.uint8)
        out = np.zeros((oh, ow), np.uint8)
        self._check(self.fn("downsample_mask")(_ptr(m), m.shape[0], m.shape[1], oh, ow, _ptr(out)))
        return out

    def dilate_mask(self, m, r):
        m = np.ascontiguousarray(m, np.uint8)
        out = np.zeros_like(m)
        self._check(self.fn("dilate_mask")(_ptr(m), m.shape[0], m.shape[1], r, _ptr(out)))
        return out

    def mask_to_block_indices(self, m, b, batch=1):
        m = np.ascontiguousarray(m, np.uint8)
        h, w = m.shape
        cap = ((h + b - 1) // b) * ((w + b - 1) // b) * batch
        idx = np.zeros((max(cap, 1), 3), np.int32)
        cnt = _i(0)
        hs = _u64(0)
        self._check(self.fn("mask_to_block_indices")(_ptr(m), h, w, b, batch, _ptr(idx), cap, C.byref(cnt), C.byref(hs)))
        return idx[: cnt.value].copy(), int(hs.value)

    # ---- blocks
    def gather(self, x, idx, b, ih, iw, k, s, epi=None):
        x = np.ascontiguousarray(x, np.float32)
        idx = np.ascontiguousarray(idx, np.int32)
        n, c, h, w = x.shape
        win = s * b + k - s
        out = np.zeros((len(idx), c, win, win), np.float32)
        keep = []
        e = epilogue_struct(epi or [], keep)
        self._check(self.fn("gather")(_ptr(x), n, c, h, w, _ptr(idx), len(idx), b, ih, iw, k, s, C.byref(e), _ptr(out)))
        return out

    def gather_spade(self, x, gamma, beta, idx, b, ih, iw, k, s, norm=None, act=0):
        """SPADE modulation gather — oracle only (orc_gather_spade; no reference function)."""
        x, gamma, beta = (np.ascontiguousarray(a, np.float32) for a in (x, gamma, beta))
        idx = np.ascontiguousarray(idx, np.int32)
        n, c, h, w = x.shape
        win = s * b + k - s
        out = np.zeros((len(idx), c, win, win), np.float32)
        keep = []
        e = epilogue_struct(norm or [], keep)
        f = self.lib.orc_gather_spade
        f.restype = _i
        f.argtypes = [_vp, _vp, _vp, _i, _i, _i, _i, _vp, _i, _i, _i, _i, _i, _i, C.POINTER(Epilogue), _i, _vp]
        self._check(f(_ptr(x), _ptr(gamma), _ptr(beta), n, c, h, w, _ptr(idx), len(idx), b, ih, iw, k, s, C.byref(e),
                      act, _ptr(out)))
        return out

    def resize_nearest(self, x, oh, ow):
        """Nearest integer-factor resample — oracle only (orc_resize_nearest)."""
        x = np.ascontiguousarray(x, np.float32)
        n, c, h, w = x.shape
        out = np.zeros((n, c, oh, ow), np.float32)
        f = self.lib.orc_resize_nearest
        f.restype = _i
        f.argtypes = [_vp, _i, _i, _i, _i, _i, _i, _vp]
        self._check(f(_ptr(x), n, c, h, w, oh, ow, _ptr(out)))
        return out

    def scatter(self, blocks, idx, base):
        blocks = np.ascontiguousarray(blocks, np.float32)
        idx = np.ascontiguousarray(idx, np.int32)
        base = np.ascontiguousarray(base, np.float32)
        out = np.zeros_like(base)
        G, ch, b, _ = blocks.shape
        self._check(self.fn("scatter")(_ptr(blocks), G, ch, b, _ptr(idx), _ptr(base), _ptr(out), *base.shape))
        return out

    def scatter_add_inplace(self, blocks, idx, base):
        blocks = np.ascontiguousarray(blocks, np.float32)
        idx = np.ascontiguousarray(idx, np.int32)
        G, ch, b, _ = blocks.shape
        self._check(self.fn("scatter_add_inplace")(_ptr(blocks), G, ch, b, _ptr(idx), _ptr(base), *base.shape))
        return base

    def build_scatter_map(self, idx, b, h, w):
        idx = np.ascontiguousarray(idx, np.int32)
        out = (ScatterEntry * (h * w))()
        bps = _i(0)
        self._check(self.fn("build_scatter_map")(_ptr(idx), len(idx), b, h, w, C.addressof(out), C.byref(bps)))
        arr = np.frombuffer(out, dtype=np.dtype([("block", "<i4"), ("dy", "<i2"), ("dx", "<i2")])).reshape(h, w).copy()
        return arr, bps.value

    def scatter_gather(self, blocks, prod_idx, orig_out, cons_idx, cb, ch, cw, k, s, epi=None):
        blocks = np.ascontiguousarray(blocks, np.float32)
        prod_idx = np.ascontiguousarray(prod_idx, np.int32)
        cons_idx = np.ascontiguousarray(cons_idx, np.int32)
        orig_out = np.ascontiguousarray(orig_out, np.float32)
        n, c, h, w = orig_out.shape
        win = s * cb + k - s
        out = np.zeros((len(cons_idx), c, win, win), np.float32)
        keep = []
        e = epilogue_struct(epi or [], keep)
        self._check(
            self.fn("scatter_gather")(
                _ptr(blocks), len(prod_idx), blocks.shape[2], _ptr(prod_idx), _ptr(orig_out), n, c, h, w,
                _ptr(cons_idx), len(cons_idx), cb, ch, cw, k, s, C.byref(e), _ptr(out),
            )
        )
        return out

    def scatter_with_block_residual(self, mb, midx, sb, sidx, ssum, orig_sc, fused=True):
        mb, sb = (np.ascontiguousarray(a, np.float32) for a in (mb, sb))
        midx, sidx = (np.ascontiguousarray(a, np.int32) for a in (midx, sidx))
        ssum, orig_sc = (np.ascontiguousarray(a, np.float32) for a in (ssum, orig_sc))
        out = np.zeros_like(ssum)
        self._check(
            self.fn("scatter_with_block_residual")(
                _ptr(mb), len(midx), mb.shape[2], _ptr(midx), _ptr(sb), len(sidx), sb.shape[2], _ptr(sidx),
                _ptr(ssum), _ptr(orig_sc), _ptr(out), *ssum.shape, int(fused),
            )
        )
        return out

    def apply_epilogue_on_blocks(self, blocks, idx, ih, iw, epi):
        blocks = np.ascontiguousarray(blocks, np.float32).copy()
        idx = np.ascontiguousarray(idx, np.int32)
        keep = []
        e = epilogue_struct(epi or [], keep)
        G, ch, bh, _ = blocks.shape
        self._check(self.fn("apply_epilogue_on_blocks")(_ptr(blocks), G, ch, bh, _ptr(idx), ih, iw, C.byref(e)))
        return blocks

    def conv_on_blocks(self, blocks, weight, bias, k, stride, block, with_bias=True):
        blocks = np.ascontiguousarray(blocks, np.float32)
        keep = []
        cv = conv_struct(weight, bias, k, stride, keep)
        out = np.zeros((blocks.shape[0], cv.c_out, block, block), np.float32)
        self._check(self.fn("conv_on_blocks")(_ptr(blocks), blocks.shape[0], blocks.shape[2], C.byref(cv), int(with_bias), _ptr(out), block))
        return out

    def conv2d(self, x, weight, bias, k, stride, with_bias=True):
        x = np.ascontiguousarray(x, np.float32)
        keep = []
        cv = conv_struct(weight, bias, k, stride, keep)
        n, c, h, w = x.shape
        oh = (h + 2 * ((k - 1) // 2) - k) // stride + 1
        ow = (w + 2 * ((k - 1) // 2) - k) // stride + 1
        out = np.zeros((n, cv.c_out, oh, ow), np.float32)
        self._check(self.fn("conv2d")(_ptr(x), n, c, h, w, C.byref(cv), int(with_bias), _ptr(out)))
        return out

    def group_norm_fold(self, x, groups, gamma, beta, eps=1e-5):
        x = np.ascontiguousarray(x, np.float32)
        n, c, h, w = x.shape
        g = np.ascontiguousarray(gamma, np.float32)
        b = np.ascontiguousarray(beta, np.float32)
        sc = np.zeros(n * c, np.float32)
        sh = np.zeros(n * c, np.float32)
        self._check(self.fn("group_norm_fold")(_ptr(x), n, c, h, w, groups, eps, _ptr(g), _ptr(b), _ptr(sc), _ptr(sh)))
        return sc, sh

    # ---- models / executor
    def model(self, name_or_desc):
        """Build a named model, or adopt a ModelDesc (host pointers)."""
        if isinstance(name_or_desc, str):
            if self.p == "orc_":
                h = self.lib.orc_model_build(name_or_desc.encode())
                if not h:
                    raise OracleError(2, self.fn("last_error")().decode())
                return Model(self, h, owner=True)
            h = self.lib.ref_model_build(name_or_desc.encode())
        else:
            if self.p == "orc_":
                return Model(self, self.lib.orc_model_clone(name_or_desc), owner=True)
            h = self.lib.ref_model_from_desc(name_or_desc)
        if not h:
            raise OracleError(2, self.fn("last_error")().decode())
        return Model(self, h, owner=True)


class Model:
    def __init__(self, impl: _Impl, handle, owner=True):
        self.impl, self.h, self.owner = impl, handle, owner

    def _hv(self):
        return C.cast(self.h, C.c_void_p) if self.impl.p == "orc_" else self.h

    @property
    def desc(self):
        """ModelDesc pointer (oracle models only)."""
        assert self.impl.p == "orc_"
        return self.h

    def __del__(self):
        try:
            if self.owner and self.h:
                self.impl.fn("model_free")(self._hv())
        except Exception:
            pass

    def weight_hash(self) -> int:
        return int(self.impl.fn("model_weight_hash")(self._hv()))

    def required_dilation(self) -> int:
        return int(self.impl.fn("model_required_dilation")(self._hv()))

    def output_shape(self):
        c, h, w = _i(), _i(), _i()
        self.impl._check(self.impl.fn("model_output_shape")(self._hv(), C.byref(c), C.byref(h), C.byref(w)))
        return c.value, h.value, w.value

    def precompute(self, original):
        original = np.ascontiguousarray(original, np.float32)
        args = [self._hv(), _ptr(original), *original.shape]
        if self.impl.p == "ref_":
            args.append(0)
        h = self.impl.fn("cache_precompute")(*args)
        if not h:
            raise OracleError(2, self.impl.fn("last_error")().decode())
        return Cache(self.impl, h)

    def sparse_forward(self, cache, edited, mask, cfg: RunConfig | None = None, trace_cap=512):
        edited = np.ascontiguousarray(edited, np.float32)
        mask = np.ascontiguousarray(mask, np.uint8)
        cfg = cfg or default_config()
        n = edited.shape[0]
        c, h, w = self.output_shape()
        out = np.zeros((n, c, h, w), np.float32)
        rows = np.zeros((trace_cap, 6), np.uint64)
        nr = _i(0)
        self.impl._check(
            self.impl.fn("sparse_forward")(
                self._hv(), cache.h, _ptr(edited), *edited.shape, _ptr(mask), C.byref(cfg), _ptr(out),
                _ptr(rows), trace_cap, C.byref(nr),
            )
        )
        return out, rows[: nr.value].copy()

    def dense_forward(self, x, cache=None, step=0):
        x = np.ascontiguousarray(x, np.float32)
        c, h, w = self.output_shape()
        out = np.zeros((x.shape[0], c, h, w), np.float32)
        if cache is None:
            self.impl._check(self.impl.fn("dense_forward")(self._hv(), _ptr(x), *x.shape, _ptr(out)))
        else:
            self.impl._check(
                self.impl.fn("dense_forward_reused_stats")(self._hv(), _ptr(x), *x.shape, cache.h, step, _ptr(out))
            )
        return out


class Cache:
    def __init__(self, impl: _Impl, handle):
        self.impl, self.h = impl, handle

    def __del__(self):
        try:
            self.impl.fn("cache_free")(self.h)
        except Exception:
            pass

    def tensor(self, key, step=0):
        dims = (_i * 4)()
        self.impl._check(self.impl.fn("cache_tensor")(self.h, step, key.encode(), None, 0, C.byref(dims)))
        out = np.zeros(tuple(dims), np.float32)
        self.impl._check(self.impl.fn("cache_tensor")(self.h, step, key.encode(), _ptr(out), out.size, C.byref(dims)))
        return out

    def norm(self, key, step=0):
        cnt = _i(0)
        self.impl._check(self.impl.fn("cache_norm")(self.h, step, key.encode(), None, None, 0, C.byref(cnt)))
        sc = np.zeros(cnt.value, np.float32)
        sh = np.zeros(cnt.value, np.float32)
        self.impl._check(self.impl.fn("cache_norm")(self.h, step, key.encode(), _ptr(sc), _ptr(sh), cnt.value, C.byref(cnt)))
        return sc, sh

    def total_elements(self) -> int:
        return int(self.impl.fn("cache_total_elements")(self.h))

    def entries(self):
        """[(kind, key)] — oracle caches only."""
        L = self.impl.lib
        L.orc_cache_count.restype = _i
        L.orc_cache_count.argtypes = [_vp]
        L.orc_cache_entry.restype = _i
        L.orc_cache_entry.argtypes = [_vp, _i, C.POINTER(_i), C.c_char_p, _sz, C.POINTER(_sz)]
        out = []
        buf = C.create_string_buffer(128)
        for i in range(L.orc_cache_count(self.h)):
            kind, numel = _i(), _sz()
            L.orc_cache_entry(self.h, i, C.byref(kind), buf, 128, C.byref(numel))
            out.append((kind.value, buf.value.decode(), numel.value))
        return out


_ORC = None
_REF = None


def orc() -> _Impl:
    global _ORC
    if _ORC is None:
        _ORC = _Impl(ORC_PATH, "orc_")
    return _ORC


def ref() -> _Impl:
    global _REF
    if _REF is None:
        _REF = _Impl(REF_PATH, "ref_")
    return _REF


def ref_available() -> bool:
    return REF_PATH.exists()
