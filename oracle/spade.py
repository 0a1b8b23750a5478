"""TEST INFRASTRUCTURE ONLY — the dense checker for BASELINE config 3 (the
GauGAN SPADE generator). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg may import this module; the product path never does.

The reference (SIGE's C++ proj/) has no SPADE layer: SPADE's per-pixel
gamma/beta do not fit its per-channel Epilogue and it has no label-map
resample. So config 3 is PARITY UNPINNED against the reference
itself. This module restates the published SPADE generator (Park et al. 2019,
SPADEGenerator / SPADEResnetBlock / SPADE, "normal" upsampling, param-free
instance norm) over the weights of a `sige_model_desc`:

  seg_k   = nearest(seg, h_k, w_k)
  a       = ReLU(conv3x3_shared(seg_k))
  gamma   = conv3x3_gamma(a);  beta = conv3x3_beta(a)
  spade(x)= instnorm(x) * (1 + gamma) + beta           (instnorm eps 1e-5, biased var)
  block(x)= conv_1(lrelu(spade_1(conv_0(lrelu(spade_0(x)))))) + (conv_s(spade_s(x)) | x)

in float64 (the dot products and the norm statistics) so that it checks the
CUDA path's FP32_FMA / EXACT modes to ~1e-6 and the fp16 / tf32 modes to
their own bound. The elementwise building blocks it uses (the modulation
order, nearest resize) are the ones pinned bit for bit against the C
restatement in tests/test_spade_ops.py; the convolution and residual
arithmetic are the reference's (conv: kernels.cpp:48-107, residual add:
graph.cpp:854-879) and are pinned through configs 1 and 2.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

LAYER_CONV, LAYER_NORM, LAYER_ACT, LAYER_RES, LAYER_DOWN, LAYER_UP, LAYER_SPADE, LAYER_RESIZE = range(8)
ACT_NONE, ACT_RELU, ACT_SILU, ACT_LEAKY = 0, 1, 2, 3


def _arr(ptr, n):
    if not ptr:
        return None
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_float)), shape=(n,)).astype(np.float64)


def conv_weights(cd):
    """(weight [co, ci, k, k], bias [co] or None, stride) of a sige_conv_desc."""
    w = _arr(cd.weight, cd.c_out * cd.c_in * cd.k * cd.k).reshape(cd.c_out, cd.c_in, cd.k, cd.k)
    return w, _arr(cd.bias, cd.c_out), cd.stride


def conv2d(x, cw):
    """Zero-padded 'same' convolution (pad (k-1)/2), NCHW float64."""
    w, b, s = cw
    n, ci, h, wd = x.shape
    co, _, k, _ = w.shape
    p = (k - 1) // 2
    xp = np.pad(x, ((0, 0), (0, 0), (p, p), (p, p)))
    oh, ow = (h + 2 * p - k) // s + 1, (wd + 2 * p - k) // s + 1
    out = np.zeros((n, co, oh, ow))
    for ky in range(k):
        for kx in range(k):
            win = xp[:, :, ky:ky + s * (oh - 1) + 1:s, kx:kx + s * (ow - 1) + 1:s]
            out += np.einsum("nchw,oc->nohw", win, w[:, :, ky, kx], optimize=True)
    if b is not None:
        out += b[None, :, None, None]
    return out


def nearest(x, h, w):
    """F.interpolate(mode='nearest') for integer factors (the engine rejects others)."""
    n, c, H, W = x.shape
    ys = np.arange(h) * H // h if h <= H else np.arange(h) // (h // H)
    xs = np.arange(w) * W // w if w <= W else np.arange(w) // (w // W)
    return x[:, :, ys][:, :, :, xs]


def act(x, kind):
    if kind == ACT_RELU:
        return np.maximum(x, 0)
    if kind == ACT_LEAKY:
        return np.where(x > 0, x, 0.2 * x)
    if kind == ACT_SILU:
        return x / (1 + np.exp(-x))
    return x


def instnorm(x, eps):
    m = x.mean(axis=(2, 3), keepdims=True)
    v = ((x - m) ** 2).mean(axis=(2, 3), keepdims=True)
    return (x - m) / np.sqrt(v + eps)


def spade(x, seg, sd):
    segk = nearest(seg, x.shape[2], x.shape[3])
    a = act(conv2d(segk, conv_weights(sd.shared)), ACT_RELU)
    gamma = conv2d(a, conv_weights(sd.gamma))
    beta = conv2d(a, conv_weights(sd.beta))
    return instnorm(x, sd.eps) * (1 + gamma) + beta


def spade_block(x, seg, L):
    sp = L.spade
    dx = conv2d(act(spade(x, seg, sp[0]), L.act), conv_weights(L.conv))
    dx = conv2d(act(spade(dx, seg, sp[1]), L.act), conv_weights(L.conv2))
    xs = conv2d(spade(x, seg, sp[2]), conv_weights(L.shortcut)) if L.has_shortcut else x
    return xs + dx


def forward(desc, seg):
    """Dense forward of a SPADE generator description (sige_model_desc*,
    ctypes) on a one-hot segmentation map seg [n, label_nc, H, W]."""
    d = desc.contents
    seg = np.asarray(seg, np.float64)
    x = seg
    for i in range(d.num_layers):
        L = d.layers[i]
        if L.kind in (LAYER_CONV, LAYER_DOWN):
            x = conv2d(x, conv_weights(L.conv))
        elif L.kind == LAYER_ACT:
            x = act(x, L.act)
        elif L.kind == LAYER_UP:
            x = x.repeat(2, axis=2).repeat(2, axis=3)
        elif L.kind == LAYER_RESIZE:
            x = nearest(seg, L.resize_h, L.resize_w)
        elif L.kind == LAYER_SPADE:
            x = spade_block(x, seg, L)
        else:
            raise ValueError(f"oracle/spade.py: layer kind {L.kind} is not part of a SPADE generator")
    return x
