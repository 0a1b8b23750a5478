"""Dense baseline on B200 through PyTorch / cuDNN (not part of the product):
the same model (weights read from the model description through the C ABI)
as eager torch ops — conv2d (cuDNN, fp16, channels-last), group_norm, SiLU,
nearest upsample — replayed as one CUDA graph. Semantics follow the
reference's dense walk (proj/src/graph.cpp:343-412): ResBlock = conv1 ->
norm -> act -> conv2, plus the 1x1 shortcut (or identity), summed."""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.nn.functional as F

from paper_2211_02048_b200 import _capi


def _arr(ptr, n):
    if not ptr:
        return None
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_float)), shape=(n,)).copy()


class TorchDense:
    def __init__(self, model, dtype=torch.float16, device="cuda"):
        d = model.desc.contents
        self.dtype, self.device = dtype, device
        self.layers = []

        def conv(cd):
            w = _arr(cd.weight, cd.c_out * cd.c_in * cd.k * cd.k).reshape(cd.c_out, cd.c_in, cd.k, cd.k)
            b = _arr(cd.bias, cd.c_out)
            wt = torch.from_numpy(w).to(device, dtype).contiguous(memory_format=torch.channels_last)
            bt = torch.from_numpy(b).to(device, dtype) if b is not None else None
            return (wt, bt, cd.stride, (cd.k - 1) // 2)

        def norm(nd):
            return (nd.kind, nd.groups, nd.eps, torch.from_numpy(_arr(nd.gamma, nd.channels)).to(device, dtype),
                    torch.from_numpy(_arr(nd.beta, nd.channels)).to(device, dtype),
                    None if not nd.running_mean else torch.from_numpy(_arr(nd.running_mean, nd.channels)).to(device, dtype),
                    None if not nd.running_var else torch.from_numpy(_arr(nd.running_var, nd.channels)).to(device, dtype))

        for i in range(d.num_layers):
            L = d.layers[i]
            if L.kind in (_capi.LAYER_CONV, _capi.LAYER_DOWNSAMPLE):
                self.layers.append(("conv", conv(L.conv)))
            elif L.kind == _capi.LAYER_NORM:
                self.layers.append(("norm", norm(L.norm)))
            elif L.kind == _capi.LAYER_ACTIVATION:
                self.layers.append(("act", L.act))
            elif L.kind == _capi.LAYER_UPSAMPLE:
                self.layers.append(("up", None))
            elif L.kind == _capi.LAYER_RESBLOCK:
                self.layers.append(("res", (conv(L.conv), norm(L.norm), L.act, conv(L.conv2),
                                            conv(L.shortcut) if L.has_shortcut else None)))
        self.graph = None

    @staticmethod
    def _conv(x, c):
        w, b, s, p = c
        return F.conv2d(x, w, b, stride=s, padding=p)

    @staticmethod
    def _norm(x, n):
        kind, groups, eps, g, b, rm, rv = n
        if kind == _capi.NORM_BATCH:
            return F.batch_norm(x, rm, rv, g, b, False, 0.0, eps)
        return F.group_norm(x, groups, g, b, eps)

    @staticmethod
    def _act(x, a):
        if a == _capi.ACT_RELU:
            return F.relu(x)
        if a == _capi.ACT_SILU:
            return F.silu(x)
        return x

    def forward(self, x):
        x = x.to(self.dtype).contiguous(memory_format=torch.channels_last)
        for kind, p in self.layers:
            if kind == "conv":
                x = self._conv(x, p)
            elif kind == "norm":
                x = self._norm(x, p)
            elif kind == "act":
                x = self._act(x, p)
            elif kind == "up":
                x = F.interpolate(x, scale_factor=2, mode="nearest")
            else:
                c1, nrm, a, c2, sc = p
                h = self._act(self._norm(self._conv(x, c1), nrm), a)
                x = self._conv(h, c2) + (self._conv(x, sc) if sc is not None else x)
        return x

    def capture(self, x_static):
        """CUDA-graph the forward on a static input (launch overhead out of the way)."""
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(3):
                self.out = self.forward(x_static)
        torch.cuda.current_stream().wait_stream(s)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.out = self.forward(x_static)
        return self

    def replay(self):
        self.graph.replay()
        return self.out
