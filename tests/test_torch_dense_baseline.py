"""The PyTorch / cuDNN dense baseline (tools/torch_dense.py, reported by
bench.py as dense_cudnn_ms) computes the reference's dense forward: checked
here in float64 on the CPU against the oracle's dense walk
(proj/src/graph.cpp:343-412) on three models."""
import os
import sys

import numpy as np
import pytest
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))

import paper_2211_02048_b200 as sb  # noqa: E402
from torch_dense import TorchDense  # noqa: E402


@pytest.mark.parametrize("name", ["mini_unet_gn", "ddim_stack_64x32", "gaugan_stack_in"])
def test_torch_dense_matches_oracle(orc, name):
    m = sb.Model(name)
    om = orc.model(name)
    c, h, w = m.in_shape
    _, e = orc.make_edit_fixture("rect5", 1, c, h, w, 3)
    want = om.dense_forward(e)
    got = TorchDense(m, dtype=torch.float64, device="cpu").forward(torch.from_numpy(e).double()).numpy()
    assert np.abs(got - want).max() / np.abs(want).max() < 1e-4
