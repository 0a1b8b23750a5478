"""GPU parity on the headline workload: BASELINE config 2 at full size.

ddim_stack (3x256x256 input, 128-512 channels, 51 layers / 80 conv sites,
random init Rng seed 2211), rect1 edit seed 7 (784 px, 1.196 %), dilate_full 5,
dilate_scale 1, min_sparse_res 64, block 6 / 4 — the configuration bench.py
times. The checker is the UNMODIFIED reference (oracle/_ref, compiled from
proj/src) running sigeref::precompute and sigeref::sparse_forward
(graph.cpp:426-435, 619-901) on the host.

* SIGE_MATH_EXACT: bit-exact, with the reference's own cache uploaded and with
  the device precompute (whose every cache tensor must equal the reference's).
* SIGE_MATH_F16 / SIGE_MATH_TF32 (the bench's mode is F16): the north star's
  max relative error <= 1e-2 (normalised max |d| / max |ref|) and
  every pixel outside the reference's output_coverage (graph.cpp:1078-1129)
  bit-identical to the cached output. The elementwise figure
  |d| <= 1e-2 (|ref| + 1e-3 max|ref|) of SURVEY §8(c) is measured and printed
  for every mode; it bounds the error at near-zero outputs by 1e-5 max|ref|,
  which 11-bit significands (fp16 / tf32 operands) cannot reach where a
  1152-term dot product cancels to ~0 (measured: 0.46 % of the elements, worst
  73x, normalised max 1.9e-3), so it is asserted for the FP32 modes only.
* SIGE_MATH_FP32_FMA (fp32 CUDA cores, FMA contraction — the north star's
  check mode): normalised max error <= 1e-4 and the elementwise floor.
* The same edit through the host-buffer C-ABI entry point (the e2e path) and
  through 8 engines in flight on one GPU under set_sm_budget (the batched
  requests path) gives the same bits as the direct device call.
"""
import ctypes as C

import numpy as np
import pytest
import torch

import paper_2211_02048_b200 as sb

pytestmark = pytest.mark.gpu

WORKLOAD = dict(dilate_full=5, dilate_scale=1, min_sparse_res=64, block3=6, block1=4)


def errors(got, want):
    """(normalised max error, fraction of elements outside the elementwise
    floor, worst elementwise ratio |d| / (1e-2 (|ref| + 1e-3 max|ref|)))."""
    d = np.abs(got.astype(np.float64) - want.astype(np.float64))
    m = float(np.abs(want).max())
    floor = 1e-2 * (np.abs(want).astype(np.float64) + 1e-3 * m)
    ratio = d / floor
    return float(d.max() / max(m, 1e-30)), float((ratio > 1).mean()), float(ratio.max())


@pytest.fixture(scope="module")
def c2(ref):
    """Reference precompute + sparse_forward of config 2 (host, all threads)."""
    import os

    os.environ.setdefault("SIGE_THREADS", str(os.cpu_count() or 1))
    rm = ref.model("ddim_stack")
    orig, edited = ref.make_edit_fixture("rect1", 1, 3, 256, 256, 7)
    mask = ref.difference_mask(orig, edited)
    cfg = sb.default_config(**WORKLOAD)
    cache = rm.precompute(orig)
    want, wtrace = rm.sparse_forward(cache, edited, mask, cfg)
    cov = np.zeros((256, 256), np.uint8)
    oh, ow = C.c_int(), C.c_int()
    assert ref.lib.ref_output_coverage(rm.h, mask.ctypes.data, 256, 256, 1, C.byref(cfg), cov.ctypes.data,
                                       C.byref(oh), C.byref(ow)) == 0
    assert (oh.value, ow.value) == (256, 256)
    return dict(rm=rm, orig=orig, edited=edited, mask=mask, cfg=cfg, cache=cache, want=want, wtrace=wtrace,
                outside=np.broadcast_to(cov[None, None] == 0, want.shape), final=cache.tensor("final"))


def upload_ref_cache(eng, c2):
    """Every entry of the reference's cache (the key list comes from the
    engine's own cache layout, which mirrors graph.cpp:356-410)."""
    for kind, key, shp in eng.cache_entries():
        if kind == "T":
            t = c2["orig"] if key == "input" else c2["cache"].tensor(key)
            assert t.shape == tuple(shp), key
            eng.put_tensor(key, t)
        else:
            sc, sh = c2["cache"].norm(key)
            assert sc.size == shp, key
            eng.put_norm(key, sc, sh)


def new_engine(math, device_precompute, c2):
    eng = sb.Engine(sb.Model("ddim_stack"), batch=1, math=math)
    eng.precompute(torch.from_numpy(c2["orig"]).cuda())  # also lays out every cache entry
    if not device_precompute:
        upload_ref_cache(eng, c2)
    torch.cuda.synchronize()
    return eng


def run(eng, c2, reps=3):
    """Direct run, then graph capture, then replay — all must agree."""
    x = torch.from_numpy(c2["edited"]).cuda()
    out = torch.empty(eng.output_shape(), device="cuda")
    res = []
    for _ in range(reps):
        eng.sparse_forward(x, config=c2["cfg"], out=out)
        res.append(out.cpu().numpy().copy())
    for r in res[1:]:
        assert np.array_equal(r.view(np.uint32), res[0].view(np.uint32)), "graph replay changed the bits"
    return res[0]


def test_config2_reference_trace_shape(c2):
    """The workload is the one bench.py reports: 40 sparse sites, 1,132 active
    tiles in total, 25.13 G MAC."""
    tr = c2["wtrace"]
    assert len(tr) == 80
    assert int(tr[tr[:, 5] == 1, 0].sum()) == 1132
    assert int(tr[:, 3].sum()) == 25134342144


@pytest.mark.parametrize("device_precompute", [False, True], ids=["ref_cache", "device_precompute"])
def test_config2_exact_bit_exact(c2, device_precompute):
    eng = new_engine(sb.MATH_EXACT, device_precompute, c2)
    if device_precompute:  # the device dense walk reproduces sigeref::precompute bit for bit
        for kind, key, shp in eng.cache_entries():
            if key == "input":
                continue
            if kind == "T":
                want = c2["cache"].tensor(key)
                got = eng.get_tensor(key, shp).numpy()
            else:
                want = np.concatenate(c2["cache"].norm(key))
                got = np.concatenate([a.numpy() for a in eng.get_norm(key, shp)])
            assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), key
    got = run(eng, c2)
    assert np.array_equal(got.view(np.uint32), c2["want"].view(np.uint32)), \
        f"max diff {np.abs(got - c2['want']).max()}"
    assert np.array_equal(eng.trace().numpy().astype(np.uint64), c2["wtrace"])


@pytest.mark.parametrize("math", [sb.MATH_F16, sb.MATH_TF32], ids=["f16", "tf32"])
@pytest.mark.parametrize("device_precompute", [False, True], ids=["ref_cache", "device_precompute"])
def test_config2_tensor_core_tolerance(c2, math, device_precompute):
    eng = new_engine(math, device_precompute, c2)
    got = run(eng, c2)
    want = c2["want"]
    nerr, frac_out, worst = errors(got, want)
    print(f"\nconfig2 math={math} device_precompute={device_precompute}: max_norm_err={nerr:.3e} "
          f"elementwise: {frac_out * 100:.4f}% of elements above the floor, worst ratio {worst:.2f}")
    assert nerr <= 1e-2
    # outside the sparse footprint the output is the cache, bit for bit
    fin = c2["final"] if not device_precompute else eng.get_tensor("final", want.shape).numpy()
    out = c2["outside"]
    assert out.any() and np.array_equal(got[out].view(np.uint32), fin[out].view(np.uint32))
    assert np.array_equal(eng.trace().numpy().astype(np.uint64), c2["wtrace"])


@pytest.mark.parametrize("device_precompute", [False, True], ids=["ref_cache", "device_precompute"])
def test_config2_fp32_fma_check_mode(c2, device_precompute):
    eng = new_engine(sb.MATH_FP32_FMA, device_precompute, c2)
    got = run(eng, c2)
    nerr, frac_out, worst = errors(got, c2["want"])
    print(f"\nconfig2 math=fp32_fma device_precompute={device_precompute}: max_norm_err={nerr:.3e} "
          f"elementwise: {frac_out * 100:.4f}% above the floor, worst ratio {worst:.3f}")
    assert nerr <= 1e-4
    assert frac_out == 0.0, worst
    fin = c2["final"] if not device_precompute else eng.get_tensor("final", got.shape).numpy()
    assert np.array_equal(got[c2["outside"]].view(np.uint32), fin[c2["outside"]].view(np.uint32))


def test_config2_host_entry_point(c2):
    """sige_engine_sparse_forward_host (the e2e path) == the device call."""
    eng = new_engine(sb.MATH_F16, True, c2)
    dev = run(eng, c2)
    edited_h = torch.from_numpy(c2["edited"]).pin_memory()
    out_h = torch.empty(eng.output_shape()).pin_memory()
    for _ in range(3):  # direct, capture, replay
        eng.sparse_forward_host(edited_h, config=c2["cfg"], out_host=out_h)
        assert np.array_equal(out_h.numpy().view(np.uint32), dev.view(np.uint32))
    # pageable buffers and an explicit mask too
    got = eng.sparse_forward_host(torch.from_numpy(c2["edited"]), torch.from_numpy(c2["mask"]), config=c2["cfg"])
    assert np.array_equal(got.numpy().view(np.uint32), dev.view(np.uint32))
    assert errors(dev, c2["want"])[0] <= 1e-2


def test_config2_concurrent_engines_sm_budget(c2):
    """8 independent requests (own original and edit, seeds 7..14), each its own
    engine on its own stream with set_sm_budget(37) (the bench's batched-requests
    path), all in flight together: every output equals the same engine run
    alone, and request 0 (seed 7) is within tolerance of the reference."""
    R = 8
    model = sb.Model("ddim_stack")
    engines, inputs, outs, alone, streams = [], [], [], [], []
    for i in range(R):
        o, e = sb.make_edit_fixture("rect1", 1, 3, 256, 256, 7 + i)
        eng = sb.Engine(model, batch=1, math=sb.MATH_F16)
        eng.set_sm_budget(37)
        eng.precompute(o.cuda())
        x = e.cuda()
        y = torch.empty(eng.output_shape(), device="cuda")
        eng.sparse_forward(x, config=c2["cfg"], out=y)  # alone, direct launches
        torch.cuda.synchronize()
        alone.append(y.cpu().numpy().copy())
        engines.append(eng)
        inputs.append(x)
        outs.append(y)
        streams.append(torch.cuda.Stream())
    main = torch.cuda.current_stream()
    for _ in range(4):  # capture + replays, all requests in flight
        for y in outs:
            y.fill_(float("nan"))
        for st in streams:
            st.wait_stream(main)
        for eng, st, x, y in zip(engines, streams, inputs, outs):
            with torch.cuda.stream(st):
                eng.sparse_forward(x, config=c2["cfg"], out=y)
        for st in streams:
            main.wait_stream(st)
        torch.cuda.synchronize()
        for i in range(R):
            assert np.array_equal(outs[i].cpu().numpy().view(np.uint32), alone[i].view(np.uint32)), i
    assert errors(alone[0], c2["want"])[0] <= 1e-2
