"""Generate tests/golden/golden.npz + golden.json from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libsigeref.so, built from
/root/reference by oracle/Makefile):

    python tests/golden/make_golden.py

Every input comes from the reference's own seeded generators
(make_edit_fixture, toy models; proj/src/fixtures.cpp, proj/src/models.cpp),
so only outputs are stored. The CPU suite checks the oracle restatement
against these vectors; the GPU suite checks the CUDA path against them.
"""
import json
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_2211_02048_b200._capi import default_config  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent


def main():
    R = oracle.ref()
    arrays, meta = {}, {}

    # --- config 1 inputs and the mask / index / gather chain
    o, e = R.make_edit_fixture("rect1", 1, 64, 256, 256, 7)
    hs = lambda t: R.fnv1a64(t, R.fnv1a64(np.array(t.shape, np.int32)))  # Tensor::content_hash
    meta["rect1_64x256_original_hash"] = hs(o)
    meta["rect1_64x256_edited_hash"] = hs(e)
    m = R.difference_mask(o, e, 1e-3)
    meta["rect1_mask_hash"] = R.fnv1a64(m)
    meta["rect1_mask_count"] = int(m.sum())
    d = R.dilate_mask(R.dilate_mask(m, 1), 1)
    idx6, h6 = R.mask_to_block_indices(d, 6, 1)
    idx4, _ = R.mask_to_block_indices(d, 4, 1)
    meta["rect1_idx6_hash"] = h6
    meta["rect1_idx6_count"] = len(idx6)
    meta["rect1_idx4_count"] = len(idx4)
    arrays["rect1_idx6"] = idx6
    g = R.gather(e, idx6, 6, 256, 256, 3, 1)
    meta["rect1_gather_hash"] = R.fnv1a64(g)

    # --- a gather with the GroupNorm scale-shift + SiLU epilogue (libm expf)
    rng = np.random.default_rng(2024)
    sc = rng.uniform(0.5, 1.5, 64).astype(np.float32)
    sh = rng.uniform(-0.4, 0.4, 64).astype(np.float32)
    arrays["silu_scale"], arrays["silu_shift"] = sc, sh
    arrays["rect1_gather_silu"] = R.gather(e, idx6[:8], 6, 256, 256, 3, 1, [("ss", sc, sh), ("act", 2)])

    # --- model weight hashes / required dilation (test_graph.cpp:151-166)
    for name in ["conv3x3_128", "mini_unet_gn", "mini_unet_bn", "gaugan_stack_in", "single_conv64",
                 "ddim_stack", "ddim_stack_64x32"]:
        mm = R.model(name)
        meta[f"weight_hash_{name}"] = mm.weight_hash()
        meta[f"required_dilation_{name}"] = mm.required_dilation()

    # --- end-to-end sparse_forward outputs on small models
    cases = {
        "mini_unet_gn_rect5_s17": ("mini_unet_gn", "rect5", 1, 17, {}),
        "mini_unet_bn_rect15_s11": ("mini_unet_bn", "rect15", 1, 11, {"dilate_full": 3}),
        "gaugan_multi15_s3": ("gaugan_stack_in", "multi15", 1, 3, {}),
        "mini_unet_gn_blob5_n2_s5_raw": ("mini_unet_gn", "blob5", 2, 5, {"norm_precompute": 0}),
        "ddim64x32_rect5_s7": ("ddim_stack_64x32", "rect5", 1, 7, {"dilate_full": 5, "min_sparse_res": 16}),
    }
    for tag, (name, fx, n, seed, over) in cases.items():
        mm = R.model(name)
        o, e = R.make_edit_fixture(fx, n, 3, 64, 64, seed)
        mask = R.difference_mask(o, e, 1e-3)
        over = dict(over)
        df = over.pop("dilate_full", mm.required_dilation())
        cfg = default_config(dilate_full=df, **over)
        cache = mm.precompute(o)
        out, trace = mm.sparse_forward(cache, e, mask, cfg)
        arrays[f"{tag}_out"] = out
        arrays[f"{tag}_trace"] = trace
        meta[f"{tag}_config"] = {"model": name, "fixture": fx, "batch": n, "seed": seed, "dilate_full": df, **over}
        meta[f"{tag}_cache_total_elements"] = cache.total_elements()
    np.savez_compressed(OUT / "golden.npz", **arrays)
    with open(OUT / "golden.json", "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", OUT / "golden.npz", sum(a.nbytes for a in arrays.values()), "bytes raw")


if __name__ == "__main__":
    main()
