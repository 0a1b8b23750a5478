"""Config-3 settings probe: sparse edit time and quality of the GauGAN SPADE
generator over (min_sparse_res, dilate_full). Quality = normalised max error
against the dense pass with the cached instance-norm statistics (what the
dilation loses) and against the fresh-statistics dense pass (what the whole
approximation loses), plus PSNR of the latter over the output range."""
import json
import sys

import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2211_02048_b200 as sb  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    m = sb.Model(sys.argv[1] if len(sys.argv) > 1 else "gaugan_spade")
    c, h, w = m.in_shape
    orig, edited = sb.make_seg_fixture(1, c, h, w, 11)
    eng = sb.Engine(m, batch=1, math=sb.MATH_F16)
    x0, x1 = orig.to(dev), edited.to(dev)
    eng.precompute(x0)
    cached = eng.dense_forward(x1, reused_stats=True).clone()
    fresh = eng.dense_forward(x1).clone()
    flush = torch.empty(128 << 20, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream()

    def timed(fn, reps=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            fn()
            b.record(st)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return sorted(ts)[len(ts) // 2]

    dense = timed(lambda: eng.dense_forward(x1))
    print(json.dumps({"dense_ms": round(dense, 4)}))
    rng = float(fresh.max() - fresh.min())
    for msr in (1, 16, 32):
        for df, ds in ((5, 1), (5, 2), (5, 4), (5, 8), (5, 16), (20, 4)):
            cfg = sb.default_config(dilate_full=df, dilate_scale=ds, min_sparse_res=msr)
            out = torch.empty(eng.output_shape(), device=dev)
            t = timed(lambda: eng.sparse_forward(x1, config=cfg, out=out))
            tr = eng.trace().numpy()
            got = eng.sparse_forward(x1, config=cfg).clone()
            ne = lambda a, b: round(float((a - b).abs().max() / b.abs().max()), 5)
            mse = float(((got - fresh) ** 2).mean())
            psnr = 10 * torch.log10(torch.tensor(rng * rng / max(mse, 1e-30))).item()
            print(json.dumps({"min_sparse_res": msr, "dilate_full": df, "dilate_scale": ds, "sparse_ms": round(t, 4),
                              "speedup": round(dense / t, 3),
                              "mac_reduction": round(float(tr[:, 4].sum() / max(tr[:, 3].sum(), 1)), 3),
                              "err_vs_cached": ne(got, cached), "err_vs_fresh": ne(got, fresh),
                              "psnr_vs_fresh_db": round(psnr, 2),
                              "mean_abs_err_vs_fresh": round(float((got - fresh).abs().mean()), 6)}))


if __name__ == "__main__":
    main()
