"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of
`bench.py`: per-kernel totals over the whole run and the launch-by-launch list
of the last complete sparse step (delimited by k_mask_bits launches).
ncu serialises launches with cold caches: compare SHARES, not absolutes.

usage: python tools/launch_summary.py gpurun_out/launches.csv > profiles/rNN_launches.txt
"""
import collections
import csv
import sys


def load(path):
    hdr, rows = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                name = d["Kernel Name"].split("(")[0].replace("sige_b200::<unnamed>::", "").replace("void ", "")
                rows.append((name, float(d["Metric Value"]) / 1e3, d["Grid Size"]))
    return rows


def main(path):
    rows = load(path)
    starts = [i for i, r in enumerate(rows) if r[0].startswith("k_mask_bits")]
    print(f"# {path}: {len(rows)} launches, sparse steps start at {starts}")
    if len(starts) >= 2:
        step = rows[starts[-2]:starts[-1]]
        tot = sum(t for _, t, _ in step)
        agg = collections.defaultdict(lambda: [0, 0.0])
        for n, t, _ in step:
            agg[n][0] += 1
            agg[n][1] += t
        print(f"\n## last complete sparse step: {len(step)} launches, sum {tot:.1f} us (ncu, serialised)")
        for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            print(f"{c:5d} {t:9.1f} us {100 * t / tot:5.1f}%  {n}")
        print("\n## launch by launch")
        for n, t, g in step:
            print(f"{t:8.1f} us {g:>14} {n}")


if __name__ == "__main__":
    main(sys.argv[1])
