"""Per-launch DRAM traffic and tensor-pipe activity of the k_conv_tc launches
of the last complete sparse step in an ncu capture of bench.py, written as
profiles/r1_conv_traffic.json (read by bench.py for roofline.traffic).

capture (tools/gpu_traffic.sh):
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,
      sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
      --clock-control none -c 2000 --csv --log-file gpurun_out/traffic.csv
      python bench.py --steps 2 --warmup 1 --no-cpu-baseline --requests 1
usage: python tools/conv_traffic.py gpurun_out/traffic.csv > profiles/r1_conv_traffic.json
"""
import collections
import csv
import json
import sys


def main(path):
    hdr, launches = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"].split("(")[0].replace("sige_b200::<unnamed>::", "").replace("void ", "")
            e = launches.setdefault(d["ID"], {"name": name})
            v = float(d["Metric Value"].replace(",", "")) if d["Metric Value"] not in ("", "n/a") else 0.0
            unit = d.get("Metric Unit", "")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1,
                     "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3}.get(unit, 1)
            e[d["Metric Name"]] = v * scale
    rows = list(launches.values())
    starts = [i for i, r in enumerate(rows) if r["name"].startswith("k_mask_bits")]
    step = rows[starts[-2]:starts[-1]]
    conv = [r for r in step if r["name"].startswith("k_conv_tc")]
    n = len(conv)
    byts = [r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0) for r in conv]
    tp = [r.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 0) for r in conv]
    out = {
        "kernel": "k_conv_tc",
        "launches": n,
        "dram_bytes_per_launch": int(sum(byts) / n),
        "ncu_time_us_per_launch": round(sum(r.get("gpu__time_duration.sum", 0) for r in conv) / n, 3),
        "tensor_pipe_pct_mean": round(sum(tp) / n, 4),
        "tensor_pipe_pct_max": round(max(tp), 3),
        "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                  "sm__pipe_tensor_cycles_active over the k_conv_tc launches of one bench.py sparse step "
                  "(tools/gpu_traffic.sh, tools/conv_traffic.py)",
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
