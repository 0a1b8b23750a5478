"""Op-level HBM roofline only (bench.py's ops_hbm block), for kernel iteration."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2211_02048_b200 as sb  # noqa: E402

peaks = json.load(open(os.path.join(os.path.dirname(bench.__file__), "MEASURED_PEAKS.json")))
print(json.dumps(peaks)[:300])
peak = float(sys.argv[1]) if len(sys.argv) > 1 else 6534.1
print(json.dumps(bench.ops_roofline(sb, torch, peak)))
