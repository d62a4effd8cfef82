"""Run bench.py's boundary-IO leg alone (for ncu captures of k_gather_phase /
k_scatter_phase):  python tools/bench_io.py [reps]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2308_14258_b200 as mfp  # noqa: E402

peaks = {}
p = os.path.join(ROOT, "MEASURED_PEAKS.json")
if os.path.exists(p):
    peaks = json.load(open(p))
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
print(json.dumps(bench.boundary_io_bench(mfp, torch, peaks, reps)))
if len(sys.argv) > 2:
    print(json.dumps(bench.boundary_io_bench(mfp, torch, peaks, reps, flush_l2=False)))
