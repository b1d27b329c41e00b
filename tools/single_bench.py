"""Single-tree propagations/s per config (jt_propagate, CUDA events, state reset
outside the timer) — the bench's single_tree table on its own.
usage: python tools/single_bench.py [c1 c2 c3 c4B c4M c5] [--dtypes f32,f64]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ap = argparse.ArgumentParser()
ap.add_argument("configs", nargs="*", default=["c1", "c2", "c3", "c4B", "c4M", "c5"])
ap.add_argument("--dtypes", default="f32,f64")
a = ap.parse_args()

import bench  # noqa: E402

print(json.dumps(bench.single_tree_table(tuple(a.dtypes.split(",")), tuple(a.configs)), indent=1))
