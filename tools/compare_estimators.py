"""NEXT f1: equal-sample RMSE of the hybrid VPL set vs plain IR against a
dense IR reference on a seeded config; prints one JSON line.

  python tools/compare_estimators.py --config 3 --M 1024 4096 16384 --ref-M 262144
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2203_11484_b200 as V  # noqa: E402
import scenegen  # noqa: E402
from paper_2203_11484_b200.compare import compare_estimators  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--M", type=int, nargs="+", default=[1024, 4096, 16384])
ap.add_argument("--ref-M", type=int, default=262144)
a = ap.parse_args()
V.load_library()
print(json.dumps(compare_estimators(scenegen.make_scene(a.config), a.M, a.ref_M)), flush=True)
