"""Per-shard kernel times of the C3 grid split over 2 / 4 / 8 ranks, each shard timed alone on this
GPU (bench.py's shard_balance), plus the whole-grid kernel time:  python tools/shard_time.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import bench

out = bench.shard_balance(torch)
for k, v in out.items():
    print(os.environ.get("AB_TAG", ""), k, "min %.4f max %.4f ms" % (min(v["shard_ms"]), max(v["shard_ms"])),
          "max/mean %.3f" % v["max_over_mean"], flush=True)
