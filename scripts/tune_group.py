"""Rasterisation group size (CUASM_OPT_GROUP_M: m-blocks per group; W13 column
block re-use vs x residency in L2) per shape, L2 flushed, median of 20.

    python scripts/tune_group.py [--shapes MxKxN,...] [--groups 2,4,8,16]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import bench
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs
from scripts.tune import time_cfg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="4096x8192x28672,4096x8192x3584,2048x4096x11008,8192x4096x11008,"
                                        "16384x4096x11008")
    ap.add_argument("--groups", default="0,2,4,6,8,12,16")
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    flush = bench.L2Flush(dev)
    for shp in a.shapes.split(","):
        M, K, N = map(int, shp.split("x"))
        t = make_device_inputs(M, K, N, 11, dev)
        out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
        r = {"shape": shp}
        for g in map(int, a.groups.split(",")):
            h = ffn.FusedFFN(dev)
            h.set_option(ffn.OPT_GROUP_M, g)
            r[f"g{g}"] = round(time_cfg(h, t["x"], t, out, a.steps, flush), 2)
            del h
        print(json.dumps(r), flush=True)
        del t, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
