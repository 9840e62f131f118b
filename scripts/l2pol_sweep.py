"""TMA L2 cache-policy sweep (CUASM_OPT_L2_POLICY: bits 0-1 x, bits 2-3 W13; 0 normal, 1 evict_first,
2 evict_last) on given shapes, L2 flushed, trimmed mean of 30 (scripts/tune.py time_cfg).

    python scripts/l2pol_sweep.py [--shapes MxKxN,...] [--pols 0,2,8,10,1,4,6,9]
"""
import argparse
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
    ap.add_argument("--shapes", default="2048x4096x1376,2048x4096x2752,2048x4096x11008")
    ap.add_argument("--pols", default="0,2,8,10,1,4,6,9")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    flush = bench.L2Flush(dev)
    for shp in a.shapes.split(","):
        M, K, N = map(int, shp.split("x"))
        t = make_device_inputs(M, K, N, 5, dev)
        out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
        res = {}
        for pol in map(int, a.pols.split(",")):
            h = ffn.FusedFFN(dev)
            h.set_option(ffn.OPT_L2_POLICY, pol)
            res[pol] = round(time_cfg(h, t["x"], t, out, 30, flush), 2)
            del h
        print(shp, res, flush=True)


if __name__ == "__main__":
    main()
