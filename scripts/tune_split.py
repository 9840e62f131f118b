"""Stream-K ranges per tile (CUASM_OPT_SK_SPLIT) for shapes with fewer tiles
than CTAs: decode-like and tensor-parallel shard shapes.  Times the forward
(L2 flushed, median) for each (variant, split), stream-K over all tiles.

    python scripts/tune_split.py [--shapes MxKxN,...] [--out path.json]
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
    ap.add_argument("--shapes", default="16x4096x1376,128x4096x1376,512x4096x1376,16x4096x2752,16x4096x5504,"
                                        "256x4096x1376,1024x4096x1376")
    ap.add_argument("--splits", default="2,3,4,6,8,12,16")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    flush = bench.L2Flush(dev)
    rows = []
    for shp in a.shapes.split(","):
        M, K, N = map(int, shp.split("x"))
        t = make_device_inputs(M, K, N, 11, dev)
        out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
        r = {"M": M, "K": K, "N": N}
        for v in (1, 2):
            hdp = ffn.FusedFFN(dev)
            hdp.set_variant(v)
            hdp.set_option(ffn.OPT_SCHEDULE, 1)
            r[f"{v}sm-dp"] = round(time_cfg(hdp, t["x"], t, out, a.steps, flush), 2)
            for s in map(int, a.splits.split(",")):
                h = ffn.FusedFFN(dev)
                h.set_variant(v)
                h.set_option(ffn.OPT_SCHEDULE, 2)
                h.set_option(ffn.OPT_SK_SPLIT, s)
                r[f"{v}sm-s{s}"] = round(time_cfg(h, t["x"], t, out, a.steps, flush), 2)
        r["auto"] = round(time_cfg(ffn.FusedFFN(dev), t["x"], t, out, a.steps, flush), 2)
        r["best"] = min((k for k in r if k not in ("M", "K", "N")), key=lambda k: r[k])
        rows.append(r)
        print(json.dumps(r), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"unit": "us per forward (median, L2 flushed)", "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
