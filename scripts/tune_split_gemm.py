"""GEMM + activation mode (the paper's mmLeakyReLu): stream-K ranges per tile
(CUASM_OPT_SK_SPLIT) for few-tile shapes, per variant and MMA width; trimmed-mean L2-flushed time.

    python scripts/tune_split_gemm.py [--shapes MxKxN,...]
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
    ap.add_argument("--shapes", default="512x2048x512,512x4096x4096,256x2048x2048")
    ap.add_argument("--splits", default="2,3,4,6")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    flush = bench.L2Flush(dev)
    for shp in a.shapes.split(","):
        M, K, N = map(int, shp.split("x"))
        t = make_device_inputs(M, K, N, 11, dev)
        out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
        r = {"shape": shp, "plan": ffn.plan_config(M, K, N, "gemm")}
        r["auto"] = round(time_cfg(ffn.FusedFFN(dev), t["x"], t, out, 30, flush, "gemm"), 2)
        for v in (1, 2):
            for tn in (128, 256):
                for s in [0] + [int(x) for x in a.splits.split(",")]:
                    h = ffn.FusedFFN(dev)
                    h.set_variant(v)
                    h.set_option(ffn.OPT_TILE_N, tn)
                    h.set_option(ffn.OPT_SCHEDULE, 1 if s == 0 else 2)
                    if s:
                        h.set_option(ffn.OPT_SK_SPLIT, s)
                    r[f"{v}sm-n{tn}-{'dp' if s == 0 else f's{s}'}"] = round(time_cfg(h, t["x"], t, out, 30, flush, "gemm"), 2)
        r["best"] = min((k for k in r if k not in ("shape", "plan")), key=lambda k: r[k])
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
