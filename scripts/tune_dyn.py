"""A/B of dynamic whole-tile claiming (CUASM_OPT_DYNAMIC off = 1 / on = 2) on the
many-round shapes, with the bench protocol (L2 flushed before every step, CUDA events).

    python scripts/tune_dyn.py [--shapes M:K:N,...] [--dyn 1,2] [--steps 20]
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

DEFAULT = "2048:4096:11008,4096:8192:28672,4096:8192:3584,4096:8192:7168,16384:4096:11008,2048:4096:1376,4096:4096:11008"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default=DEFAULT)
    ap.add_argument("--dyn", default="1,2")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--groups", default="0", help="CUASM_OPT_GROUP_M values (0 = auto)")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    flush = bench.L2Flush(dev)
    for sh in a.shapes.split(","):
        M, K, N = (int(v) for v in sh.split(":"))
        t = make_device_inputs(M, K, N, 11, dev)
        out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
        res = {}
        for dyn in (int(v) for v in a.dyn.split(",")):
            for g in (int(v) for v in a.groups.split(",")):
                h = ffn.FusedFFN(dev)
                h.set_option(ffn.OPT_DYNAMIC, dyn)
                h.set_option(ffn.OPT_GROUP_M, g)
                res[f"{dyn}/g{g}"] = time_cfg(h, t["x"], t, out, a.steps, flush)
                del h
        flops = 4.0 * M * K * N
        print(f"{M}x{K}x{N} plan {ffn.plan_config(M, K, N)}: " +
              " ".join(f"dyn{k}={v:.1f}us ({flops / v / 1e6:.0f} TF/s)" for k, v in res.items()), flush=True)
        del t, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
