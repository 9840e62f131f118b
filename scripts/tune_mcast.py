"""A/B of 4-CTA multicast clusters (CUASM_OPT_MCAST) against the planned kernel, per shape, bench
protocol (L2 flushed before every step, CUDA events); both with the plan's tile width.

    python scripts/tune_mcast.py [--shapes M:K:N,...]
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

DEFAULT = ("2048:4096:11008,2048:4096:1376,2048:4096:2752,2048:4096:5504,4096:8192:3584,4096:8192:28672,"
           "4096:4096:11008,1024:4096:11008")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default=DEFAULT)
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    flush = bench.L2Flush(dev)
    for sh in a.shapes.split(","):
        M, K, N = (int(v) for v in sh.split(":"))
        t = make_device_inputs(M, K, N, 11, dev)
        out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
        plan = ffn.plan_config(M, K, N)
        res = {}
        for name, opts in (("plan", {}), ("plan-dp", {ffn.OPT_SCHEDULE: 1}), ("mcast", {ffn.OPT_MCAST: 1})):
            h = ffn.FusedFFN(dev)
            h.set_option(ffn.OPT_TILE_BN, plan[4])
            for k, v in opts.items():
                h.set_option(k, v)
            res[name] = time_cfg(h, t["x"], t, out, a.steps, flush)
            del h
        flops = 4.0 * M * K * N
        print(f"{M}x{K}x{N} plan {plan}: " + " ".join(f"{k}={v:.1f}us ({flops / v / 1e6:.0f} TF/s)" for k, v in res.items()),
              flush=True)
        del t, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
