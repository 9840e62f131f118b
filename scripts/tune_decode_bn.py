"""Decode shards: the 128-output tile's planned cluster split-K against the 1-SM
64-output tile split S ways (CUASM_OPT_TILE_BN = 64, CUASM_OPT_CSPLIT = S), bench
protocol (L2 flushed before every step, CUDA events).

    python scripts/tune_decode_bn.py [--shapes M:K:N,...] [--splits 2,3,4,6,8]
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

DEFAULT = ("16:4096:1376,16:4096:2752,16:4096:5504,16:4096:11008,16:8192:3584,16:8192:7168,32:4096:1376,"
           "1:4096:1376,16:8192:14336")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default=DEFAULT)
    ap.add_argument("--splits", default="1,2,3,4,6,8")
    ap.add_argument("--steps", type=int, default=30)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    flush = bench.L2Flush(dev)
    for sh in a.shapes.split(","):
        M, K, N = (int(v) for v in sh.split(":"))
        t = make_device_inputs(M, K, N, 11, dev)
        out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
        res = {}
        h = ffn.FusedFFN(dev)
        res["auto"] = time_cfg(h, t["x"], t, out, a.steps, flush)
        del h
        for S in (int(v) for v in a.splits.split(",")):
            if (N + 63) // 64 * S > 148:
                continue
            h = ffn.FusedFFN(dev)
            h.set_option(ffn.OPT_TILE_BN, 64)
            h.set_variant(ffn.VARIANT_1SM)
            h.set_option(ffn.OPT_CSPLIT, S)
            res[f"64/S{S}"] = time_cfg(h, t["x"], t, out, a.steps, flush)
            del h
        bytes_ = 2.0 * (M * K + 2 * K * N + M * N)
        best = min(res, key=res.get)
        print(f"{M}x{K}x{N} plan {ffn.plan_config(M, K, N)} | best {best} {res[best]:.2f} us "
              f"({bytes_ / res[best] / 1e3:.0f} GB/s) | " + " ".join(f"{k}={v:.2f}" for k, v in res.items()),
              flush=True)
        del t, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
