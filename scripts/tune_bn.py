"""Time the SwiGLU tile widths (CUASM_OPT_TILE_BN) x schedules of the 2-SM kernel on the
shapes the widths are for (tensor-parallel shards of the 7B / 70B FFN, the crossover
region): the data behind bn_frac() and the width choice in csrc/cuasm_ffn.cu
plan_config (the paper's tile-config search, done offline).

    python scripts/tune_bn.py [--shapes M:K:N,...] [--out profiles/r02/tune_bn.json]
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

DEFAULT = ("2048:4096:1376,2048:4096:2752,2048:4096:5504,2048:4096:11008,1024:4096:1376,1024:4096:2752,"
           "512:4096:11008,384:4096:11008,256:4096:11008,4096:8192:3584,4096:8192:7168,16384:4096:1376")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default=DEFAULT)
    ap.add_argument("--bns", default="128,112,96,80,64")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    flush = bench.L2Flush(dev)
    res = []
    for sh in a.shapes.split(","):
        M, K, N = (int(v) for v in sh.split(":"))
        t = make_device_inputs(M, K, N, 11, dev)
        out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
        row = {"M": M, "K": K, "N": N, "auto": None, "plan": list(ffn.plan_config(M, K, N)), "us": {}}
        h = ffn.FusedFFN(dev)
        row["auto"] = time_cfg(h, t["x"], t, out, a.steps, flush)
        del h
        for bn in (int(b) for b in a.bns.split(",")):
            for sch, name in ((1, "dp"), (0, "auto")):
                h = ffn.FusedFFN(dev)
                h.set_variant(ffn.VARIANT_2SM)
                h.set_option(ffn.OPT_TILE_BN, bn)
                h.set_option(ffn.OPT_SCHEDULE, sch)
                row["us"][f"{bn}-{name}"] = round(time_cfg(h, t["x"], t, out, a.steps, flush), 2)
                del h
        flops = 4.0 * M * K * N
        best = min(row["us"], key=row["us"].get)
        print(f"{M}x{K}x{N}: auto {row['auto']:.1f} us plan {row['plan']} | best {best} {row['us'][best]:.1f} us "
              f"({flops / row['us'][best] / 1e6:.0f} TF/s) | " +
              " ".join(f"{k}={v:.1f}" for k, v in row["us"].items()), flush=True)
        res.append(row)
        del t, out
        torch.cuda.empty_cache()
    if a.out:
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
