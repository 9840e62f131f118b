"""Tall tiles (CUASM_OPT_TALL) vs the other plans in the crossover region (configs[4]:
K = 4096, N = 11008, M = 257..384), per-step median with the L2 flushed (scripts/tune.py
time_cfg): the data behind kTallFrac in csrc/cuasm_ffn.cu plan_config_raw.

    python scripts/tune_tall.py [--ms 257,288,...] [--out profiles/r02/tall/tune_tall.json]
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
    ap.add_argument("--ms", default="257,288,320,352,384")
    ap.add_argument("--K", type=int, default=4096)
    ap.add_argument("--N", type=int, default=11008)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    flush = bench.L2Flush(dev)
    rows = []
    for M in (int(m) for m in a.ms.split(",")):
        t = make_device_inputs(M, a.K, a.N, 11, dev)
        out = torch.empty((M, a.N), dtype=torch.bfloat16, device=dev)
        row = {"M": M, "K": a.K, "N": a.N, "plan": list(ffn.plan_config(M, a.K, a.N)), "us": {}}
        for name, opts in (("auto", {}), ("tall", {ffn.OPT_TALL: 2}), ("no-tall", {ffn.OPT_TALL: 1}),
                           ("1sm-128", {ffn.OPT_TALL: 1, ffn.OPT_VARIANT: ffn.VARIANT_1SM}),
                           ("2sm-80", {ffn.OPT_TALL: 1, ffn.OPT_VARIANT: ffn.VARIANT_2SM, ffn.OPT_TILE_BN: 80})):
            h = ffn.FusedFFN(dev)
            for k, v in opts.items():
                h.set_option(k, v)
            row["us"][name] = round(time_cfg(h, t["x"], t, out, a.steps, flush), 2)
            del h
        flops = 4.0 * M * a.K * a.N
        best = min(row["us"], key=row["us"].get)
        print(f"{M}x{a.K}x{a.N} plan {row['plan']} | best {best} {row['us'][best]} us "
              f"({flops / row['us'][best] / 1e6:.0f} TF/s) | " +
              " ".join(f"{k}={v}" for k, v in row["us"].items()), flush=True)
        rows.append(row)
    if a.out:
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        with open(a.out, "w") as f:
            json.dump({"unit": "us per forward (median, L2 flushed)", "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
