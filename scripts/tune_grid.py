"""The library's autotuner (cuasm_ffn_tune, L2-flushed, 3 interleaved rounds) over a grid of
tensor-parallel shard shapes: the measured best plan per shape next to the cost model's, written
as JSON rows (the data behind plan_config_raw's small-M shard rules).

    python scripts/tune_grid.py [--ms 1,...] [--kns 4096:1376,...] [--out profiles/r02/tune/grid.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ms", default="16,32,48,64,96,128,192,256,384,512,768,1024")
    ap.add_argument("--kns", default="4096:1376,4096:2752,4096:5504,8192:3584,8192:7168")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--out", default=None)
    ap.add_argument("--op", default="ffn", choices=["ffn", "gemm"], help="gemm: the GEMM + LeakyReLU op")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    rows = []
    for kn in a.kns.split(","):
        K, N = (int(v) for v in kn.split(":"))
        for M in (int(m) for m in a.ms.split(",")):
            t = make_device_inputs(M, K, N, 3, dev)
            h = ffn.FusedFFN(dev)
            if a.op == "ffn":
                plan, us = h.tune(t["x"], t["g"], t["w1"], t["w3"], 1e-6, warmup=a.warmup, iters=a.iters, flush_l2=True)
            else:
                plan, us = h.tune_gemm_act(t["x"], t["w1"], "leaky_relu", 0.01, warmup=a.warmup, iters=a.iters,
                                           flush_l2=True)
            log = {str(list(p)): u for p, u in h.tune_log()}
            model = list(ffn.plan_config(M, K, N, a.op))
            row = {"M": M, "K": K, "N": N, "model": model, "model_us": log.get(str(model)), "best": list(plan),
                   "best_us": round(us, 2), "all": {k: (round(v, 2) if v is not None else None) for k, v in log.items()}}
            rows.append(row)
            print(f"{M}x{K}x{N}: model {model} {row['model_us'] and round(row['model_us'], 2)} | best {list(plan)} "
                  f"{us:.2f}", flush=True)
            del h, t
            torch.cuda.empty_cache()
    if a.out:
        os.makedirs(os.path.dirname(a.out), exist_ok=True)
        json.dump({"unit": "us per forward, L2 flushed, best of 3 interleaved rounds", "rows": rows},
                  open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
