"""Per-rank cost of the N-sharded (Megatron column) path, measured on ONE GPU.

With W1/W3 column-sharded over P ranks every rank runs the same
problem (M, K, N/P) on its own GPU, with no data-path collective, so the time
of an 8-GPU step is the time of rank 0's shard problem (plus skew).  This
script times those shard problems on a single B200 -- every (variant,
schedule) and the library's auto plan -- and reports the projected strong-
scaling efficiency T(1) / (P * T(N/P)) per BASELINE.json's scaling configs.
It is a projection (no NVLink, no rank skew, one box's clock), labelled so.

    python scripts/shard_projection.py [--out profiles/r01/shard_projection.json]
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
from paper_2501_08071_b200.tp import shard_bounds
from scripts.tune import CONFIGS, time_cfg

WORKLOADS = {"llama7b_prefill": (2048, 4096, 11008), "llama70b": (4096, 8192, 28672),
             "llama7b_decode": (16, 4096, 11008)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workloads", default="llama7b_prefill,llama70b,llama7b_decode")
    ap.add_argument("--ps", default="1,2,4,8")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--all-configs", action="store_true", help="also time every (variant, schedule)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    flush = bench.L2Flush(dev)
    report = {"unit": "us per forward (median, L2 flushed)", "note": "projection: rank 0's shard problem timed "
              "alone on one B200; efficiency = T(P=1) / (P * T(shard))", "rows": []}
    for wl in a.workloads.split(","):
        M, K, N = WORKLOADS[wl]
        t1 = None
        for P in [int(p) for p in a.ps.split(",")]:
            n0, n1 = shard_bounds(N, 0, P)
            Nl = n1 - n0
            t = make_device_inputs(M, K, Nl, 11, dev)
            out = torch.empty((M, Nl), dtype=torch.bfloat16, device=dev)
            r = {"workload": wl, "P": P, "M": M, "K": K, "N_per_rank": Nl, "plan": ffn.plan_config(M, K, Nl)}
            h = ffn.FusedFFN(dev)
            r["auto"] = round(time_cfg(h, t["x"], t, out, a.steps, flush), 2)
            if a.all_configs:
                for v, sch, name in CONFIGS:
                    hc = ffn.FusedFFN(dev)
                    hc.set_variant(v)
                    hc.set_option(ffn.OPT_SCHEDULE, sch)
                    r[name] = round(time_cfg(hc, t["x"], t, out, a.steps, flush), 2)
                    del hc
            if P == 1:
                t1 = r["auto"]
            if t1:
                r["projected_efficiency"] = round(t1 / (P * r["auto"]), 3)
            r["tflops_per_gpu"] = round(4.0 * M * K * Nl / (r["auto"] * 1e-6) / 1e12, 1)
            report["rows"].append(r)
            print(json.dumps(r), flush=True)
            del t, out, h
            torch.cuda.empty_cache()
    if a.out:
        with open(a.out, "w") as f:
            json.dump(report, f, indent=1)


if __name__ == "__main__":
    main()
