"""L2 residency study for the dual GEMM: rasterisation group (CUASM_OPT_GROUP_M)
x TMA L2 eviction policies (CUASM_OPT_L2_POLICY) per shape.

    python scripts/l2_study.py --time            # L2-flushed median time per config
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:ffn_dual_gemm \\
        python scripts/l2_study.py --ncu         # 3 launches per config; the 3rd is the one to read
Config order is printed first (and is deterministic) so the ncu launch list maps back to it.
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

SHAPES = ["4096x8192x28672", "4096x8192x3584", "2048x4096x11008"]
GROUPS = [0, 4, 16]
POLS = [2, 0, 2 | (1 << 2), 0 | (1 << 2)]   # x last/W normal, both normal, x last/W first, x normal/W first


def configs():
    if os.environ.get("L2_STUDY_SHAPES"):
        pols = [int(x) for x in os.environ.get("L2_STUDY_POLS", "2").split(",")]
        return [(s, 0, pol) for s in os.environ["L2_STUDY_SHAPES"].split(",") for pol in pols]
    return [(s, g, p) for s in SHAPES for g in GROUPS for p in POLS]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--time", action="store_true")
    ap.add_argument("--ncu", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    flush = bench.L2Flush(dev)
    cur, t, out = None, None, None
    for i, (shp, g, pol) in enumerate(configs()):
        if shp != cur:
            M, K, N = map(int, shp.split("x"))
            t = out = None
            torch.cuda.empty_cache()
            t = make_device_inputs(M, K, N, 11, dev)
            out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
            cur = shp
        h = ffn.FusedFFN(dev)
        h.set_option(ffn.OPT_GROUP_M, g)
        h.set_option(ffn.OPT_L2_POLICY, pol)
        h.prepare(t["g"], t["w1"], t["w3"])
        rec = {"i": i, "shape": shp, "group_m": g, "l2pol": pol}
        if a.time:
            rec["us"] = round(time_cfg(h, t["x"], t, out, 10, flush), 2)
        if a.ncu:
            for _ in range(3):
                flush.zero_()
                h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
            torch.cuda.synchronize()
        print(json.dumps(rec), flush=True)
        del h


if __name__ == "__main__":
    main()
