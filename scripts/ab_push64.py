"""A/B of the cluster split-K at 33..64 rows (64-output 1-SM tiles, forced S): push form (new lib)
vs pull form (old lib), L2-flushed bench-protocol step times.
python scripts/ab_push64.py LABEL [MxKxN,...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json
import torch

import bench
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs
from scripts.tune import time_cfg

dev = torch.device("cuda:0")
flush = bench.L2Flush(dev)
res = {}
SHAPES = ((33, 4096, 1376), (48, 4096, 1376), (64, 4096, 1376), (64, 4096, 2752), (48, 8192, 3584))
if len(sys.argv) > 2:
    SHAPES = tuple(tuple(int(v) for v in sh.split("x")) for sh in sys.argv[2].split(","))
for (M, K, N) in SHAPES:
    t = make_device_inputs(M, K, N, 3, dev)
    out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    for S in (2, 3, 4):
        h = ffn.FusedFFN(dev)
        h.set_variant(ffn.VARIANT_1SM)
        h.set_option(ffn.OPT_TILE_BN, 64)
        h.set_option(ffn.OPT_CSPLIT, S)
        res[f"{M}x{K}x{N}/S{S}"] = round(time_cfg(h, t["x"], t, out, 30, flush), 2)
print(sys.argv[1], json.dumps(res), flush=True)
