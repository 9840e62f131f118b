"""Decode-shard launches for an ncu A/B (kernel durations, cold L2 per launch under ncu's
default cache control):  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python scripts/ncu_ab_decode.py  -> one NVTX-free launch sequence, labelled by order.

Order: for each shape, for each csplit setting in CS, REPS launches.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs

SHAPES = [(16, 4096, 1376), (16, 4096, 2752), (16, 8192, 3584)][:int(os.environ.get("NSHAPES", "3"))]
if os.environ.get("SHAPES"):  # e.g. SHAPES=16x4096x5504,32x4096x1376
    SHAPES = [tuple(int(v) for v in sh.split("x")) for sh in os.environ["SHAPES"].split(",")]
CS = [int(c) for c in os.environ.get("CS", "1,4,8").split(",")]
REPS = int(os.environ.get("REPS", "10"))
dev = torch.device("cuda:0")
for (M, K, N) in SHAPES:
    t = make_device_inputs(M, K, N, 1, dev)
    out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    for cs in CS:
        h = ffn.FusedFFN(dev)
        if cs >= 0:
            h.set_option(ffn.OPT_CSPLIT, cs)
        else:  # -1: the few-tile stream-K plan (1-SM, split 3 ways), no cluster split
            h.set_option(ffn.OPT_CSPLIT, 1)
            h.set_variant(ffn.VARIANT_1SM)
            h.set_option(ffn.OPT_SCHEDULE, ffn.SCHEDULE_STREAM_K_TAIL)
        h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)  # packs W13 (extra launches)
        torch.cuda.synchronize()
        print(f"MARK {M}x{K}x{N} cs{cs}", flush=True)
        for _ in range(REPS):
            h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
        torch.cuda.synchronize()
        del h
