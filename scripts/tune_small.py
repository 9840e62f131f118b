"""The paper's own fused_ff shape (B, M, N, K = 1, 512, 512, 2048) and other
latency-bound shapes: stream-K split widths (CUASM_OPT_SK_SPLIT) x tile widths, L2-flushed step
medians (scripts/tune.py time_cfg).

    python scripts/tune_small.py [M:K:N,...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs
from scripts.tune import time_cfg

dev = torch.device("cuda:0")
flush = bench.L2Flush(dev)
for sh in (sys.argv[1] if len(sys.argv) > 1 else "512:2048:512,1024:2048:512,512:2048:1024").split(","):
    M, K, N = (int(v) for v in sh.split(":"))
    t = make_device_inputs(M, K, N, 5, dev)
    out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    res = {"auto": round(time_cfg(ffn.FusedFFN(dev), t["x"], t, out, 30, flush), 2)}
    for v, bn in ((ffn.VARIANT_2SM, 64), (ffn.VARIANT_2SM, 128), (ffn.VARIANT_1SM, 128), (ffn.VARIANT_1SM, 64)):
        for split in (2, 3, 4, 6, 8):
            h = ffn.FusedFFN(dev)
            h.set_variant(v)
            h.set_option(ffn.OPT_TILE_BN, bn)
            h.set_option(ffn.OPT_SCHEDULE, ffn.SCHEDULE_STREAM_K_ALL)
            h.set_option(ffn.OPT_SK_SPLIT, split)
            try:
                res[f"{'2sm' if v == ffn.VARIANT_2SM else '1sm'}-{bn}-sk{split}"] = round(
                    time_cfg(h, t["x"], t, out, 30, flush), 2)
            except ffn.CuasmError as e:
                res[f"{'2sm' if v == ffn.VARIANT_2SM else '1sm'}-{bn}-sk{split}"] = str(e)[:40]
    best = min((k for k in res if isinstance(res[k], float)), key=res.get)
    print(f"{M}x{K}x{N}: plan {ffn.plan_config(M, K, N)} best {best} {res[best]} us | {res}", flush=True)
