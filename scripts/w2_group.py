"""Down projection W2 (cuasm_gemm_act identity, 2048 x 11008 -> 4096): rasterisation
group and schedule vs time (L2 flushed) -- with --ncu, 3 launches per group for a dram__bytes launch list.

    python scripts/w2_group.py [--ncu]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import bench
import paper_2501_08071_b200 as ffn

dev = torch.device("cuda:0")
flush = bench.L2Flush(dev)
M, K, N = 2048, 11008, 4096
x = (torch.randn(M, K, device=dev) * 0.5).to(torch.bfloat16)
w = (torch.randn(N, K, device=dev) / K ** 0.5).to(torch.bfloat16)
out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
CFGS = [(g, 0) for g in (0, 1, 2, 4, 8)] + [(0, sch) for sch in (1, 2, 3)]
for g, sch in CFGS:
    h = ffn.FusedFFN(dev)
    h.set_option(ffn.OPT_GROUP_M, g)
    h.set_option(ffn.OPT_SCHEDULE, sch)
    for _ in range(3):
        flush.zero_()
        h.gemm_act(x, w, "identity", out=out)
    torch.cuda.synchronize()
    if "--ncu" in sys.argv:
        print(json.dumps({"group_m": g, "schedule": sch}), flush=True)
        continue
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    torch.cuda._sleep(int(1e8))
    for a, b in ev:
        flush.zero_()
        a.record()
        h.gemm_act(x, w, "identity", out=out)
        b.record()
    torch.cuda.synchronize()
    us = sum(a.elapsed_time(b) for a, b in ev) / len(ev) * 1e3
    print(json.dumps({"group_m": g, "schedule": sch, "us": round(us, 2), "plan": ffn.plan_config(M, K, N, "gemm")}),
          flush=True)
