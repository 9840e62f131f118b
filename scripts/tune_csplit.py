"""Cluster split-K (CUASM_OPT_CSPLIT) vs the auto plan on few-tile shapes; (time us, CTAs launched)."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch, bench
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs
from scripts.tune import time_cfg
dev = torch.device("cuda:0"); flush = bench.L2Flush(dev)
for (M, K, N) in [(16, 4096, 1376), (512, 2048, 512), (16, 4096, 2752), (128, 4096, 1376), (16, 8192, 3584), (64, 4096, 1376), (256, 4096, 1376)]:
    t = make_device_inputs(M, K, N, 3, dev); out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    res = {"auto": round(time_cfg(ffn.FusedFFN(dev), t["x"], t, out, 30, flush), 2)}
    for S in (2, 3, 4, 6, 8):
        h = ffn.FusedFFN(dev); h.set_variant(1); h.set_option(ffn.OPT_CSPLIT, S); h.set_option(ffn.OPT_SCHEDULE, 1)
        us = round(time_cfg(h, t["x"], t, out, 30, flush), 2)
        h.set_option(ffn.OPT_TRACE, 1); h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out); torch.cuda.synchronize()
        res[f"cs{S}"] = (us, h.trace_read().shape[0])
    print((M, K, N), res, flush=True)
