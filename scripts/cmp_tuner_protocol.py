import sys, os
sys.path.insert(0, os.getcwd())
import torch, bench
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs
from scripts.tune import time_cfg
dev = torch.device("cuda:0"); flush = bench.L2Flush(dev)
K, N = 4096, 1376
for M in (48, 64, 96, 128):
    t = make_device_inputs(M, K, N, 3, dev); out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    h = ffn.FusedFFN(dev)
    a = time_cfg(h, t["x"], t, out, 30, flush)
    h2 = ffn.FusedFFN(dev)
    plan, us = h2.tune(t["x"], t["g"], t["w1"], t["w3"], 1e-6, warmup=3, iters=10)
    log = dict((str(list(p)), u) for p, u in h2.tune_log())
    b = time_cfg(h2, t["x"], t, out, 30, flush)
    # sweep-style: one handle prepared for the 128-wide pack, x sliced from a bigger tensor
    base = make_device_inputs(2048, K, N, 7, dev)
    h3 = ffn.FusedFFN(dev); h3.prepare(base["g"], base["w1"], base["w3"])
    x = base["x"][:M].contiguous()
    c = time_cfg(h3, x, base, out, 30, flush)
    print(M, ffn.plan_config(M, K, N), 'time_cfg model', round(a, 2), '| tuner says model', log.get(str(list(ffn.plan_config(M, K, N)))), 'best', plan, round(us, 2), '| time_cfg tuned', round(b, 2), '| sweep-style', round(c, 2), flush=True)
