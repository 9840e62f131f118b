import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs
dev = torch.device("cuda:0")
for M in (48, 128, 256, 512):
    K, N = 4096, 1376
    t = make_device_inputs(M, K, N, 3, dev)
    h = ffn.FusedFFN(dev)
    plan, us = h.tune(t["x"], t["g"], t["w1"], t["w3"], 1e-6, warmup=5, iters=20, flush_l2=True)
    print(f"{M}x{K}x{N}: model {ffn.plan_config(M, K, N)} | tuned {plan} {us:.2f}", flush=True)
    for pl, t_us in sorted(h.tune_log(), key=lambda r: r[1] if r[1] is not None else 1e9)[:8]:
        print(f"      {str(pl):34s} {'skipped' if t_us is None else f'{t_us:8.2f} us'}")
