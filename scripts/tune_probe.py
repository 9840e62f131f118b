"""The autotuner (cuasm_ffn_tune) on the bench workloads and shards: the measured best per shape
vs the cost model's plan, and every candidate's time (back-to-back forwards, no L2 flush).

    python scripts/tune_probe.py
"""
import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs
dev = torch.device("cuda:0")
FLUSH = os.environ.get("NOFLUSH") is None
for (M, K, N) in [(2048, 4096, 11008), (16, 4096, 11008), (2048, 4096, 1376), (16, 4096, 1376), (384, 4096, 11008),
                  (512, 2048, 512), (4096, 8192, 3584), (2048, 4096, 2752), (2048, 4096, 5504)]:
    t = make_device_inputs(M, K, N, 3, dev)
    h = ffn.FusedFFN(dev)
    t0 = time.time()
    plan, us = h.tune(t["x"], t["g"], t["w1"], t["w3"], 1e-6, warmup=10, iters=30, flush_l2=FLUSH)
    print(f"{M}x{K}x{N}: model {ffn.plan_config(M, K, N)} | tuned {plan} {us:.2f} us (search {time.time() - t0:.1f} s)", flush=True)
    print(h.tuned_export().strip(), flush=True)
    for pl, t_us in sorted(h.tune_log(), key=lambda r: r[1] if r[1] is not None else 1e9):
        print(f"      {str(pl):34s} {'skipped' if t_us is None else f'{t_us:8.2f} us'}")
