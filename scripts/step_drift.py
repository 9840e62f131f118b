"""Per-step time drift over a long run of the bench protocol (7B prefill, L2 flushed before each
step, CUDA-graph step): mean per 50-step block after W warm-up steps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs

dev = torch.device("cuda:0")
flush = bench.L2Flush(dev)
M, K, N = 2048, 4096, 11008
t = make_device_inputs(M, K, N, 3, dev)
out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
h = ffn.FusedFFN(dev)
for _ in range(3):
    h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
for W in (int(a) for a in (sys.argv[1] if len(sys.argv) > 1 else "10,100").split(",")):
    torch.cuda.synchronize()
    for _ in range(W):
        flush.zero_()
        g.replay()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(600)]
    torch.cuda.synchronize()
    torch.cuda._sleep(int(2e8))
    for a, b in ev:
        flush.zero_()
        a.record()
        g.replay()
        b.record()
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) * 1e3 for a, b in ev]
    print(f"W={W}: " + " ".join(f"{sum(ms[i:i + 50]) / 50:.1f}" for i in range(0, 600, 50)), flush=True)
    torch.cuda._sleep(int(2e9))  # ~1 s idle-ish spin between configurations
    torch.cuda.synchronize()
