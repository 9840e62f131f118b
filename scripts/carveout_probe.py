"""Is part of the per-step floor the SM's shared-memory carveout switch between the flush kernels
(torch fill + sum: little shared memory) and our GEMM (~227 KB)?  Time the same CUDA-graph step after
(a) bench.L2Flush, (b) an L2 flush made of one of our own FFN forwards over ~300 MB of unrelated
weights (same carveout as the step), (c) no flush."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs

dev = torch.device("cuda:0")
flush = bench.L2Flush(dev)
# the "FFN flush": a decode-shaped forward streaming 2 x 18432 x 4096 bf16 = 302 MB of weights
fw = make_device_inputs(16, 4096, 18432, 9, dev)
fout = torch.empty((16, 18432), dtype=torch.bfloat16, device=dev)
hf = ffn.FusedFFN(dev)
for _ in range(3):
    hf.forward(fw["x"], fw["g"], fw["w1"], fw["w3"], 1e-6, out=fout)
gf = torch.cuda.CUDAGraph()
with torch.cuda.graph(gf):
    hf.forward(fw["x"], fw["g"], fw["w1"], fw["w3"], 1e-6, out=fout)


def run(g, fl, n=60):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    torch.cuda.synchronize()
    torch.cuda._sleep(int(1e8))
    for e0, e1 in ev:
        fl()
        e0.record()
        g.replay()
        e1.record()
    torch.cuda.synchronize()
    ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    return round(sum(ms) / len(ms) * 1e3, 2)


for (M, K, N) in ((16, 4096, 1376), (16, 4096, 11008), (2048, 4096, 1376), (512, 2048, 512)):
    t = make_device_inputs(M, K, N, 3, dev)
    out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    h = ffn.FusedFFN(dev)
    for _ in range(3):
        h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
    print(f"{M}x{K}x{N}: torch flush {run(g, flush.zero_)} | FFN flush {run(g, gf.replay)} | "
          f"no flush {run(g, lambda: None)} us", flush=True)
