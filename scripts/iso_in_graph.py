"""Per-step timing floor of the iso protocol: the event pair and the forward's
launch outside a CUDA graph (bench.py today) vs flush + event pair + forward all
captured in one graph (event record nodes, cudaEventRecordExternal), so the span
holds the forward's device time plus one graph-node hand-over only.

    python scripts/iso_in_graph.py            (on a GPU box)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs

dev = torch.device("cuda:0")
flush = bench.L2Flush(dev)
tiny = torch.zeros(1, device=dev)
R = 10  # steps per graph


def eager_pairs(fn, n=60):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    torch.cuda.synchronize()
    torch.cuda._sleep(int(1e8))
    for a, b in ev:
        flush.zero_()
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)
    return ms[len(ms) // 2] * 1e3, sum(ms) / len(ms) * 1e3


def graph_pairs(fn, reps=6):
    ev = [(torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True))
          for _ in range(R)]
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for a, b in ev:
            flush.zero_()
            a.record()
            fn()
            b.record()
    ms = []
    for _ in range(reps):
        g.replay()
        torch.cuda.synchronize()
        ms += [a.elapsed_time(b) for a, b in ev]
    ms.sort()
    return ms[len(ms) // 2] * 1e3, sum(ms) / len(ms) * 1e3


print(f"{'':44s} {'eager pair med/mean':>22s} {'in-graph med/mean':>22s}")
m1 = eager_pairs(lambda: None)
m2 = graph_pairs(lambda: None)
print(f"{'empty event pair':44s} {m1[0]:9.2f} {m1[1]:9.2f}    {m2[0]:9.2f} {m2[1]:9.2f}")
m1 = eager_pairs(lambda: tiny.zero_())
m2 = graph_pairs(lambda: tiny.zero_())
print(f"{'trivial kernel':44s} {m1[0]:9.2f} {m1[1]:9.2f}    {m2[0]:9.2f} {m2[1]:9.2f}")

for (M, K, N) in [(16, 4096, 11008), (16, 4096, 1376), (2048, 4096, 1376), (2048, 4096, 11008), (384, 4096, 11008)]:
    t = make_device_inputs(M, K, N, 3, dev)
    out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    h = ffn.FusedFFN(dev)

    def fwd():
        h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)

    fwd()
    gf = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gf):
        fwd()
    gf.replay()
    m1 = eager_pairs(gf.replay)
    m2 = graph_pairs(fwd)
    print(f"{f'ffn {M}x{K}x{N}':44s} {m1[0]:9.2f} {m1[1]:9.2f}    {m2[0]:9.2f} {m2[1]:9.2f}", flush=True)
