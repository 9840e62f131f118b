"""Why the autotuner's per-forward time and bench.py's differ for some plans: the same forward
(CUDA graph) timed after (a) bench.L2Flush (256 MiB memset + torch sum of another 256 MiB) with a GPU
sleep first, (b) the same without the sleep, (c) a memset + a plain-load read (the tuner's flush)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs

dev = torch.device("cuda:0")
flush = bench.L2Flush(dev)
w = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
r = torch.ones(64 << 20, dtype=torch.float32, device=dev)


def flush_max():
    w.zero_()
    flush.sink = r.max()


def run(g, fl, sleep, n=40):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    torch.cuda.synchronize()
    if sleep:
        torch.cuda._sleep(int(1e8))
    for e0, e1 in ev:
        fl()
        e0.record()
        g.replay()
        e1.record()
    torch.cuda.synchronize()
    ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    return round(sum(ms) / len(ms) * 1e3, 2)


K, N = 4096, 1376
for M, opts in ((48, {}), (48, {ffn.OPT_CSPLIT: 1, ffn.OPT_TILE_BN: 128}), (16, {}), (2048, {})):
    t = make_device_inputs(M, K, N, 3, dev)
    out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    h = ffn.FusedFFN(dev)
    for k, v in opts.items():
        h.set_option(k, v)
    for _ in range(3):
        h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
    print(M, opts, "flush+sleep", run(g, flush.zero_, True), "flush no sleep", run(g, flush.zero_, False),
          "memset+max", run(g, flush_max, True), "no flush", run(g, lambda: None, True), flush=True)
