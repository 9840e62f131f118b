"""A/B timing of two builds of the library: mean L2-flushed step time per shape.

    python scripts/ab_lib.py LABEL [MxKxN,...]   (swap paper_2501_08071_b200/libcuasm_ffn.so between runs)
"""
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch, bench
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs
dev = torch.device("cuda:0"); flush = bench.L2Flush(dev)
res = {}
for shp in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["2048x4096x11008", "4096x4096x11008", "4096x8192x28672"]):
    M, K, N = map(int, shp.split("x"))
    t = make_device_inputs(M, K, N, 3, dev); out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    h = ffn.FusedFFN(dev)
    for _ in range(3): h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g): h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
    n = 30 if M * N < 1e8 else 10
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    torch.cuda.synchronize(); torch.cuda._sleep(int(1e8))
    for a, b in ev:
        flush.zero_(); a.record(); g.replay(); b.record()
    torch.cuda.synchronize()
    res[shp] = round(sum(a.elapsed_time(b) for a, b in ev) / n * 1e3, 2)
    del g, t, out, h; torch.cuda.empty_cache()
print(sys.argv[1], json.dumps(res), flush=True)
