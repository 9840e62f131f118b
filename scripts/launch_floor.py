"""Fixed per-step cost of the bench protocol: event -> (L2 flush already done)
-> a trivial kernel -> event, vs the same with our decode forward.  Separates
launch/turnaround latency from kernel time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs

dev = torch.device("cuda:0")
flush = bench.L2Flush(dev)
tiny = torch.zeros(1, device=dev)
t = make_device_inputs(16, 4096, 11008, 3, dev)
out = torch.empty((16, 11008), dtype=torch.bfloat16, device=dev)
h = ffn.FusedFFN(dev)
h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)


def med(fn, n=50, do_flush=True):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    torch.cuda.synchronize()
    torch.cuda._sleep(int(1e8))
    for a, b in ev:
        if do_flush:
            flush.zero_()
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)
    return ms[len(ms) // 2] * 1e3


g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
print(f"empty event pair (after flush):           {med(lambda: None):7.2f} us")
print(f"trivial fill kernel (after flush):        {med(lambda: tiny.zero_()):7.2f} us")
print(f"decode forward, graph (after flush):      {med(g.replay):7.2f} us")
print(f"decode forward, graph (no flush):         {med(g.replay, do_flush=False):7.2f} us")
for n in (2, 4, 8):
    def many(n=n):
        for _ in range(n):
            g.replay()
    print(f"{n} decode forwards back to back / {n} (no flush): {med(many, do_flush=False) / n:7.2f} us")

# launch modes of the same decode forward, each after a flush, own event pair
def eager():
    h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)


print(f"decode forward, eager launch (after flush):    {med(eager):7.2f} us")
h.set_option(ffn.OPT_PDL, 0)
print(f"decode forward, eager, no PDL (after flush):   {med(eager):7.2f} us")
g2 = torch.cuda.CUDAGraph()
with torch.cuda.graph(g2):
    eager()
print(f"decode forward, graph, no PDL (after flush):   {med(g2.replay):7.2f} us")
h.set_option(ffn.OPT_PDL, 1)
# the flush's last kernel is a 256 MiB read; a tiny kernel between it and the
# start event separates "previous kernel drain" from the event pair itself
print(f"trivial kernel, then event pair around forward: {med(lambda: g.replay()):7.2f} us")
