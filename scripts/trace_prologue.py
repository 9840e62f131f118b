"""Producer prologue timeline from a library built with -DCUASM_DIAG_PROLOGUE=1 (trace slots
12 after the CTA-pair barrier, 13 after the first early weight load, 14 after all of them, 15 after
griddepcontrol.wait; 0 entry, 1 first x TMA issued, 4 epilogue start), per CTA relative to the
earliest entry.

    python scripts/trace_prologue.py [MxKxN,...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs

dev = torch.device("cuda:0")
wbuf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
rbuf = torch.ones(64 << 20, dtype=torch.float32, device=dev)
for shp in (sys.argv[1] if len(sys.argv) > 1 else "2048x4096x1376,2048x4096x11008").split(","):
    M, K, N = map(int, shp.split("x"))
    t = make_device_inputs(M, K, N, 1, dev)
    out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    h = ffn.FusedFFN(dev)
    for _ in range(3):
        h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
    h.set_option(ffn.OPT_TRACE, 1)
    wbuf.zero_()
    rbuf.sum()
    torch.cuda.synchronize()
    torch.cuda._sleep(int(1e8))
    h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
    tr = h.trace_read().double()
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    print(shp, ffn.plan_config(M, K, N))
    for slot, name in [(0, "entry"), (12, "pair barrier done"), (13, "1st early W load"), (14, "early W loads done"),
                       (15, "griddep.wait done"), (1, "first x TMA issued"), (4, "epilogue start")]:
        c = tr[:, slot]
        c = c[c > 0]
        if c.numel():
            r = (c - t0) / 1e3
            print(f"   {name:20s} min {r.min():6.2f} med {r.median():6.2f} max {r.max():6.2f} us")
