"""Per-CTA timeline (CUASM_OPT_TRACE) of the decode shards after an L2 flush: where the ~20 us go.

    python scripts/trace_decode.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs
from scripts.trace_gemm import SLOTS

dev = torch.device("cuda:0")
flush = bench.L2Flush(dev)
for (M, K, N, cs) in [(16, 4096, 1376, 0), (16, 4096, 1376, 8), (16, 4096, 1376, 1), (16, 4096, 11008, 0),
                      (16, 8192, 3584, 0)]:
    t = make_device_inputs(M, K, N, 1, dev)
    out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    h = ffn.FusedFFN(dev)
    if cs:
        h.set_option(ffn.OPT_CSPLIT, cs)
    for _ in range(3):
        h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
    h.set_option(ffn.OPT_TRACE, 1)
    for rep in range(2):
        torch.cuda.synchronize()
        if not os.environ.get("NOFLUSH"):
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
        b.record()
        torch.cuda.synchronize()
    tr = h.trace_read().double()
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    print((M, K, N), "csplit_opt", cs, "plan", ffn.plan_config(M, K, N), "ctas", tr.shape[0],
          "event us", round(a.elapsed_time(b) * 1e3, 2))
    for i, name in enumerate(SLOTS):
        col = tr[:, i]
        col = col[col > 0]
        if col.numel():
            d = (col - t0) / 1e3
            print(f"   {name:14s} min {d.min().item():7.2f} med {d.median().item():7.2f} max {d.max().item():7.2f} us")
    if cs != 1 and ffn.plan_config(M, K, N)[3]:
        c = tr[:, 12:16]
        print("   csplit reduce cycles (copy, acquired, loaded, stored): med", c.median(0).values.tolist(), "max",
              c.max(0).values.tolist())
        continue
    c = tr[:, 12:16]
    c = c[c[:, 1] > 0]
    if c.numel():
        print("   mma cycles/kblock med", round((c[:, 0] / c[:, 1]).median().item(), 1), "wait_full/kb",
              round((c[:, 2] / c[:, 1]).median().item(), 1), "kblocks med", c[:, 1].median().item())
