"""Per-CTA-pair finish times (last MMA issue, exit) of one traced launch, sorted: how much a schedule
that gave the slowest pairs less work could save (2048x4096x1376 by default)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs

dev = torch.device("cuda:0")
M, K, N = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "2048x4096x1376").split("x"))
t = make_device_inputs(M, K, N, 1, dev)
out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
wbuf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
rbuf = torch.ones(64 << 20, dtype=torch.float32, device=dev)
h = ffn.FusedFFN(dev)
for _ in range(3):
    h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
h.set_option(ffn.OPT_TRACE, 1)
for rep in range(3):
    wbuf.zero_()
    rbuf.sum()
    torch.cuda.synchronize()
    torch.cuda._sleep(int(1e8))
    h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
    tr = h.trace_read().double()
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    lm = ((tr[0::2, 3] - t0) / 1e3)  # leader CTAs: last MMA issue
    ex = ((tr[:, 6] - t0) / 1e3).view(-1, 2).max(1).values
    lm_s, _ = lm.sort()
    ex_s, _ = ex.sort()
    print(f"rep {rep}: pairs {lm.numel()}; last MMA (sorted, us): " + " ".join(f"{v:.1f}" for v in lm_s.tolist()[-12:]))
    print(f"         exit (sorted, top 12): " + " ".join(f"{v:.1f}" for v in ex_s.tolist()[-12:]) +
          f" | median {ex_s[len(ex_s) // 2]:.1f}", flush=True)
