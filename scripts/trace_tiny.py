"""Per-CTA timeline (CUASM_OPT_TRACE) of tiny launches: the fixed latency of one tile (prologue, first MMA, epilogue)."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs
from scripts.trace_gemm import SLOTS
dev = torch.device("cuda:0")
for dt, (M, K, N) in [(torch.float32, (16, 64, 128)), (torch.bfloat16, (16, 64, 128)), (torch.bfloat16, (16, 4096, 256))]:
    t = make_device_inputs(M, K, N, 1, dev, dtype=dt)
    out = torch.empty((M, N), dtype=dt, device=dev)
    h = ffn.FusedFFN(dev, dt)
    for _ in range(3): h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
    h.set_option(ffn.OPT_TRACE, 1)
    torch.cuda.synchronize(); torch.cuda._sleep(int(1e8))
    h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
    tr = h.trace_read().double()
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    print(dt, M, K, N, "ctas", tr.shape[0])
    for i, name in enumerate(SLOTS):
        col = tr[:, i]; col = col[col > 0]
        if col.numel(): print(f"   {name:14s} {(col.min() - t0).item() / 1e3:8.2f} {(col.max() - t0).item() / 1e3:8.2f} us")
