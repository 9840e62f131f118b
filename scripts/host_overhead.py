"""Host time per eager forward (no CUDA graph): the C-ABI call's host cost, which an eager decode
loop pays per layer.  python scripts/host_overhead.py LABEL"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2501_08071_b200 as ffn
from ffn_inputs import make_device_inputs

dev = torch.device("cuda:0")
res = {}
for (M, K, N) in ((16, 4096, 11008), (2048, 4096, 1376)):
    t = make_device_inputs(M, K, N, 3, dev)
    out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
    h = ffn.FusedFFN(dev)
    for _ in range(5):
        h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
    torch.cuda.synchronize()
    n = 200  # (below the launch-queue depth: 2000 calls of a 30 us kernel fill it and time the GPU)
    t0 = time.perf_counter()
    for _ in range(n):
        h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    res[f"{M}x{K}x{N}"] = round((t1 - t0) / n * 1e6, 2)
print(sys.argv[1], "host us per eager forward (enqueue only):", res, flush=True)

# breakdown at the decode shape: the binding's Python work vs the C call alone
M, K, N = 16, 4096, 11008
t = make_device_inputs(M, K, N, 3, dev)
out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
h = ffn.FusedFFN(dev)
h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
torch.cuda.synchronize()
args = (h._h, t["x"].data_ptr(), t["g"].data_ptr(), t["w1"].data_ptr(), t["w3"].data_ptr(), out.data_ptr(), M, K, N,
        1e-6, torch.cuda.current_stream(dev).cuda_stream)
n = 2000
for label, fn in (("C call only", lambda: h.lib.cuasm_ffn_forward(*args)),
                  ("validate", lambda: h._validate(t["x"], t["g"], t["w1"], t["w3"], out)),
                  ("weights_changed", lambda: h._weights_changed({0: (t["g"], t["w1"], t["w3"])})),
                  ("current_stream", lambda: torch.cuda.current_stream(dev).cuda_stream)):
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"  {label:18s} {(t1 - t0) / n * 1e6:6.2f} us", flush=True)

# other entry points' C calls: small kernels with few parameters
r = torch.empty((M,), dtype=torch.float32, device=dev)
xn = torch.empty_like(t["x"])
s_ = torch.cuda.current_stream(dev).cuda_stream
for label, fn in (("rms_inv C call", lambda: h.lib.cuasm_ffn_rms_inv(h._h, t["x"].data_ptr(), r.data_ptr(), M, K, 1e-6, s_)),
                  
                  ("torch add_", lambda: r.add_(1.0))):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"  {label:18s} {(t1 - t0) / n * 1e6:6.2f} us", flush=True)

# device time per eager forward (host far ahead): would reveal a re-pack per call
M, K, N = 16, 4096, 11008
t = make_device_inputs(M, K, N, 3, dev)
out = torch.empty((M, N), dtype=torch.bfloat16, device=dev)
h = ffn.FusedFFN(dev)
for _ in range(3):
    h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(int(5e8))
e0.record()
for _ in range(500):
    h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
e1.record()
torch.cuda.synchronize()
print(f"  device us per eager forward (decode, back to back): {e0.elapsed_time(e1) / 500 * 1e3:.2f}", flush=True)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, out=out)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=6), flush=True)
